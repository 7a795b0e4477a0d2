/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 CPU restatement of the reference's Sparse Proximal SAGA
 * hot path (package `sparsesaga`, /root/reference/pkg/src/sparsesaga).  It is
 * the checker the CUDA path is compared against and the CPU baseline arm of
 * bench.py ("kind": "port").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * package never does.
 *
 * Pinning: tests/test_oracle.py checks this restatement against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py imports the
 * reference package in the build container) and against the reference tests'
 * own known answers.
 *
 * Every function cites the reference file:line it restates.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { LOSS_LOGISTIC = 0, LOSS_SQUARED = 1 };
enum { PEN_ZERO = 0, PEN_L1 = 1, PEN_GROUP = 2, PEN_BOX = 3 };

typedef struct {
    int64_t n, p;
    const int64_t *row_ptr;   /* n+1 */
    const int64_t *col;       /* nnz, strictly increasing per row */
    const double *val;        /* nnz */
    const double *y;          /* n */
    int64_t n_blocks;
    const int64_t *block_of;  /* p */
    const int64_t *blk_ptr;   /* n_blocks+1 : coords of block b = blk_coords[blk_ptr[b]:blk_ptr[b+1]] (sorted) */
    const int64_t *blk_coords;/* p */
    const double *d_B;        /* n_blocks */
    int loss;
    double lambda1;
    int pen;
    double lam2, lo, hi;
    int singleton;            /* block_of == identity: T_i = S_i (fast path, same arithmetic) */
} oracle_problem;

/* losses.py:73-86 (loss_scalar): branchy, overflow-safe logistic. */
static inline double deriv(int loss, double z, double b)
{
    if (loss == LOSS_LOGISTIC) {
        double t = -b * z, sig;
        if (t > 0) {
            sig = 1.0 / (1.0 + exp(-t));
        } else {
            double et = exp(t);
            sig = et / (1.0 + et);
        }
        return -b * sig;
    }
    return z - b;
}

static inline double loss_value(int loss, double z, double b)
{
    if (loss == LOSS_LOGISTIC) { /* losses.py:53-59 (_log1pexp) */
        double t = -b * z;
        if (t > 0) return t + log1p(exp(-t));
        return log1p(exp(t));
    }
    double d = z - b;
    return 0.5 * d * d;
}

/* data.py:236-262 (build_support_index): n_B = #rows whose support meets B,
 * d_B = n/n_B (0 for dead blocks), delta = max n_B / n.  Returns #dead. */
int64_t oracle_block_weights(int64_t n, const int64_t *row_ptr, const int64_t *col,
                             int64_t n_blocks, const int64_t *block_of,
                             int64_t *counts, double *d_B, double *delta)
{
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_blocks > 0 ? n_blocks : 1));
    for (int64_t b = 0; b < n_blocks; b++) { last[b] = -1; counts[b] = 0; }
    for (int64_t i = 0; i < n; i++)
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
            int64_t b = block_of[col[e]];
            if (last[b] != i) { last[b] = i; counts[b]++; }
        }
    int64_t dead = 0, mx = 0;
    for (int64_t b = 0; b < n_blocks; b++) {
        if (counts[b] > 0) d_B[b] = (double)n / (double)counts[b];
        else { d_B[b] = 0.0; dead++; }
        if (counts[b] > mx) mx = counts[b];
    }
    *delta = mx > 0 ? (double)mx / (double)n : 0.0;
    free(last);
    return dead;
}

/* Per-thread scratch for one step. */
typedef struct {
    int64_t cap;
    int64_t *coords, *blocks, *pos;
    double *w, *xe, *ae, *v, *z;
    char *mark; /* n_blocks */
    int64_t *tmp;
} scratch_t;

static void scratch_init(scratch_t *s, const oracle_problem *P, int64_t cap)
{
    s->cap = cap;
    s->coords = malloc(sizeof(int64_t) * cap);
    s->blocks = malloc(sizeof(int64_t) * cap);
    s->pos = malloc(sizeof(int64_t) * cap);
    s->w = malloc(sizeof(double) * cap);
    s->xe = malloc(sizeof(double) * cap);
    s->ae = malloc(sizeof(double) * cap);
    s->v = malloc(sizeof(double) * cap);
    s->z = malloc(sizeof(double) * cap);
    s->tmp = malloc(sizeof(int64_t) * cap);
    s->mark = calloc((size_t)P->n_blocks, 1);
}

static void scratch_free(scratch_t *s)
{
    free(s->coords); free(s->blocks); free(s->pos); free(s->w); free(s->xe);
    free(s->ae); free(s->v); free(s->z); free(s->tmp); free(s->mark);
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* data.py:249-283: extended support of row i = sorted coordinates of the
 * blocks meeting S_i, with per-coordinate weights d_B and the positions of
 * S_i inside it.  Returns m (number of ext coords), fills s->blocks[0:g]. */
static int64_t ext_support(const oracle_problem *P, int64_t i, scratch_t *s, int64_t *g_out)
{
    int64_t lo = P->row_ptr[i], hi = P->row_ptr[i + 1];
    int64_t g = 0;
    if (P->singleton) {
        for (int64_t e = lo; e < hi; e++) {
            s->coords[e - lo] = s->blocks[e - lo] = P->col[e];
            s->w[e - lo] = P->d_B[P->col[e]];
            s->pos[e - lo] = e - lo;
        }
        *g_out = hi - lo;
        return hi - lo;
    }
    for (int64_t e = lo; e < hi; e++) {
        int64_t b = P->block_of[P->col[e]];
        if (!s->mark[b]) { s->mark[b] = 1; s->blocks[g++] = b; }
    }
    qsort(s->blocks, (size_t)g, sizeof(int64_t), cmp_i64);
    int64_t m = 0;
    for (int64_t t = 0; t < g; t++) {
        int64_t b = s->blocks[t];
        s->mark[b] = 0;
        for (int64_t q = P->blk_ptr[b]; q < P->blk_ptr[b + 1]; q++) s->tmp[m++] = P->blk_coords[q];
    }
    /* sorted coordinate order (data.py:271-273) */
    memcpy(s->coords, s->tmp, sizeof(int64_t) * (size_t)m);
    qsort(s->coords, (size_t)m, sizeof(int64_t), cmp_i64);
    for (int64_t q = 0; q < m; q++) s->w[q] = P->d_B[P->block_of[s->coords[q]]];
    /* positions of S_i (data.py:278, np.searchsorted) — both lists sorted */
    int64_t q = 0;
    for (int64_t e = lo; e < hi; e++) {
        while (s->coords[q] != P->col[e]) q++;
        s->pos[e - lo] = q;
    }
    *g_out = g;
    return m;
}

static inline int64_t bsearch_pos(const int64_t *a, int64_t m, int64_t key)
{
    int64_t lo = 0, hi = m;
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (a[mid] < key) lo = mid + 1; else hi = mid; }
    return lo;
}

/* penalties.py:170-186 (prox_extended_slice) on u = s->v (in place into s->z). */
static void prox_slice(const oracle_problem *P, double gamma, scratch_t *s, int64_t m, int64_t g)
{
    if (P->pen == PEN_GROUP) { /* non-separable: per block, penalties.py:103-108 */
        for (int64_t q = 0; q < m; q++) s->z[q] = s->v[q];
        for (int64_t t = 0; t < g; t++) {
            int64_t b = s->blocks[t];
            double ss = 0.0;
            for (int64_t c = P->blk_ptr[b]; c < P->blk_ptr[b + 1]; c++) {
                double u = s->v[bsearch_pos(s->coords, m, P->blk_coords[c])];
                ss += u * u;
            }
            double norm = sqrt(ss);
            double eff = gamma * P->d_B[b];
            double f = (norm == 0.0) ? 0.0 : fmax(0.0, 1.0 - eff * P->lam2 / norm);
            for (int64_t c = P->blk_ptr[b]; c < P->blk_ptr[b + 1]; c++) {
                int64_t q = bsearch_pos(s->coords, m, P->blk_coords[c]);
                s->z[q] = (norm == 0.0) ? 0.0 : s->v[q] * f;
            }
        }
        return;
    }
    for (int64_t q = 0; q < m; q++) {
        double u = s->v[q];
        if (P->pen == PEN_L1) { /* penalties.py:78-81 */
            double thr = (gamma * s->w[q]) * P->lam2;
            double a = fmax(fabs(u) - thr, 0.0);
            s->z[q] = (u > 0) ? a : (u < 0 ? -a : 0.0);
        } else if (P->pen == PEN_BOX) { /* penalties.py:134-135 */
            s->z[q] = u < P->lo ? P->lo : (u > P->hi ? P->hi : u);
        } else {
            s->z[q] = u; /* penalties.py:60-61 */
        }
    }
}

/* ---- atomics (restating _atomics.c:42-75,260-283 with C11 builtins) ---- */
static inline double a_load(const double *c)
{
    uint64_t bits = __atomic_load_n((const uint64_t *)c, __ATOMIC_SEQ_CST);
    double d; memcpy(&d, &bits, 8); return d;
}
static inline void a_add(double *c, double delta)
{
    uint64_t exp_bits = __atomic_load_n((uint64_t *)c, __ATOMIC_SEQ_CST);
    for (;;) {
        double cur; memcpy(&cur, &exp_bits, 8);
        double upd = cur + delta; uint64_t des; memcpy(&des, &upd, 8);
        if (__atomic_compare_exchange_n((uint64_t *)c, &exp_bits, des, 0, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST))
            return;
    }
}
static inline double a_exch(double *c, double v)
{
    uint64_t bits; memcpy(&bits, &v, 8);
    uint64_t old = __atomic_exchange_n((uint64_t *)c, bits, __ATOMIC_SEQ_CST);
    double d; memcpy(&d, &old, 8); return d;
}

/* One step.  atomic=0: saga.py:150-185 (sparse_gradient_estimate + sps_step);
 * atomic=1: asynchronous.py:80-117 (worker_iteration). */
static void step(const oracle_problem *P, int64_t i, double gamma, double *x, double *alpha,
                 double *abar, scratch_t *s, int atomic)
{
    int64_t lo = P->row_ptr[i], hi = P->row_ptr[i + 1], k = hi - lo, g = 0;
    int64_t m = ext_support(P, i, s, &g);
    double old;
    for (int64_t q = 0; q < m; q++) s->xe[q] = atomic ? a_load(&x[s->coords[q]]) : x[s->coords[q]];
    old = atomic ? a_load(&alpha[i]) : alpha[i];
    for (int64_t q = 0; q < m; q++) s->ae[q] = atomic ? a_load(&abar[s->coords[q]]) : abar[s->coords[q]];
    double margin = 0.0;                             /* saga.py:162 */
    for (int64_t e = 0; e < k; e++) margin += P->val[lo + e] * s->xe[s->pos[e]];
    double nw = deriv(P->loss, margin, P->y[i]);      /* saga.py:163 */
    for (int64_t q = 0; q < m; q++)                   /* saga.py:164 */
        s->v[q] = s->w[q] * (s->ae[q] + P->lambda1 * s->xe[q]);
    for (int64_t e = 0; e < k; e++)                   /* saga.py:165 */
        s->v[s->pos[e]] += (nw - old) * P->val[lo + e];
    if (m) {
        for (int64_t q = 0; q < m; q++) s->v[q] = s->xe[q] - gamma * s->v[q];   /* saga.py:180 */
        prox_slice(P, gamma, s, m, g);
        for (int64_t q = 0; q < m; q++) {
            if (atomic) a_add(&x[s->coords[q]], s->z[q] - s->xe[q]);        /* asynchronous.py:104-106 */
            else x[s->coords[q]] = s->xe[q] + (s->z[q] - s->xe[q]);         /* saga.py:181 */
        }
    }
    double replaced = atomic ? a_exch(&alpha[i], nw) : old;                 /* asynchronous.py:113 */
    double t = (nw - replaced) / (double)P->n;                              /* saga.py:182-184 */
    for (int64_t e = 0; e < k; e++) {
        if (atomic) a_add(&abar[P->col[lo + e]], t * P->val[lo + e]);
        else abar[P->col[lo + e]] += t * P->val[lo + e];
    }
    if (!atomic) alpha[i] = nw;                                             /* saga.py:185 */
}

static int64_t max_ext(const oracle_problem *P)
{
    /* upper bound on m: sum of block sizes over a row's distinct blocks <= p */
    return P->p > 0 ? P->p : 1;
}

/* saga.py:248-256: replay a fixed sample sequence sequentially. */
int oracle_run_sequential(const oracle_problem *P, double gamma, const int64_t *samples, int64_t count,
                          double *x, double *alpha, double *abar)
{
    scratch_t s;
    scratch_init(&s, P, max_ext(P));
    for (int64_t t = 0; t < count; t++) step(P, samples[t], gamma, x, alpha, abar, &s, 0);
    scratch_free(&s);
    return 0;
}

/* ---- asynchronous.py:131-210: lock-free Hogwild workers (pthreads) ---- */
typedef struct {
    const oracle_problem *P;
    double gamma;
    const int64_t *samples;
    int64_t count;
    double *x, *alpha, *abar;
    int64_t *counter;
    int64_t batch;
} worker_arg;

static void *worker_main(void *vp)
{
    worker_arg *a = (worker_arg *)vp;
    scratch_t s;
    scratch_init(&s, a->P, max_ext(a->P));
    int64_t pending = 0;
    for (int64_t t = 0; t < a->count; t++) {
        step(a->P, a->samples[t], a->gamma, a->x, a->alpha, a->abar, &s, 1);
        if (++pending == a->batch) { __atomic_fetch_add(a->counter, pending, __ATOMIC_SEQ_CST); pending = 0; }
    }
    if (pending) __atomic_fetch_add(a->counter, pending, __ATOMIC_SEQ_CST);
    scratch_free(&s);
    return NULL;
}

/* samples: concatenation of per-worker sequences, counts[w] each
 * (asynchronous.py:120-128: split_iterations + worker_sample_sequence). */
int oracle_run_async(const oracle_problem *P, double gamma, int threads, const int64_t *samples,
                     const int64_t *counts, double *x, double *alpha, double *abar, int64_t *counter,
                     int64_t batch)
{
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)threads);
    worker_arg *args = malloc(sizeof(worker_arg) * (size_t)threads);
    int64_t off = 0;
    for (int w = 0; w < threads; w++) {
        args[w] = (worker_arg){P, gamma, samples + off, counts[w], x, alpha, abar, counter, batch};
        off += counts[w];
        pthread_create(&th[w], NULL, worker_main, &args[w]);
    }
    for (int w = 0; w < threads; w++) pthread_join(th[w], NULL);
    free(th); free(args);
    return 0;
}

/* losses.py:134-136 (full_objective) = smooth_value (:112-115) + penalty.value
 * (penalties.py:75-76, :97-101 with the partition, :128-132). */
double oracle_objective(const oracle_problem *P, const double *x)
{
    double acc = 0.0;
    for (int64_t i = 0; i < P->n; i++) {
        double z = 0.0;
        for (int64_t e = P->row_ptr[i]; e < P->row_ptr[i + 1]; e++) z += P->val[e] * x[P->col[e]];
        acc += loss_value(P->loss, z, P->y[i]);
    }
    double sm = acc / (double)P->n, xx = 0.0;
    for (int64_t j = 0; j < P->p; j++) xx += x[j] * x[j];
    sm += 0.5 * P->lambda1 * xx;
    double pen = 0.0;
    if (P->pen == PEN_L1) {
        for (int64_t j = 0; j < P->p; j++) pen += fabs(x[j]);
        pen *= P->lam2;
    } else if (P->pen == PEN_GROUP) {
        for (int64_t b = 0; b < P->n_blocks; b++) {
            double ss = 0.0;
            for (int64_t c = P->blk_ptr[b]; c < P->blk_ptr[b + 1]; c++) ss += x[P->blk_coords[c]] * x[P->blk_coords[c]];
            pen += sqrt(ss);
        }
        pen *= P->lam2;
    } else if (P->pen == PEN_BOX) {
        for (int64_t j = 0; j < P->p; j++)
            if (!(x[j] >= P->lo && x[j] <= P->hi)) return INFINITY;
    }
    return sm + pen;
}

/* losses.py:118-122 (smooth_gradient): A^T l'(Ax)/n + lambda1 x. */
void oracle_smooth_gradient(const oracle_problem *P, const double *x, double *grad)
{
    for (int64_t j = 0; j < P->p; j++) grad[j] = 0.0;
    for (int64_t i = 0; i < P->n; i++) {
        double z = 0.0;
        for (int64_t e = P->row_ptr[i]; e < P->row_ptr[i + 1]; e++) z += P->val[e] * x[P->col[e]];
        double d = deriv(P->loss, z, P->y[i]);
        for (int64_t e = P->row_ptr[i]; e < P->row_ptr[i + 1]; e++) grad[P->col[e]] += d * P->val[e];
    }
    for (int64_t j = 0; j < P->p; j++) grad[j] = grad[j] / (double)P->n + P->lambda1 * x[j];
}

/* saga.py:299-317 (fixed_point_residual). */
double oracle_fixed_point_residual(const oracle_problem *P, const double *x, double gamma)
{
    double *grad = malloc(sizeof(double) * (size_t)P->p);
    double *inner = malloc(sizeof(double) * (size_t)P->p);
    oracle_smooth_gradient(P, x, grad);
    for (int64_t j = 0; j < P->p; j++) inner[j] = x[j] - gamma * P->d_B[P->block_of[j]] * grad[j];
    double res = 0.0;
    if (P->pen == PEN_GROUP) {
        for (int64_t b = 0; b < P->n_blocks; b++) {
            double ss = 0.0;
            for (int64_t c = P->blk_ptr[b]; c < P->blk_ptr[b + 1]; c++) ss += inner[P->blk_coords[c]] * inner[P->blk_coords[c]];
            double norm = sqrt(ss), eff = gamma * P->d_B[b];
            double f = norm == 0.0 ? 0.0 : fmax(0.0, 1.0 - eff * P->lam2 / norm);
            for (int64_t c = P->blk_ptr[b]; c < P->blk_ptr[b + 1]; c++) {
                int64_t j = P->blk_coords[c];
                double z = norm == 0.0 ? 0.0 : inner[j] * f, d = x[j] - z;
                res += d * d;
            }
        }
    } else {
        for (int64_t j = 0; j < P->p; j++) {
            double u = inner[j], z;
            if (P->pen == PEN_L1) {
                double thr = (gamma * P->d_B[P->block_of[j]]) * P->lam2, a = fmax(fabs(u) - thr, 0.0);
                z = u > 0 ? a : (u < 0 ? -a : 0.0);
            } else if (P->pen == PEN_BOX) z = u < P->lo ? P->lo : (u > P->hi ? P->hi : u);
            else z = u;
            double d = x[j] - z;
            res += d * d;
        }
    }
    free(grad); free(inner);
    return sqrt(res);
}

/* _atomics.c:136-158 (add_repeat): threads x count seq-cst CAS adds. */
typedef struct { double *cell; double delta; int64_t count; } rep_arg;
static void *rep_main(void *vp)
{
    rep_arg *a = vp;
    for (int64_t k = 0; k < a->count; k++) a_add(a->cell, a->delta);
    return NULL;
}
void oracle_add_repeat_threads(double *cell, double delta, int64_t count, int threads)
{
    pthread_t th[64];
    rep_arg a = {cell, delta, count};
    if (threads > 64) threads = 64;
    for (int w = 0; w < threads; w++) pthread_create(&th[w], NULL, rep_main, &a);
    for (int w = 0; w < threads; w++) pthread_join(th[w], NULL);
}
