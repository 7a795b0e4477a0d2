/*
 * proxsaga.h — C ABI of the B200 (sm_100a) Sparse Proximal SAGA / ProxASAGA
 * hot path (libproxsaga.so).
 *
 * The reference (`sparsesaga`, /root/reference/pkg/src/sparsesaga) runs the
 * SPS step in Python and exposes one native module, `_atomics`
 * (_atomics.c:306-335), whose element-level atomics the Python worker loop
 * calls five times per update (asynchronous.py:92-116).  On B200 the whole
 * worker loop runs on the device, so the boundary moves up one level: each
 * entry point below replaces a reference routine (cited per function) and
 * operates on DEVICE memory owned by the caller (borrowed for the call, like
 * the Py_buffer views of _atomics.c:16-30).  No torch / CPython types appear.
 *
 * Conventions
 *   - all pointers are device pointers unless stated; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream);
 *   - return value: PS_OK or an error code; ps_last_error() gives the text.
 *     The Python layer maps PS_EINVAL -> ValueError, PS_ERANGE -> IndexError,
 *     PS_ECUDA -> RuntimeError, the conventions of _atomics.c:26,36 and
 *     saga.py:89-95;
 *   - coordinate state is one 32-byte record per feature j
 *       coord[4j+0] = x_j, coord[4j+1] = abar_j, coord[4j+2] = D_j (weight),
 *       coord[4j+3] = hot-slot tag (reserved)
 *     so the x / abar / D gather of one coordinate is one 32-byte sector.
 */
#ifndef PROXSAGA_H
#define PROXSAGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 3

enum ps_status { PS_OK = 0, PS_EINVAL = 1, PS_ERANGE = 2, PS_ECUDA = 3, PS_ENOMEM = 4 };
/* losses.py:15-19 */
enum ps_loss { PS_LOSS_LOGISTIC = 0, PS_LOSS_SQUARED = 1 };
/* penalties.py:56-138 */
enum ps_penalty { PS_PEN_ZERO = 0, PS_PEN_L1 = 1, PS_PEN_GROUP = 2, PS_PEN_BOX = 3 };
enum ps_dtype { PS_F32 = 0, PS_F64 = 1 };
enum ps_itype { PS_I32 = 0, PS_I64 = 1 };
/* data.py:164-191: singleton / contiguous groups (G coords each) / general */
enum ps_part_kind { PS_PART_SINGLETON = 0, PS_PART_CONTIG = 1, PS_PART_GENERAL = 2 };

/* Row-major CSR, data.py:31-72.  Columns strictly increasing per row. */
typedef struct ps_csr {
    int64_t n_rows, n_cols, nnz;
    const void *row_ptr;     /* n_rows+1, int32 or int64 (row_ptr_type) */
    const int32_t *col_idx;  /* nnz */
    const void *values;      /* nnz, fp32 or fp64 (value_type); widened to fp64 before use */
    const void *labels;      /* n_rows, same type as values */
    int32_t row_ptr_type;    /* ps_itype */
    int32_t value_type;      /* ps_dtype */
} ps_csr_t;

/* Block partition + extended-support index, data.py:121-161, 194-297. */
typedef struct ps_part {
    int32_t kind;            /* ps_part_kind */
    int32_t G;               /* CONTIG: block size (block b = [bG, min(bG+G,p)) ) */
    int64_t n_blocks;
    /* GENERAL only (host-provided partition description): */
    const int32_t *block_of; /* p */
    const int32_t *blk_ptr;  /* n_blocks+1 */
    const int32_t *blk_coords; /* p, sorted within each block */
    /* filled by ps_prepare (device, caller-allocated): */
    int32_t *blk_count;      /* n_blocks: n_B */
    double *blk_weight;      /* n_blocks: d_B = n/n_B, 0 if dead */
    int32_t *row_blk;        /* GENERAL: nnz slots, row i's sorted T_i at row_ptr[i].. */
    int32_t *row_g;          /* GENERAL: |T_i| */
    int32_t *spos;           /* GENERAL: nnz, ext slot of each nonzero */
    int32_t max_slots;       /* set by ps_prepare: max ext slots over rows */
    int32_t max_row_nnz;     /* set by ps_prepare: max nonzeros of a row */
} ps_part_t;

typedef struct ps_params {
    int32_t loss;            /* ps_loss */
    int32_t penalty;         /* ps_penalty */
    double lambda1;          /* Loss.lambda1 (losses.py:22-31) */
    double lam2;             /* L1Penalty / GroupL2Penalty weight */
    double lo, hi;           /* BoxPenalty */
    double gamma;            /* resolved step (saga.py:25-42) */
} ps_params_t;

/* Problem statistics written by ps_prepare (host struct). */
typedef struct ps_stats {
    int64_t max_count;       /* max_B n_B  (delta = max_count / n, data.py:262) */
    int64_t n_dead;          /* blocks with n_B = 0 (DeadBlockError, data.py:255-257) */
    double max_row_sqnorm;   /* max_i ||a_i||^2 (losses.py:99-105) */
    int32_t max_row_nnz;
    int32_t max_slots;
} ps_stats_t;

/* Sample schedule of one ps_run call. */
typedef struct ps_sched {
    const int64_t *samples;  /* non-NULL: replay this sequence (deterministic, saga.py:233-256) */
    int64_t count;           /* updates to perform */
    uint64_t seed;           /* samples == NULL: on-device counter-based sampler stream */
    uint64_t slot_base;      /* first slot of the stream used by this call (resume) */
    unsigned long long *counter; /* device: slots claimed so far (asynchronous.py:68-72) */
    int32_t batch;           /* 0: static split of the slots over warps (split_iterations,
                                asynchronous.py:125-128), counter bumped once per warp;
                                > 0: warps claim `batch` slots at a time from the counter */
    int32_t ctas;            /* 0 = one wave at full occupancy */
    int32_t warps_per_cta;   /* 0 = default */
    int32_t hot_cols;        /* H of ps_hot_layout: columns [0,H) staged in shared memory (async) */
    double contention;       /* c > 0: per-coordinate step gamma_j = gamma * min(1, c * D_j / tau),
                                tau = effective delay in updates (async only; the fixed point is
                                unchanged); 0 = plain gamma (the reference's step) */
    int32_t hot_period;      /* CTA updates between hot flushes (0 = default) */
    int32_t flags;           /* PS_FLAG_* below (0 = defaults) */
    int32_t hot_shift;       /* log2 of the hot-record stride of ps_hot_layout */
    int32_t reserved;
    /* deterministic mode only (NULL = off), p doubles each, device: per
     * coordinate of T_i of each replayed step, the gradient estimate v of
     * sparse_gradient_estimate (saga.py:150-166) and the applied delta z - x^
     * (worker_iteration's return value, asynchronous.py:97-117).  The
     * reference's step-level entry points (sps_step, worker_iteration,
     * sparse_gradient_estimate) read them after a one-sample replay. */
    double *trace_v;
    double *trace_dx;
} ps_sched_t;

/* ps_sched_t.flags (async only; diagnostics except where noted) */
#define PS_FLAG_SCRAMBLE 4        /* permute the slot order within the call */
#define PS_FLAG_GENERIC 16        /* force the generic kernel (no pipelined fast path) */
#define PS_FLAG_GROUP_WARP 64     /* group lasso: the warp-cooperative kernel even when staging */
#define PS_FLAG_GROUP_LANE 128    /* group lasso: the lane-per-block kernel without staging */
#define PS_FLAG_DELTA_ZERO 32     /* commit prox-zeroed coordinates as the delta -x_hat, the
                                     reference's literal scatter_add (asynchronous.py:105-107);
                                     default: store 0 */
/* bits 8..15: extra divisor of the staged columns' contention scale */
#define PS_FLAG_MON_DEVICE_X 524288 /* ps_run_monitored: snaps is DEVICE memory of max_snaps*p doubles and
                                        receives x only (stride 1), copied by a few CTAs beside the solve,
                                        whose default grid leaves them their SMs (host snapshots of a large
                                        problem's records take longer than an epoch over PCIe) */
#define PS_FLAG_MON_ENDS_IN_PLACE 65536 /* ps_run_monitored: skip the copies of the first and last
                                           snapshots (the caller reads coord itself) */
#define PS_FLAG_ZERO_IMMEDIATE 131072 /* fast kernel: a staged coordinate the prox zeroes is stored by
                                         the update itself, not by the CTA's next flush (DESIGN.md
                                         "zero commits"; diagnostics) */
#define PS_FLAG_GROUP_STORE_ZEROS 262144 /* lane-per-block group kernel, unstaged blocks: also store a
                                            block that was read as zero and stays zero (default: its
                                            zero delta is skipped; diagnostics) */
#define PS_FLAG_FAST_V1 4194304   /* singleton fast path: the round-1 kernel (sps_fast_kernel: dirty bitmasks,
                                      two pending copies) instead of sps_hot_kernel (A/B, diagnostics) */
#define PS_FLAG_NO_CLUSTER 2097152 /* fast kernel: no CTA pairs (each CTA refreshes its hot snapshot
                                      from L2; default: clusters of 2 share one refresh) */
#define PS_FLAG_LOCAL_VIEW 134217728 /* hot kernel: a staged commit also writes its prox result into the
                                        CTA's snapshot (the CTA reads its own commits at once; opt-in,
                                        DESIGN.md K2'' "local view") */

int ps_abi_version(void);
const char *ps_last_error(void);
int ps_device_count(void);

/* data.py:236-297 (build_support_index) + losses.py:99-105: block counts,
 * weights d_B, delta, dead blocks, max ||a_i||^2, per-row T_i (GENERAL), and
 * the per-coordinate weight D_j written into coord[4j+2].  Synchronous;
 * `stats` is host memory. */
int ps_prepare(const ps_csr_t *csr, ps_part_t *part, double *coord, ps_stats_t *stats, void *stream);

/* Scratch bytes ps_run needs in global memory for `warps` resident warps
 * (0 when every row fits the register path). */
int64_t ps_scratch_bytes(const ps_csr_t *csr, const ps_part_t *part, int32_t warps);

/* The grid ps_run will launch for this schedule (occupancy-derived when
 * sched->ctas == 0) and the global scratch it then needs (0 when the
 * per-warp scratch fits shared memory or is not needed). */
int ps_launch_config(const ps_csr_t *csr, const ps_part_t *part, const ps_sched_t *sched,
                     int32_t *ctas, int32_t *warps_per_cta, int64_t *scratch_bytes);

/* The SPS inner loop.
 *   sched->samples != NULL: deterministic replay on one warp — saga.py:248-256
 *     around sps_step (:169-185); fp64 iterates agree with the reference.
 *   sched->samples == NULL: ProxASAGA, one warp per in-flight sample,
 *     inconsistent reads, atomicAdd commits on x / abar, atomicExch on alpha_i —
 *     asynchronous.py:131-210 around worker_iteration (:80-117).
 * `scratch` may be NULL when ps_scratch_bytes() == 0. */
int ps_run(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, double *coord,
           double *alpha, const ps_sched_t *sched, void *scratch, void *stream);

/* losses.py:134-136 full_objective, computed from x at stride `x_stride`
 * doubles.  out (device, 3 doubles) = {mean loss, 0.5*lambda1*||x||^2, h(x)}. */
int ps_objective(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm,
                 const double *x, int32_t x_stride, double *out, void *stream);

/* losses.py:118-122 smooth_gradient: grad = A^T l'(Ax)/n + lambda1 x. */
int ps_smooth_gradient(const ps_csr_t *csr, const ps_params_t *prm, const double *x,
                       int32_t x_stride, double *grad, void *stream);

/* saga.py:299-317 fixed_point_residual; `grad` is p doubles of workspace;
 * out (device, 1 double) = ||x - prox_{gamma D phi}(x - gamma D grad f(x))||. */
int ps_fixed_point_residual(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm,
                            const double *coord, double *grad, double *out, void *stream);

/* saga.py:75-78 resync_average: abar = A^T alpha / n, into coord[4j+1]. */
int ps_resync_average(const ps_csr_t *csr, const double *alpha, double *coord, void *stream);

/* penalties.py:78-81,103-108,134-135,60-61: prox of a vector v[m] with
 * per-coordinate effective step eff[m] (separable) or eff[0] for the whole
 * vector as ONE block (group, prox_block). */
int ps_prox(const ps_params_t *prm, const double *v, const double *eff, int64_t m, double *out,
            void *stream);

/* losses.py:73-86 loss derivative, elementwise: out[i] = l'(z[i], b[i]).
 * fast = 0: the deterministic kernels' arithmetic (libdevice exp, IEEE
 * division: bit-identical to the reference's scalar formula); fast = 1: the
 * asynchronous hot kernel's (sps_hot_kernel: table exp + one-Newton reciprocal
 * division, ~1 ulp); fast = 2: the round-1 fast kernel's (sps_fast_kernel).
 * Device pointers; an inspection / test hook for the kernels' loss code. */
int ps_loss_deriv(int32_t loss, int32_t fast, const double *z, const double *b, int64_t m, double *out,
                  void *stream);

/* Lambda-batched group-lasso SPS (a regularisation path, BASELINE config 5):
 * B in {1,2,4,8,16} solves of the same problem that differ only in the group
 * weight lam2[beta] (device, B doubles; prm->lam2 is ignored), sharing each
 * sampled row: saga.py:150-185 / asynchronous.py:80-117 per state.  State:
 * ps_batch_state_doubles(p, G, B) doubles (NB = ceil(p/G)), coordinate j of
 * state beta at (beta/S)*RPAD + (((beta/S)*NB*G + j)*S + beta%S)*2 + {0: x, 1: abar}
 * with S = min(B, 2) and RPAD the region pad (use ps_batch_field); alpha[i*B + beta]; d_B from ps_prepare (part->blk_weight).
 * CONTIG partitions of G <= 16, rows <= 32 nonzeros, int32 row pointers.
 * sched->samples != NULL: deterministic replay of the sequence on one warp
 * (every state takes the same samples); else asynchronous, one warp per
 * in-flight row (sched->counter counts rows). */
int ps_batch_run(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *lam2,
                 int32_t B, double *state, double *alpha, const ps_sched_t *sched, void *stream);
/* ps_batch_run with replicated x-delta accumulators for the hottest blocks of a
 * spread hot-unit layout (ps_hot_layout; sched->hot_shift = its log2 stride):
 * in asynchronous mode the nrb most frequent stored units (unit r << hot_shift,
 * r < nrb) commit their x deltas to one of nrep replicas (chosen by warp), so a
 * hot block's REDs queue on nrep L2 lines instead of one; reads sum the state
 * and the replicas, and the replicas are folded into the state after the
 * launch (same stream).  xrep: device, nrep*nrb*G*B doubles, zero on entry and
 * left zero.  nrep = 0 or xrep = NULL: ps_batch_run. */
int ps_batch_run_rep(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *lam2,
                     int32_t B, double *state, double *alpha, const ps_sched_t *sched, double *xrep, int32_t nrep,
                     int32_t nrb, void *stream);
/* doubles of a ps_batch_run state for p coordinates, blocks of G, B states
 * (regions of two states: the contiguous records, the scattered hot blocks' area, the pad), and of the
 * replica accumulators of ps_batch_run_rep */
int64_t ps_batch_state_doubles(int64_t p, int32_t G, int32_t B);
int64_t ps_batch_rep_doubles(int32_t nrep, int32_t nrb, int32_t G, int32_t B);
/* diagnostics: the state's region pad and the replica chunk stride, in doubles
 * (process-wide; allocate states after setting them) */
int ps_batch_tune(int64_t rpad, int64_t rstride);
/* diagnostics: the scattered hot blocks of the batched state -- the nhot most frequent stored
 * blocks (stored index rank << hot_shift: ps_hot_layout's spread order) keep coordinate q in the
 * region's hot area at (rank*G + q)*hstride doubles, one sector per hstride (defaults: 128 blocks
 * from B = 8 and 32 below (nhot = -1), 128 doubles = 1 KB; nhot = 0 or hstride = 0: every block in
 * the contiguous record).
 * hshare: a warp loads stored block 0 from L2 on every hshare-th of its rows and reads the CTA's
 * shared copy of it on the others (default 4; 0 = every row).  hab: a hot slot keeps the states' x in
 * one sector and their abar in another, hab doubles later (default -1: 64 = 512 B from B = 4, packed
 * below; needs hstride >= hab + 2;
 * 0 = one packed (x, abar) sector as everywhere else).
 * Process-wide; allocate states after setting */
int ps_batch_tune2(int32_t nhot, int64_t hstride, int32_t hshare, int32_t hab);
/* the grid (CTAs, warps per CTA: rows in flight = their product) of this process's last ps_batch_run launch */
int ps_batch_last_grid(int32_t *ctas, int32_t *warps_per_cta);
/* field (0 x, 1 abar) of state beta <-> a p-vector (set = 0: state -> vec, 1: vec -> state);
 * hot_shift = the ps_sched_t.hot_shift the state is run with (it places the scattered hot blocks) */
int ps_batch_field(double *state, int64_t p, int32_t G, int32_t B, int32_t hot_shift, int32_t beta, int32_t field,
                   double *vec, int32_t set, void *stream);

/* losses.py:73-86 loss_scalar, elementwise: value[i] = l(z[i], b[i]) (overflow-safe
 * log1p forms) and deriv[i] = l'(z[i], b[i]), the deterministic kernels' arithmetic;
 * either output may be NULL.  Device pointers. */
int ps_loss_eval(int32_t loss, const double *z, const double *b, int64_t m, double *value, double *deriv,
                 void *stream);

/* Hot layout (SINGLETON: unit = 1, columns; CONTIG: unit = G, whole blocks):
 * units present in at least max(ceil(min_frac * n), theta) rows — theta the
 * smallest threshold letting at most hot_max units qualify — are the H hot
 * units; hot rank r is stored at unit index r * S (S = *stride_inout, a power
 * of two, reduced until S * H <= #units) so consecutive hot records sit in
 * different L2 slices; cold units fill the remaining indices in original
 * order.  The device CSR's columns (col_inout) are remapped in place and each
 * row re-sorted (values in val_inout move along), so rows stay strictly
 * increasing (data.py:58-61).  perm[old coordinate] = new coordinate (p
 * int32); counts_ws: ceil(p/unit) int32.  Coordinates are padded to whole
 * units: *p_pad_out = ceil(p/unit) * unit (padding never touched).  The SPS
 * kernel stages hot units in shared memory (sched->hot_cols = H,
 * sched->hot_shift = log2 S).  Synchronous; H / S / p_pad are host memory. */
int ps_hot_layout(const ps_csr_t *csr, int32_t *col_inout, void *val_inout, int32_t unit,
                  int32_t hot_max, double min_frac, int32_t *stride_inout, int32_t *counts_ws,
                  int32_t *perm, int32_t *H_out, int64_t *p_pad_out, void *stream);

/* Solver state to x0 = 0, abar = 0, alpha = 0, counter = 0 (D untouched):
 * saga.py:231-232. `counter` may be NULL. */
int ps_state_reset(double *coord, int64_t p, double *alpha, int64_t n, unsigned long long *counter,
                   void *stream);

/* One asynchronous ps_run with the reference's live monitor
 * (asynchronous.py:181-198): this call blocks, polls sched->counter and, each
 * time it crosses a multiple of `every`, copies the live coordinate records
 * (p x 4 doubles, an inconsistent snapshot while the warps keep updating) into
 * snaps[k] (pinned HOST memory: a copy-engine DMA beside the kernel).  snaps[0] is the state before the first update,
 * the last one the state after the launch; snap_counts / snap_ms (host) get
 * the counter value and the device time (ms since the launch) of each;
 * *n_snaps <= max_snaps.  The solve never stops for a checkpoint.  With
 * PS_FLAG_MON_ENDS_IN_PLACE in sched->flags, snaps[0] and the last snapshot
 * are not copied (their counts and times are still reported): the caller
 * evaluates those two states on coord itself, before and after the call.
 * With PS_FLAG_MON_DEVICE_X, snaps is device memory and each snapshot is x
 * only (p doubles). */
int ps_run_monitored(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, double *coord,
                     double *alpha, const ps_sched_t *sched, void *scratch, void *stream, int64_t every,
                     int32_t max_snaps, double *snaps, int64_t *snap_counts, float *snap_ms, int32_t *n_snaps);

/* Fenchel dual objective at the dual point induced by x (theta_i = -l'(a_i.x, b_i)):
 * out[0] = D, out[1] = the scaling applied to theta (lambda1 = 0 with L1 / group,
 * else 1); duality gap = ps_objective - D >= 0.  No reference counterpart (the
 * north star's "duality-gap evaluation"); formulas in aux.cu. */
int ps_dual_objective(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *x,
                      int32_t x_stride, double *out, void *stream);

/* FISTA (fista.py:38-58): x_new = prox_{h/L}(y - grad * inv_L) over all p
 * coordinates (group penalty: per block of `part`), sums[0] = grad.(x_new - y),
 * sums[1] = ||x_new - y||^2 (device); and y = x_new + beta (x_new - x). */
int ps_fista_prox(const ps_part_t *part, const ps_params_t *prm, const double *y, const double *grad,
                  double inv_L, int64_t p, double *x_new, double *sums, void *stream);
int ps_fista_extrapolate(const double *x_new, const double *x, double beta, int64_t p, double *y, void *stream);

/* LibSVM text -> CSR on the device (the reference's parse_libsvm,
 * data.py:309-363).  `buf` holds the file's bytes on the device.
 * ps_libsvm_index: start offset of each of the m lines (m = newlines + a final
 * unterminated line).  ps_libsvm_scan: per line the label, feature count,
 * status (0 ok, 1 blank/comment, 3 token without ':' at byte detail[j],
 * 4 non-increasing index detail[j], 5 parse this line on the host: a number
 * outside the exact fast path) and the largest index of the OK lines.
 * ps_libsvm_fill: the OK lines' (idx - 1, value) pairs at
 * row_ptr[row_of_line[j]]. */
int ps_libsvm_index(const uint8_t *buf, int64_t n, int64_t *line_start, int64_t m, void *stream);
int ps_libsvm_scan(const uint8_t *buf, int64_t n, const int64_t *line_start, int64_t m, double *labels,
                   int32_t *nfeat, int32_t *status, int64_t *detail, unsigned long long *max_idx, void *stream);
int ps_libsvm_fill(const uint8_t *buf, int64_t n, const int64_t *line_start, int64_t m, const int32_t *status,
                   const int64_t *row_of_line, const int64_t *row_ptr, int64_t *cols, double *vals, void *stream);

/* *dst = the device's %globaltimer (ns), stream-ordered (capturable into a
 * CUDA graph): checkpoint timing of DeviceProblem.run_async_checkpointed. */
int ps_timestamp(unsigned long long *dst, void *stream);

/* coord record <-> plain vectors: field 0 = x, 1 = abar, 2 = D. */
int ps_coord_get(const double *coord, int64_t p, int32_t field, double *out, void *stream);
int ps_coord_set(double *coord, int64_t p, int32_t field, const double *in, void *stream);
/* same through a column permutation: out[j] = coord[4 perm[j] + field] */
int ps_coord_get_perm(const double *coord, int64_t p, int32_t field, const int32_t *perm, double *out,
                      void *stream);
int ps_coord_set_perm(double *coord, int64_t p, int32_t field, const int32_t *perm, const double *in,
                      void *stream);

/* K7 device generator for BASELINE configs 3/4: n rows of
 * k = k_dense + k_zipf distinct sorted columns — [0, k_dense) in every
 * row, the rest (k_zipf <= 32, k <= 64) drawn Zipf by inverse CDF (cdf[m], device, increasing to 1)
 * over [k_dense, k_dense + m) with resample-until-distinct; values 1
 * (lognormal = 0) or lognormal(0,1), rows l2-normalised.  row_ptr int64[n+1],
 * col int32[n*k], val fp32[n*k]. */
int ps_gen_zipf_csr(int64_t n, int32_t k_dense, int32_t k_zipf, const double *cdf, int64_t m,
                    uint64_t seed, int32_t lognormal, int64_t *row_ptr, int32_t *col, float *val,
                    void *stream);
/* labels y_i = sign(a_i . w + noise N(0,1)), sign(0) = +1, for the generated CSR */
int ps_gen_labels(int64_t n, int32_t k, const int32_t *col, const float *val, const double *w,
                  double noise, uint64_t seed, float *y, void *stream);

/* _atomics.c primitives, device-scope, on caller buffers (test + tooling):
 *   gather      (_atomics.c:163-209)  out[k] = arr[idx[k]]   (L2-coherent loads)
 *   scatter_add (_atomics.c:212-258)  arr[idx[k]] += d[k]     (atomicAdd f64)
 *   exchange    (_atomics.c:260-283)  old[k] = swap(arr[idx[k]], val[k])
 *   fetch_add_i64 (_atomics.c:285-304)
 *   add_repeat  (_atomics.c:136-158)  threads x count adds of delta on one cell
 * Indices are bounds-checked on device: PS_ERANGE if any is outside [0, len). */
int ps_atomic_gather(const double *arr, int64_t len, const int64_t *idx, int64_t m, double *out,
                     void *stream);
int ps_atomic_scatter_add(double *arr, int64_t len, const int64_t *idx, int64_t m, const double *d,
                          void *stream);
int ps_atomic_exchange(double *arr, int64_t len, const int64_t *idx, int64_t m, const double *val,
                       double *old, void *stream);
int ps_atomic_fetch_add_i64(long long *arr, int64_t len, int64_t i, long long delta, long long *old,
                            void *stream);
int ps_atomic_add_repeat(double *cell, double delta, int64_t count, int32_t threads, void *stream);

#ifdef __cplusplus
}
#endif
#endif
