// The Sparse Proximal SAGA inner loop on sm_100a (ps_run).
//
// One warp owns one in-flight sample.  Per update it
//   1. reads row i of the CSR (coalesced: one nonzero per lane),
//   2. gathers x^, abar and D on the row's (extended) support -- one 32-byte
//      coordinate record per coordinate, L2-coherent loads ("inconsistent
//      read", asynchronous.py:92-96),
//   3. warp-shuffle dot product -> margin -> loss derivative
//      (saga.py:161-163, losses.py:73-86),
//   4. v = D (abar + lambda1 x^) + (new - alpha_i) a_i  (saga.py:164-165),
//      z = prox_{gamma D}(x^ - gamma v)  (penalties.py:170-186),
//   5. commits x += z - x^ (atomicAdd, asynchronous.py:104-106) -- or, when
//      the prox returns exactly 0, stores the 0 (
//      PS_FLAG_DELTA_ZERO keeps the literal delta) -- alpha_i <-> new
//      (atomicExch, :113), abar += ((new-replaced)/n) a_i (atomicAdd, :114-116).
//
// Kernels: sps_kernel (deterministic replay + generic async, any layout),
// sps_fast_kernel (async singleton rows <= 64 nnz: 1024-thread CTAs, a
// three-stage row pipeline, hot columns staged per CTA in shared memory),
// sps_group_kernel / sps_group_lane_kernel (async group lasso on contiguous
// blocks: warp-cooperative, or one lane per block with optional staging).
// Deterministic mode (sched->samples != NULL) replays a fixed sequence on a
// single warp with plain stores in the exact order of sps_step
// (saga.py:169-185): x = x^ + (z - x^), abar += (delta/n) vals, alpha_i = new.
//
// Three support layouts (ps_part kind):
//   SINGLETON  T_i = S_i; rows <= 64 nonzeros stay in registers (fast path),
//              longer rows go through the per-warp slot scratch.
//   CONTIG     blocks of G <= 32 contiguous coordinates (config 5); T_i is
//              derived on the fly from the sorted columns (block = col / G),
//              blocks are processed G lanes per block with a segmented
//              shuffle reduction for the group norm.
//   GENERAL    any BlockPartition; T_i / slot positions precomputed by
//              ps_prepare; blocks processed one at a time.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace ps {

struct KArgs {
    const void *row_ptr;
    const int32_t *col;
    const void *val;
    const void *y;
    int64_t n, p;
    double n_d;
    // partition
    int32_t G;
    const int32_t *blk_ptr, *blk_coords;
    const int32_t *row_blk, *row_g, *spos;
    const double *blk_weight;
    // state
    double *coord;
    double *alpha;
    // params
    int32_t loss, pen;
    double lambda1, lam2, lo, hi, gamma;
    double kappa;      // contention scale c / tau (INFINITY: plain gamma)
    double kappa_hot;  // the same for shared-memory-staged hot columns
    // schedule
    const int64_t *samples;
    int64_t count;
    uint64_t seed, slot_base;
    unsigned long long *counter;
    int32_t batch;
    int32_t det;
    // hot-column staging (SINGLETON, async): columns [0, H) live in shared memory
    int32_t H;          // 0 = off
    int32_t period;     // CTA updates between flushes of the pending deltas
    int32_t hot_doubles;  // shared doubles used by the staging area
    int32_t hot_shift;    // hot unit r is stored at unit index r << hot_shift
    int32_t hot_unit;     // coordinates per hot unit (1: columns, G: contiguous blocks)
    uint64_t scramble;    // diagnostics: 0, or an odd multiplier coprime to count (slot -> slot*m mod count)
    int32_t diag;         // ps_sched_t.flags (PS_FLAG_*)
    int32_t cluster;      // fast kernel: CTAs per thread-block cluster (1: none)
    int32_t ncopy;        // sps_hot_kernel: pending-delta copies per CTA
    // deterministic step outputs (ps_sched_t.trace_v / trace_dx), per coordinate
    double *trace_v, *trace_dx;
    // scratch
    double *gscratch;
    int32_t stride;  // doubles per warp
    int32_t smem;    // scratch lives in dynamic shared memory
    int32_t M, GB;   // slot / block capacity per warp
};

constexpr int NCH_MAX = 2;  // register fast path: rows of up to NCH*32 nonzeros (NCH=1 for 1024-thread CTAs)

template <typename PT> __device__ __forceinline__ int64_t rp(const void *p, int64_t i)
{
    return (int64_t)__ldg(reinterpret_cast<const PT *>(p) + i);
}
template <typename VT> __device__ __forceinline__ double rv(const void *p, int64_t e)
{
    return widen(__ldg(reinterpret_cast<const VT *>(p) + e));
}

// alpha_i read (lane 0, broadcast): asynchronous.py:94.
__device__ __forceinline__ double load_alpha(const KArgs &a, int64_t i, int lane)
{
    double old = 0.0;
    if (lane == 0) old = ld_cg(a.alpha + i);
    return __shfl_sync(FULL, old, 0);
}

// alpha_i <- new; returns the value replaced (asynchronous.py:113 / saga.py:185).
__device__ __forceinline__ double swap_alpha(const KArgs &a, int64_t i, double nw, double old, int lane)
{
    double rep = old;
    if (lane == 0) {
        if (a.det) a.alpha[i] = nw;
        else rep = atomic_exch(a.alpha + i, nw);
    }
    return __shfl_sync(FULL, rep, 0);
}

// Per-coordinate step gamma_j = gamma * min(1, kappa * D_j): damps only the
// coordinates that more than c of the tau in-flight updates touch at once
// (expected concurrent writers tau / D_j).  kappa = +inf -> exactly gamma.
__device__ __forceinline__ double step_of(const KArgs &a, double d)
{
    return a.gamma * fmin(1.0, a.kappa * d);
}

__device__ __forceinline__ void commit_x(const KArgs &a, int64_t c, double xh, double z)
{
    if (a.det) a.coord[4 * c] = xh + (z - xh);
    else if (z == 0.0 && !(a.diag & PS_FLAG_DELTA_ZERO)) atomic_exch(a.coord + 4 * c, 0.0);  // see store_zero
    else red_add(a.coord + 4 * c, z - xh);
}

__device__ __forceinline__ void commit_abar(const KArgs &a, int64_t c, double inc)
{
    if (a.det) {
        double *p = a.coord + 4 * c + 1;
        *p = ld_cg(p) + inc;
    } else {
        red_add(a.coord + 4 * c + 1, inc);
    }
}

// ---------------------------------------------------------------------------
// Hot-column staging.  Per CTA, in shared memory:
//   hx[H], hab[H], hd[H]  snapshot of x, abar, D of the hot columns
//   pend[NCOPY][2][H]     pending x / abar deltas of this CTA (fp64, smem atomics)
// Hot reads come from the snapshot (an inconsistent read, like any other);
// hot commits go to the pending arrays; each warp, after every `period` of
// its own updates, flushes the CTA's pending -> global with one RED per dirty
// (column, field) and refreshes the snapshot (~one flush per `period` CTA
// updates).  Cuts same-sector L2 atomics on the Zipf head by ~period x.
constexpr int NCOPY = 2;
// staging header after the hot area (unsigned words): dirty[0..31], the
// refresh rotation counter [32], spare [33], zero-store mask [34..65]
constexpr int HDR_DOUBLES = 33;
constexpr int ZMASK = 34;

// shared-memory layout of the staging area (doubles):
//   [0, 2H)            snapshot pairs (x_s, abar_s), 16 B each (cp.async target)
//   [2H, 3H)           D_s
//   [3H, 3H+2*NCOPY*H) pending x / abar deltas, NCOPY copies
struct HotView {
    double *xab, *d, *pend;
    int H;
};

__device__ __forceinline__ HotView hot_view(double *base, int H)
{
    return HotView{base, base + 2 * H, base + 3 * H, H};
}

__device__ __forceinline__ void mark_dirty(unsigned *dirty, int slot)
{
    unsigned *w = dirty + (slot & 31), b = 1u << (slot >> 5);
    if (!(*(volatile unsigned *)w & b)) atomicOr(w, b);
}

// a staged coordinate the prox zeroed: the store x_j = 0 is issued once by the
// CTA's next flush instead of by every update (same-address global atomics on
// the hottest records otherwise queue at L2)
__device__ __forceinline__ void mark_zero(unsigned *dirty, int slot)
{
    unsigned *w = dirty + ZMASK + (slot & 31), b = 1u << (slot >> 5);
    if (!(*(volatile unsigned *)w & b)) atomicOr(w, b);
}

__device__ __forceinline__ double smem_take(double *p)
{
    return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long *>(p), 0ull));
}
// discard this CTA's pending x delta of a staged slot (its coordinate is being stored)
__device__ __forceinline__ void drop_pending_x(const HotView &h, int s)
{
#pragma unroll
    for (int c = 0; c < NCOPY; c++) {
        double *p = h.pend + (2 * c) * h.H + s;
        if (*(volatile double *)p != 0.0) atomicExch(reinterpret_cast<unsigned long long *>(p), 0ull);
    }
}

// flush this CTA's pending deltas to global, then refresh the snapshot.
// Lane l owns slots l, l+32, ... (HOT_PER_LANE of them; the hottest columns
// spread over lanes); `dirty[l]` has bit k set when slot l+32k has pending
// deltas.  REDs are fire-and-forget and the snapshot refresh is a set of
// cp.async global->shared copies, so the flushing warp never waits on memory.
constexpr int HOT_PER_LANE = 32;  // H <= 1024 (dirty bitmask: one 32-bit word per lane)
constexpr int HOT_MAX = 32 * HOT_PER_LANE;
constexpr int HOT_TIER0 = 128;  // slots refreshed on every flush
constexpr int PROGRESS_BATCH = 16;  // fast kernel: updates per progress bump of a warp (into its CTA's count)
constexpr int CTA_PROGRESS = 512;   // ... and of a CTA into the global counter

// global coordinate of hot slot s: unit s / U stored at unit (s / U) << hot_shift
__device__ __forceinline__ int64_t hot_coord(const KArgs &a, int s)
{
    if (a.hot_unit <= 1) return (int64_t)s << a.hot_shift;
    int r = s / a.hot_unit, q = s - r * a.hot_unit;
    return (((int64_t)r << a.hot_shift) * a.hot_unit) + q;
}

struct FlushArgs {  // what the flush needs, by value (keeps KArgs out of local memory)
    double *coord;
    int shift, unit;
    unsigned lead = 0u;  // shared::cluster address of the cluster leader's staging area (0: none)
};
__device__ __forceinline__ int64_t hot_coord(const FlushArgs &f, int s)
{
    if (f.unit <= 1) return (int64_t)s << f.shift;
    int r = s / f.unit, q = s - r * f.unit;
    return (((int64_t)r << f.shift) * f.unit) + q;
}
__device__ __noinline__ void hot_flush(const FlushArgs fa, const int H, unsigned *dirty, int lane, bool refresh)
{
    extern __shared__ double smem_dyn[];  // the staging area starts the dynamic shared memory
    double *pend = smem_dyn + 3 * H;
    unsigned zm = atomicExch(dirty + ZMASK + lane, 0u);
    unsigned m = atomicExch(dirty + lane, 0u) | zm;
    while (m) {
        int k = __ffs(m) - 1;
        m &= m - 1;
        int s = lane + 32 * k;
        if (s >= H) continue;
        double dx = 0.0, dab = 0.0;
#pragma unroll
        for (int c = 0; c < NCOPY; c++) {
            dx += smem_take(pend + (2 * c) * H + s);
            dab += smem_take(pend + (2 * c + 1) * H + s);
        }
        double *g = fa.coord + 4 * hot_coord(fa, s);
        if ((zm >> k) & 1u) atomic_exch(g, 0.0);  // deferred zero store, then the deltas added since
        if (dx != 0.0) red_add(g, dx);
        if (dab != 0.0) red_add(g + 1, dab);
    }
    if (!refresh) return;
    // tiered refresh: the HOT_TIER0 hottest slots every flush, the rest a
    // rotating quarter per flush (their columns change ~p_j times slower)
    unsigned rot = 0;
    if (lane == 0) rot = atomicAdd(dirty + 32, 1u);
    rot = __shfl_sync(FULL, rot, 0) & 3u;
    const int kmax = (H + 31) >> 5;
    if (fa.lead) {
        // cluster member: refresh from the leader CTA's snapshot through
        // distributed shared memory instead of from the hot records in L2,
        // where the reads queue behind every CTA's REDs to the same lines
        for (int k = 0; k < kmax; k++) {
            int s = lane + 32 * k;
            if (s < H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
                double2 v;
                asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(fa.lead + 16u * s));
                reinterpret_cast<double2 *>(smem_dyn)[s] = v;
            }
        }
        return;
    }
    for (int k = 0; k < kmax; k++) {
        int s = lane + 32 * k;
        if (s < H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
            unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dyn + 2 * s);
            const double *src = fa.coord + 4 * hot_coord(fa, s);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void hot_async_drain() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Group-lasso flush (sps_group_kernel): hot blocks accumulate the samples'
// gradient steps (pending x) and a sample count; the flush applies ONE block
// prox with the summed threshold, prox_{m g D lam ||.||}(x^_B + sum_k -g v_k),
// and commits its delta -- a mini-batch proximal step whose fixed point is the
// optimum (-grad_B f in lam d||x_B||).  Per-sample group prox on a stale
// snapshot rectifies noise (||c + noise|| > ||c||) into a bias; summing first
// averages the noise against an m-fold threshold.  abar deltas as usual.
__device__ __noinline__ void hot_flush_group(const KArgs &a, const HotView &h, int *bcnt, int lane, bool refresh)
{
    extern __shared__ double smem_dyn[];
    const int H = h.H, G = a.G, HB = H / G;
    double *pend = smem_dyn + 3 * H;
    for (int r = lane; r < HB; r += 32) {
        // current global (x, abar) of the block: the prox must act on the value
        // the delta is added to (the snapshot may predate our previous flush)
        double2 cur[16];
#pragma unroll
        for (int q = 0; q < 16; q++)
            if (q < G) cur[q] = ld_cg2(a.coord + 4 * hot_coord(a, r * G + q));
        const int m = atomicExch(bcnt + r, 0);
        double u[16], ss = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q++) {
            if (q < G) {
                const int s = r * G + q;
                double st = 0.0;
#pragma unroll
                for (int c = 0; c < NCOPY; c++) st += smem_take(pend + (2 * c) * H + s);
                u[q] = cur[q].x + st;
                ss += u[q] * u[q];
            }
        }
        double f = 1.0;
        if (m > 0) {
            const double d = smem_dyn[2 * H + r * G];
            const double eff = (double)m * a.gamma * fmin(1.0, a.kappa_hot * d) * d;
            f = group_factor(sqrt(ss), eff, a.lam2);
        }
#pragma unroll
        for (int q = 0; q < 16; q++) {
            if (q < G) {
                const int s = r * G + q;
                const double z = m > 0 ? u[q] * f : u[q];
                const double dz = z - cur[q].x;
                double dab = 0.0;
#pragma unroll
                for (int c = 0; c < NCOPY; c++) dab += smem_take(pend + (2 * c + 1) * H + s);
                double *gp = a.coord + 4 * hot_coord(a, s);
                if (z == 0.0 && !(a.diag & PS_FLAG_DELTA_ZERO)) atomic_exch(gp, 0.0);
                else if (dz != 0.0) red_add(gp, dz);
                if (dab != 0.0) red_add(gp + 1, dab);
                if (refresh) {
                    smem_dyn[2 * s] = z;
                    smem_dyn[2 * s + 1] = cur[q].y + dab;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// SINGLETON fast path: k <= NCH*32, everything in registers.
template <typename VT, int NCH>
__device__ __forceinline__ void row_reg(const KArgs &a, int64_t i, int64_t lo, int k, int lane, const HotView &h,
                                        double *px, double *pab, unsigned *dirty)
{
    int colr[NCH], slot[NCH];
    double vr[NCH], xr[NCH], abr[NCH], dr[NCH];
    double part = 0.0;
    const int hmask = (1 << a.hot_shift) - 1, hlim = h.H << a.hot_shift;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        int e = c * 32 + lane;
        colr[c] = -1;
        slot[c] = -1;
        if (e < k) {
            int col = __ldg(a.col + lo + e);
            colr[c] = col;
            vr[c] = rv<VT>(a.val, lo + e);
            if (col < hlim && (col & hmask) == 0) slot[c] = col >> a.hot_shift;
            if (slot[c] >= 0) {
                const int sl = slot[c];
                double2 v = reinterpret_cast<const double2 *>(h.xab)[sl];
                xr[c] = v.x;
                abr[c] = v.y;
                dr[c] = h.d[sl];
            } else {
                double2 xa = ld_cg2(a.coord + 4 * (int64_t)col);
                xr[c] = xa.x;
                abr[c] = xa.y;
                dr[c] = __ldg(a.coord + 4 * (int64_t)col + 2);
            }
            part += vr[c] * xr[c];
        }
    }
    double old = load_alpha(a, i, lane);
    double y = rv<VT>(a.y, i);
    double margin = warp_sum(part);
    double nw = loss_deriv(a.loss, margin, y);
    double ds = nw - old;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        if (colr[c] >= 0) {
            double v = dr[c] * (abr[c] + a.lambda1 * xr[c]);
            v += ds * vr[c];
            double g = slot[c] >= 0 ? a.gamma * fmin(1.0, a.kappa_hot * dr[c]) : step_of(a, dr[c]);
            double u = xr[c] - g * v;
            double z = prox_sep(a.pen, u, g * dr[c], a.lam2, a.lo, a.hi);
            if (a.trace_v) {
                a.trace_v[colr[c]] = v;
                a.trace_dx[colr[c]] = z - xr[c];
            }
            if (slot[c] >= 0 && (z != 0.0 || (a.diag & PS_FLAG_DELTA_ZERO))) {
                atomicAdd(px + slot[c], z - xr[c]);
                mark_dirty(dirty, slot[c]);
            } else {
                if (slot[c] >= 0) drop_pending_x(h, slot[c]);
                commit_x(a, colr[c], xr[c], z);
            }
        }
    }
    double rep = swap_alpha(a, i, nw, old, lane);
    double t = (nw - rep) / a.n_d;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        if (colr[c] >= 0) {
            if (a.det) a.coord[4 * (int64_t)colr[c] + 1] = abr[c] + t * vr[c];
            else if (slot[c] >= 0) {
                atomicAdd(pab + slot[c], t * vr[c]);
                mark_dirty(dirty, slot[c]);
            }
            else red_add(a.coord + 4 * (int64_t)colr[c] + 1, t * vr[c]);
        }
    }
}

// ---------------------------------------------------------------------------
// Slot path: the extended support is laid out as m "slots" in per-warp
// scratch (shared or global memory):
//   sa[s] row value at slot s (0 when the coordinate is not in S_i)
//   sx[s] x^ at slot s, sv[s] = D (abar^ + lambda1 x^), sw[s] = D
//   si[s] coordinate id of slot s (-1 = padding), sb[t] block id of rank t,
//   so[t] first slot of block rank t (GENERAL).
struct Scratch {
    double *sa, *sx, *sv, *sw;
    int *si, *sb, *so;
};

__device__ __forceinline__ Scratch carve(double *base, int M, int GB)
{
    Scratch s;
    s.sa = base;
    s.sx = base + M;
    s.sv = base + 2 * M;
    s.sw = base + 3 * M;
    s.si = reinterpret_cast<int *>(base + 4 * M);
    s.sb = s.si + M;
    s.so = s.sb + GB;
    return s;
}

template <typename VT, int PART>
__device__ void row_slots(const KArgs &a, int64_t i, int64_t lo, int k, int lane, const Scratch &S)
{
    const unsigned lt = (1u << lane) - 1u;
    int g = 0, m = 0;
    // ---- 1. blocks of T_i and slot count
    if (PART == PS_PART_SINGLETON) {
        m = k;
    } else if (PART == PS_PART_CONTIG) {
        int carry = 0, prevblk = -1;
        for (int base = 0; base < k; base += 32) {
            int e = base + lane;
            int blk = e < k ? __ldg(a.col + lo + e) / a.G : -1;
            int up = __shfl_up_sync(FULL, blk, 1);
            if (lane == 0) up = prevblk;
            bool isnew = (e < k) && (blk != up);
            unsigned bal = __ballot_sync(FULL, isnew);
            if (isnew) S.sb[carry + __popc(bal & lt)] = blk;
            carry += __popc(bal);
            prevblk = __shfl_sync(FULL, blk, 31);
        }
        g = carry;
        m = g * a.G;
    } else {  // GENERAL
        g = __ldg(a.row_g + i);
        int carry = 0;
        for (int base = 0; base < g; base += 32) {
            int t = base + lane;
            int b = 0, sz = 0;
            if (t < g) {
                b = __ldg(a.row_blk + lo + t);
                sz = __ldg(a.blk_ptr + b + 1) - __ldg(a.blk_ptr + b);
                S.sb[t] = b;
            }
            int incl = sz;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            if (t < g) S.so[t] = carry + incl - sz;
            carry += __shfl_sync(FULL, incl, 31);
        }
        m = carry;
        if (lane == 0) S.so[g] = m;
    }
    __syncwarp();
    // ---- 2. slot -> coordinate map, zero the row-value slots
    if (PART == PS_PART_GENERAL) {
        for (int t = 0; t < g; t++) {
            int b = S.sb[t], off = S.so[t];
            int cb = __ldg(a.blk_ptr + b), sz = __ldg(a.blk_ptr + b + 1) - cb;
            for (int q = lane; q < sz; q += 32) S.si[off + q] = __ldg(a.blk_coords + cb + q);
        }
    }
    for (int s = lane; s < m; s += 32) {
        S.sa[s] = 0.0;
        if (PART == PS_PART_SINGLETON) {
            S.si[s] = __ldg(a.col + lo + s);
        } else if (PART == PS_PART_CONTIG) {
            int64_t c = (int64_t)S.sb[s / a.G] * a.G + (s % a.G);
            S.si[s] = c < a.p ? (int)c : -1;
        }
    }
    __syncwarp();
    // ---- 3. scatter the row values into their slots
    if (PART == PS_PART_CONTIG) {
        int carry = 0, prevblk = -1;
        for (int base = 0; base < k; base += 32) {
            int e = base + lane;
            int col = e < k ? __ldg(a.col + lo + e) : 0;
            int blk = e < k ? col / a.G : -1;
            int up = __shfl_up_sync(FULL, blk, 1);
            if (lane == 0) up = prevblk;
            bool isnew = (e < k) && (blk != up);
            unsigned bal = __ballot_sync(FULL, isnew);
            int rank = carry + __popc(bal & (lt | (1u << lane))) - 1;
            if (e < k) S.sa[rank * a.G + (col - blk * a.G)] = rv<VT>(a.val, lo + e);
            carry += __popc(bal);
            prevblk = __shfl_sync(FULL, blk, 31);
        }
    } else {
        for (int e = lane; e < k; e += 32) {
            int s = PART == PS_PART_SINGLETON ? e : __ldg(a.spos + lo + e);
            S.sa[s] = rv<VT>(a.val, lo + e);
        }
    }
    __syncwarp();
    // ---- 4. gather x^, abar^, D on the extended support; partial margin
    double part = 0.0;
    for (int s = lane; s < m; s += 32) {
        int c = S.si[s];
        double xh = 0.0, v0 = 0.0, w = 0.0;
        if (c >= 0) {
            double2 xa = ld_cg2(a.coord + 4 * (int64_t)c);
            w = __ldg(a.coord + 4 * (int64_t)c + 2);
            xh = xa.x;
            v0 = w * (xa.y + a.lambda1 * xh);
        }
        S.sx[s] = xh;
        S.sv[s] = v0;
        S.sw[s] = w;
        part += S.sa[s] * xh;
    }
    double old = load_alpha(a, i, lane);
    double y = rv<VT>(a.y, i);
    double margin = warp_sum(part);
    double nw = loss_deriv(a.loss, margin, y);
    double ds = nw - old;
    __syncwarp();
    // ---- 5. prox + commit x on T_i
    if (a.pen != PS_PEN_GROUP) {
        for (int s = lane; s < m; s += 32) {
            int c = S.si[s];
            if (c < 0) continue;
            double xh = S.sx[s];
            double v = S.sv[s] + ds * S.sa[s];
            double g = step_of(a, S.sw[s]);
            double u = xh - g * v;
            double z = prox_sep(a.pen, u, g * S.sw[s], a.lam2, a.lo, a.hi);
            if (a.trace_v) {
                a.trace_v[c] = v;
                a.trace_dx[c] = z - xh;
            }
            commit_x(a, c, xh, z);
        }
    } else if (PART == PS_PART_CONTIG) {
        // G lanes per block, bpc blocks per pass; segmented shuffle reduce.
        const int G = a.G, bpc = 32 / G;
        const int q = lane % G, tb = lane / G;
        for (int t0 = 0; t0 < g; t0 += bpc) {
            int t = t0 + tb;
            bool on = (tb < bpc) && (t < g);
            int s = t * G + q;
            int c = on ? S.si[s] : -1;
            double xh = 0.0, u = 0.0, dB = 0.0;
            if (c >= 0) {
                dB = a.blk_weight[S.sb[t]];
                xh = S.sx[s];
                double v = S.sv[s] + ds * S.sa[s];
                u = xh - step_of(a, dB) * v;
                if (a.trace_v) a.trace_v[c] = v;
            }
            double sq = u * u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                double r = __shfl_down_sync(FULL, sq, o);
                if (q + o < G && lane + o < 32) sq += r;
            }
            double ss = __shfl_sync(FULL, sq, lane - q);
            if (c >= 0) {
                double eff = step_of(a, dB) * dB;
                double f = group_factor(sqrt(ss), eff, a.lam2);
                if (a.trace_v) a.trace_dx[c] = u * f - xh;
                commit_x(a, c, xh, u * f);
            }
        }
    } else {  // GENERAL group: block at a time
        for (int t = 0; t < g; t++) {
            int off = S.so[t], sz = S.so[t + 1] - off;
            double dB = a.blk_weight[S.sb[t]];
            double gB = step_of(a, dB);
            double sq = 0.0;
            for (int q = lane; q < sz; q += 32) {
                int s = off + q;
                double u = S.sx[s] - gB * (S.sv[s] + ds * S.sa[s]);
                sq += u * u;
            }
            double ss = warp_sum(sq);
            double f = group_factor(sqrt(ss), gB * dB, a.lam2);
            for (int q = lane; q < sz; q += 32) {
                int s = off + q;
                double xh = S.sx[s];
                const double v = S.sv[s] + ds * S.sa[s];
                double u = xh - gB * v;
                if (a.trace_v) {
                    a.trace_v[S.si[s]] = v;
                    a.trace_dx[S.si[s]] = u * f - xh;
                }
                commit_x(a, S.si[s], xh, u * f);
            }
        }
    }
    // ---- 6. alpha swap, abar on S_i
    double rep = swap_alpha(a, i, nw, old, lane);
    double tt = (nw - rep) / a.n_d;
    for (int e = lane; e < k; e += 32) {
        int c = __ldg(a.col + lo + e);
        commit_abar(a, c, tt * rv<VT>(a.val, lo + e));
    }
    __syncwarp();
}

template <typename VT, typename PT, int PART, int MAXT>
__global__ void __launch_bounds__(MAXT) sps_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    // shared layout: [hot staging (hot_doubles) | dirty[32] + counters + zero mask[32] (HDR_DOUBLES) | per-warp scratch]
    HotView h = hot_view(smem_dyn, a.H);
    unsigned *dirty = reinterpret_cast<unsigned *>(smem_dyn + a.hot_doubles);
    double *px = h.pend + (2 * (wib % NCOPY)) * a.H, *pab = px + a.H;
    Scratch S{};
    if constexpr (MAXT <= 256) {  // the 1024-thread variant only runs rows of <= 32 nonzeros
        if (a.stride > 0) {
            const int hdr = a.H > 0 ? a.hot_doubles + HDR_DOUBLES : 0;
            double *base = a.smem ? smem_dyn + hdr + (int64_t)wib * a.stride : a.gscratch + gw * a.stride;
            S = carve(base, a.M, a.GB);
        }
    }
    if (a.H > 0) {
        for (int s = threadIdx.x; s < a.H; s += blockDim.x) {
            const double *g = a.coord + 4 * hot_coord(a, s);
            reinterpret_cast<double2 *>(h.xab)[s] = ld_cg2(g);
            h.d[s] = __ldg(g + 2);
        }
        for (int s = threadIdx.x; s < 2 * NCOPY * a.H; s += blockDim.x) h.pend[s] = 0.0;
        if (threadIdx.x < 2 * HDR_DOUBLES) dirty[threadIdx.x] = 0u;
        __syncthreads();
    }
    // async work split (asynchronous.py:125-128 split_iterations): warp gw owns
    // the contiguous slot range [s0, s1) of this call; no atomics on the way.
    // With batch > 0 warps instead claim `batch` slots at a time from the
    // device counter (dynamic scheduling; diagnostics).
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t q = a.count / nwarps, r = a.count % nwarps;
    uint64_t slot = (uint64_t)(gw * q + min(gw, r));
    uint64_t slot_end = a.batch > 0 ? 0 : slot + (uint64_t)(q + (gw < r ? 1 : 0));
    if (a.batch > 0) slot = 0;
    int64_t t = 0;
    // each warp flushes the CTA's pending hot deltas after every `period` of its
    // own updates (staggered start), i.e. about once per `period` CTA updates
    int until_flush = a.H > 0 ? 1 + (wib * a.period) / max(1, (int)(blockDim.x >> 5)) : 0;
    while (true) {
        int64_t i;
        if (a.det) {
            if (t >= a.count) break;
            i = __ldg(a.samples + t);
            t++;
        } else {
            if (slot >= slot_end) {
                if (a.batch <= 0) break;
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(a.counter, (unsigned long long)a.batch);
                base = __shfl_sync(FULL, base, 0);
                if (base >= (unsigned long long)a.count) break;
                slot = base;
                slot_end = min((uint64_t)(base + a.batch), (uint64_t)a.count);
            }
            uint64_t sl = a.scramble ? (slot * a.scramble) % (uint64_t)a.count : slot;
            i = sample_row(a.seed, a.slot_base + sl, (uint64_t)a.n);
            slot++;
        }
        int64_t lo = rp<PT>(a.row_ptr, i);
        int k = (int)(rp<PT>(a.row_ptr, i + 1) - lo);
        if constexpr (MAXT > 256) {
            row_reg<VT, 1>(a, i, lo, k, lane, h, px, pab, dirty);
        } else {
            if (PART == PS_PART_SINGLETON && k <= NCH_MAX * 32) row_reg<VT, NCH_MAX>(a, i, lo, k, lane, h, px, pab, dirty);
            else row_slots<VT, PART>(a, i, lo, k, lane, S);
        }
        if (a.det) {
            __threadfence();
            __syncwarp();
        }
        if (a.H > 0 && --until_flush == 0) {
            hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit}, a.H, dirty, lane, true);
            until_flush = a.period;
        }
        // progress counter, bumped every PROGRESS_BATCH updates of the warp (the
        // workers' counter_batch, asynchronous.py:155-162): the live monitor reads it
        if (!a.det && a.batch <= 0 && lane == 0 && ++t % PROGRESS_BATCH == 0)
            atomicAdd(a.counter, (unsigned long long)PROGRESS_BATCH);
    }
    if (!a.det && a.batch <= 0 && lane == 0 && t % PROGRESS_BATCH)  // the remainder
        atomicAdd(a.counter, (unsigned long long)(t % PROGRESS_BATCH));
    if (a.H > 0) {  // every warp of the CTA has left the loop: final flush
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            dirty[lane] = HOT_PER_LANE >= 32 ? 0xffffffffu : (0xffffffffu >> (32 - HOT_PER_LANE));  // every slot
            __syncwarp();
            hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit}, a.H, dirty, lane, false);
        }
        hot_async_drain();
    }
}


// ---------------------------------------------------------------------------
// Deterministic replay with the whole state on chip (SINGLETON rows of <= 64
// nonzeros, 3p + n doubles within the shared-memory budget: BASELINE config 1
// and the reference tests' problems).  The same arithmetic, in the same order,
// as row_reg's deterministic path (so the iterates are bit-identical to the
// global-memory replay, which matches the reference's to ~1e-15): x, abar, D
// and alpha live in shared memory for the whole call, so a step needs no
// global stores and no fence -- only a __syncwarp -- and the next step's row
// is fetched while the current one computes.  One warp; the state is written
// back at the end.
struct DetRow {
    int64_t i;
    double y;
    int col[2];
    double val[2];
};
template <typename VT, typename PT>
__global__ void __launch_bounds__(32) sps_det_smem_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int64_t p = a.p, n = a.n, count = a.count;
    double *const sx = smem_dyn, *const sab = sx + p, *const sdd = sab + p, *const sal = sdd + p;
    for (int64_t j = lane; j < p; j += 32) {
        sx[j] = a.coord[4 * j];
        sab[j] = a.coord[4 * j + 1];
        sdd[j] = a.coord[4 * j + 2];
    }
    for (int64_t i = lane; i < n; i += 32) sal[i] = a.alpha[i];
    __syncwarp();
    constexpr int NCH = 2;
    // samples, row extents and labels of 32 steps at a time (lane L: step t0 + L):
    // one dependent round trip per 32 steps instead of three per step
    int64_t ci = 0, clo = 0, ni = 0, nlo = 0;
    int ck = 0, nk = 0;
    double cy = 0.0, ny = 0.0;
    auto batch = [&](int64_t t0, int64_t &bi, int64_t &blo, int &bk, double &by) {
        const int64_t t = t0 + lane;
        bi = blo = 0;
        bk = 0;
        by = 0.0;
        if (t < count) {
            bi = __ldg(a.samples + t);
            blo = rp<PT>(a.row_ptr, bi);
            bk = (int)(rp<PT>(a.row_ptr, bi + 1) - blo);
            by = rv<VT>(a.y, bi);
        }
    };
    batch(0, ci, clo, ck, cy);
    batch(32, ni, nlo, nk, ny);
    // the row of step tt (fetched in order, two steps before it is used)
    auto fetch = [&](int64_t tt, DetRow &r) {
        if ((tt & 31) == 0 && tt > 0) {
            ci = ni;
            clo = nlo;
            ck = nk;
            cy = ny;
            batch(tt + 32, ni, nlo, nk, ny);
        }
        const int src = (int)(tt & 31);
        r.i = __shfl_sync(FULL, ci, src);
        r.y = __shfl_sync(FULL, cy, src);
        const int64_t lo = __shfl_sync(FULL, clo, src);
        const int k = tt < count ? __shfl_sync(FULL, ck, src) : 0;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            const int e = c * 32 + lane;
            r.col[c] = e < k ? __ldg(a.col + lo + e) : -1;
            r.val[c] = e < k ? rv<VT>(a.val, lo + e) : 0.0;
        }
    };
    DetRow r0, r1, r2;
    fetch(0, r0);
    fetch(1, r1);
    for (int64_t t = 0; t < count; t++) {
        fetch(t + 2, r2);
        // ---- the step (row_reg's deterministic arithmetic, same order)
        const int64_t i = r0.i;
        double xr[NCH], abr[NCH], dr[NCH];
        double part = 0.0;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            if (r0.col[c] >= 0) {
                xr[c] = sx[r0.col[c]];
                abr[c] = sab[r0.col[c]];
                dr[c] = sdd[r0.col[c]];
                part += r0.val[c] * xr[c];
            }
        }
        double old = 0.0;
        if (lane == 0) old = sal[i];
        old = __shfl_sync(FULL, old, 0);
        const double margin = warp_sum(part);
        const double nw = loss_deriv(a.loss, margin, r0.y);
        const double ds = nw - old;
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            if (r0.col[c] >= 0) {
                double v = dr[c] * (abr[c] + a.lambda1 * xr[c]);
                v += ds * r0.val[c];
                const double g = step_of(a, dr[c]);
                const double u = xr[c] - g * v;
                const double z = prox_sep(a.pen, u, g * dr[c], a.lam2, a.lo, a.hi);
                if (a.trace_v) {
                    a.trace_v[r0.col[c]] = v;
                    a.trace_dx[r0.col[c]] = z - xr[c];
                }
                sx[r0.col[c]] = xr[c] + (z - xr[c]);
            }
        }
        if (lane == 0) sal[i] = nw;
        const double tq = (nw - old) / a.n_d;
#pragma unroll
        for (int c = 0; c < NCH; c++)
            if (r0.col[c] >= 0) sab[r0.col[c]] = abr[c] + tq * r0.val[c];
        __syncwarp();
        r0 = r1;
        r1 = r2;
    }
    for (int64_t j = lane; j < p; j += 32) {
        a.coord[4 * j] = sx[j];
        a.coord[4 * j + 1] = sab[j];
    }
    for (int64_t q = lane; q < n; q += 32) a.alpha[q] = sal[q];
}
template <typename VT, typename PT> static void *det_smem_ptr() { return (void *)sps_det_smem_kernel<VT, PT>; }
static void *pick_det_smem(const ps_csr_t *csr)
{
    const bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (f64 && i64) return det_smem_ptr<double, long long>();
    if (f64) return det_smem_ptr<double, int>();
    if (i64) return det_smem_ptr<float, long long>();
    return det_smem_ptr<float, int>();
}

// ---------------------------------------------------------------------------
// Fast async kernel: SINGLETON rows of <= 32 nonzeros (BASELINE configs 2-4).
// Same per-update arithmetic as row_reg, specialised on loss / penalty, with
// a software pipeline across updates:
//   * the NEXT sample's CSR row (row_ptr, columns, values, label) is fetched
//     while the current update computes -- these reads do not touch x, so
//     they shorten the dependent chain without adding staleness;
//   * the alpha exchange of update t is consumed (abar credit) only after the
//     state loads of update t+1 are issued, hiding its round trip.
// One warp per in-flight sample; hot columns staged in shared memory.
template <typename VT> struct RowRegs {
    int64_t i;
    int k, col;
    VT val, y;  // raw (widened at use, so the prefetch is not forced to complete early)
};

template <typename VT, typename PT>
__device__ __forceinline__ RowRegs<VT> fetch_row(const KArgs &a, int64_t i, int lane)
{
    RowRegs<VT> r;
    r.i = i;
    int64_t lo = rp<PT>(a.row_ptr, i);
    r.k = (int)(rp<PT>(a.row_ptr, i + 1) - lo);
    r.col = -1;
    r.val = VT(0);
    if (lane < r.k) {
        r.col = __ldg(a.col + lo + lane);
        r.val = __ldg(reinterpret_cast<const VT *>(a.val) + lo + lane);
    }
    r.y = __ldg(reinterpret_cast<const VT *>(a.y) + i);
    return r;
}

template <int PEN>
__device__ __forceinline__ double prox_t(double u, double eff, double lam2, int pen, double lo, double hi)
{
    if (PEN == PS_PEN_L1) {
        double thr = eff * lam2;
        double m = fmax(fabs(u) - thr, 0.0);
        return u > 0 ? m : (u < 0 ? -m : 0.0);
    }
    return prox_sep(pen, u, eff, lam2, lo, hi);
}

// exp(x) for x <= 0 (or NaN), ~1 ulp: x = n ln2 + r (Cody-Waite, |r| <= ln2/2),
// exp(r) by its degree-12 Taylor polynomial (truncation < 2e-16 relative),
// 2^n applied as two exact power-of-two factors so subnormal results round
// once.  About 20 instructions against ~49 for the libdevice exp(), whose
// range checks this domain does not need.  Used by the asynchronous kernels
// only (async parity is on the objective); the deterministic replay keeps
// the libdevice exp of loss_deriv.
__device__ __forceinline__ double exp_nonpos(double x)
{
    x = x < -746.0 ? -746.0 : x;  // exp(-746) rounds to 0; keeps n in int range (NaN passes)
    const double shifter = 0x1.8p52;
    double kd = __fma_rn(x, 0x1.71547652b82fep+0, shifter);  // n = rint(x / ln2) in the low bits
    const int n = __double2loint(kd);
    kd = __dsub_rn(kd, shifter);
    double r = __fma_rn(kd, -0x1.62e4200000000p-1, x);  // ln2_hi: kd * ln2_hi is exact
    r = __fma_rn(kd, -0x1.fdf473de6af28p-22, r);
    double q = 0x1.1eed8eff8d898p-29;  // 1/12!
    q = __fma_rn(q, r, 0x1.ae64567f544e4p-26);
    q = __fma_rn(q, r, 0x1.27e4fb7789f5cp-22);
    q = __fma_rn(q, r, 0x1.71de3a556c734p-19);
    q = __fma_rn(q, r, 0x1.a01a01a01a01ap-16);
    q = __fma_rn(q, r, 0x1.a01a01a01a01ap-13);
    q = __fma_rn(q, r, 0x1.6c16c16c16c17p-10);
    q = __fma_rn(q, r, 0x1.1111111111111p-7);
    q = __fma_rn(q, r, 0x1.5555555555555p-5);
    q = __fma_rn(q, r, 0x1.5555555555555p-3);
    q = __fma_rn(q, r, 0.5);
    q = __fma_rn(q, r, 1.0);
    q = __fma_rn(q, r, 1.0);
    const int n1 = n >> 1, n2 = n - n1;  // n in [-1076, 0]: both halves >= -538
    q = __dmul_rn(q, __hiloint2double((n1 + 1023) << 20, 0));
    return __dmul_rn(q, __hiloint2double((n2 + 1023) << 20, 0));
}

// num / den for den in [1, 2] (den = 1 + exp(-|t|)): hardware reciprocal
// estimate, two Newton steps and one residual correction (faithful, no
// special cases in this domain).
__device__ __forceinline__ double div_1to2(double num, double den)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
    double e = __fma_rn(-den, y, 1.0);
    y = __fma_rn(y, e, y);
    e = __fma_rn(-den, y, 1.0);
    y = __fma_rn(y, e, y);
    const double q = __dmul_rn(num, y);
    return __fma_rn(__fma_rn(-den, q, num), y, q);
}

// losses.py:73-86 with one division: et = exp(-|t|); sig = (t > 0 ? 1 : et) / (1 + et)
// -- the same two expressions as the reference's branches, no divergence.
template <int LOSS> __device__ __forceinline__ double deriv_t(double z, double b)
{
    if (LOSS == PS_LOSS_LOGISTIC) {
        double t = -b * z;
        double et = exp_nonpos(-fabs(t));
        double sig = div_1to2(t > 0 ? 1.0 : et, 1.0 + et);
        return -b * sig;
    }
    return z - b;
}

// per-lane state of one update: NC nonzeros per lane (rows of <= 32 * NC)
template <typename VT, int NC> struct Row {
    int64_t i;
    int col[NC];
    VT val[NC];
    VT y;
};

template <typename VT, typename PT, int NC>
__device__ __forceinline__ void fetch_rowc(const KArgs &a, int64_t i, int lane, Row<VT, NC> &r, bool valid)
{
    r.i = i;
    int64_t lo = 0;
    int k = 0;
    if (valid) {
        lo = rp<PT>(a.row_ptr, i);
        k = (int)(rp<PT>(a.row_ptr, i + 1) - lo);
    }
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const int e = lane + 32 * c;
        r.col[c] = -1;
        r.val[c] = VT(0);
        if (e < k) {
            r.col[c] = __ldg(a.col + lo + e);
            r.val[c] = __ldg(reinterpret_cast<const VT *>(a.val) + lo + e);
        }
    }
    r.y = valid ? __ldg(reinterpret_cast<const VT *>(a.y) + i) : VT(0);
}

// the row's nonzeros given its extent (row_ptr already read a stage earlier)
template <typename VT, int NC>
__device__ __forceinline__ void fetch_cols(const int32_t *__restrict__ colp, const VT *__restrict__ valp,
                                           const VT *__restrict__ yp, int64_t i, int64_t lo, int k, int lane,
                                           Row<VT, NC> &r)
{
    r.i = i;
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const int e = lane + 32 * c;
        r.col[c] = -1;
        r.val[c] = VT(0);
        if (e < k) {
            r.col[c] = __ldg(colp + lo + e);
            r.val[c] = __ldg(valp + lo + e);
        }
    }
    r.y = k >= 0 ? __ldg(yp + i) : VT(0);
}

template <typename VT, typename PT, int LOSS, int PEN, int NC, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) sps_fast_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    __shared__ unsigned long long cta_prog;  // this CTA's updates reported so far (progress counter)
    if (threadIdx.x == 0) cta_prog = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    HotView h = hot_view(smem_dyn, a.H);
    unsigned *dirty = reinterpret_cast<unsigned *>(smem_dyn + a.hot_doubles);
    double *px = h.pend + (2 * (wib % NCOPY)) * a.H, *pab = px + a.H;
    if (a.H > 0) {
        for (int s = threadIdx.x; s < a.H; s += blockDim.x) {
            const double *g = a.coord + 4 * hot_coord(a, s);
            reinterpret_cast<double2 *>(h.xab)[s] = ld_cg2(g);
            h.d[s] = __ldg(g + 2);
        }
        for (int s = threadIdx.x; s < 2 * NCOPY * a.H; s += blockDim.x) h.pend[s] = 0.0;
        if (threadIdx.x < 2 * HDR_DOUBLES) dirty[threadIdx.x] = 0u;
        __syncthreads();
    }
    // thread-block cluster: members refresh their hot snapshot from the
    // leader's (rank 0), whose snapshot must be initialised first
    unsigned lead = 0u;
    if (a.cluster > 1) {
        unsigned rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        if (rank != 0 && a.H > 0) {
            const unsigned mine = (unsigned)__cvta_generic_to_shared(smem_dyn);
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(mine));
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    // kernel parameters used in the loop, hoisted
    double *const coord = a.coord;
    double *const alpha = a.alpha;
    const double gamma = a.gamma, lambda1 = a.lambda1, kappa = a.kappa, kappa_hot = a.kappa_hot, lam2 = a.lam2;
    const double plo = a.lo, phi = a.hi;
    const int pen = a.pen;
    const int shift = a.hot_shift;
    const int hmask = (1 << shift) - 1, hlim = a.H << shift;
    const uint64_t seed = a.seed, base = a.slot_base, nrows = (uint64_t)a.n;
    const double inv_n = 1.0 / a.n_d;
    const bool store_zero = !(a.diag & PS_FLAG_DELTA_ZERO);
    const bool zero_now = (a.diag & PS_FLAG_ZERO_IMMEDIATE) != 0;
    const int64_t nwarps = (int64_t)gridDim.x * nwib;
    const int64_t q = a.count / nwarps, rr = a.count % nwarps;
    uint64_t slot = (uint64_t)(gw * q + min(gw, rr));
    const uint64_t slot_end = slot + (uint64_t)(q + (gw < rr ? 1 : 0));
    int until_flush = a.H > 0 ? 1 + (wib * a.period) / max(1, nwib) : 0;

    // pending abar credit of the previous update
    int pcol[NC], pslot[NC];
    double pval[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) pcol[c] = -1;
    double pnw = 0.0, prep = 0.0;

    const int32_t *const colp = a.col;
    const VT *const valp = reinterpret_cast<const VT *>(a.val);
    const VT *const yp = reinterpret_cast<const VT *>(a.y);
    const void *const rowp = a.row_ptr;
    if (slot < slot_end) {
        // pipeline: samples and row extents are drawn 32 at a time (lane L holds
        // slot first + L) one batch ahead and handed out by shuffles; a row's
        // nonzeros are fetched one update ahead; the state reads and the update
        // itself run now
        const uint64_t first = slot;
        int64_t bi, blo, ni, nlo;
        int bk, nk;
        auto load_batch = [&](uint64_t s0, int64_t &bi_, int64_t &blo_, int &bk_) {
            const uint64_t sl = s0 + (uint64_t)lane;
            bi_ = 0;
            blo_ = 0;
            bk_ = -1;
            if (sl < slot_end) {
                bi_ = sample_row(seed, base + sl, nrows);
                blo_ = rp<PT>(rowp, bi_);
                bk_ = (int)(rp<PT>(rowp, bi_ + 1) - blo_);
            }
        };
        load_batch(first, bi, blo, bk);
        load_batch(first + 32, ni, nlo, nk);
        Row<VT, NC> cur;
        fetch_cols<VT, NC>(colp, valp, yp, __shfl_sync(FULL, bi, 0), __shfl_sync(FULL, blo, 0),
                           __shfl_sync(FULL, bk, 0), lane, cur);
        while (true) {
            // ---- state reads (hot: CTA snapshot in shared memory; cold: one
            // 16-B L2 read + D through the read-only path)
            int sl[NC];
            double xh[NC], ab[NC], d[NC];
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int col = cur.col[c];
                sl[c] = (col >= 0 && col < hlim && (col & hmask) == 0) ? (col >> shift) : -1;
                xh[c] = ab[c] = d[c] = 0.0;
                if (col >= 0) {
                    if (sl[c] >= 0) {
                        double2 v = reinterpret_cast<const double2 *>(h.xab)[sl[c]];
                        xh[c] = v.x;
                        ab[c] = v.y;
                        d[c] = h.d[sl[c]];
                    } else {
                        double2 v = ld_cg2(coord + 4 * (int64_t)col);
                        xh[c] = v.x;
                        ab[c] = v.y;
                        d[c] = __ldg(coord + 4 * (int64_t)col + 2);
                    }
                }
            }
            double old = 0.0;
            if (lane == 0) old = ld_cg(alpha + cur.i);
            // ---- abar credit of the previous update (its exchange has returned by now)
            {
                const double t = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    if (pcol[c] >= 0) {
                        if (pslot[c] >= 0) {
                            atomicAdd(pab + pslot[c], t * pval[c]);
                            mark_dirty(dirty, pslot[c]);
                        } else {
                            red_add(coord + 4 * (int64_t)pcol[c] + 1, t * pval[c]);
                        }
                    }
                }
            }
            // ---- prefetch: the next row's nonzeros (its extent from the batch)
            const bool more = slot + 1 < slot_end;
            slot++;
            const uint32_t t1 = (uint32_t)(slot - first);
            if ((t1 & 31u) == 0) {
                bi = ni;
                blo = nlo;
                bk = nk;
                load_batch(first + t1 + 32, ni, nlo, nk);
            }
            const int src = (int)(t1 & 31u);
            Row<VT, NC> nxt;
            fetch_cols<VT, NC>(colp, valp, yp, __shfl_sync(FULL, bi, src), __shfl_sync(FULL, blo, src),
                               more ? __shfl_sync(FULL, bk, src) : -1, lane, nxt);
            // ---- margin -> derivative -> prox -> commit x
            double part = 0.0;
#pragma unroll
            for (int c = 0; c < NC; c++) part += widen(cur.val[c]) * xh[c];
            const double margin = warp_sum(part);
            old = __shfl_sync(FULL, old, 0);
            const double nw = deriv_t<LOSS>(margin, widen(cur.y));
            const double ds = nw - old;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int col = cur.col[c];
                if (col >= 0) {
                    const double cval = widen(cur.val[c]);
                    double v = d[c] * (ab[c] + lambda1 * xh[c]);
                    v += ds * cval;
                    const double g = gamma * fmin(1.0, (sl[c] >= 0 ? kappa_hot : kappa) * d[c]);
                    const double u = xh[c] - g * v;
                    const double z = prox_t<PEN>(u, g * d[c], lam2, pen, plo, phi);
                    if (z == 0.0 && store_zero) {
                        // the prox zeroed the coordinate: commit it as a store, not as the
                        // delta -x_hat; drops this CTA's pending
                        // delta.  A staged column read as 0 already: the store only undoes
                        // other CTAs' drift, so it is deferred to the CTA's next flush
                        // (mark_zero: one store per flush instead of one per update)
                        if (sl[c] >= 0) {
                            drop_pending_x(h, sl[c]);
                            if (zero_now || xh[c] != 0.0) atomic_exch(coord + 4 * (int64_t)col, 0.0);
                            else mark_zero(dirty, sl[c]);
                        } else {
                            atomic_exch(coord + 4 * (int64_t)col, 0.0);
                        }
                    } else if (sl[c] >= 0) {
                        atomicAdd(px + sl[c], z - xh[c]);
                        mark_dirty(dirty, sl[c]);
                    } else {
                        red_add(coord + 4 * (int64_t)col, z - xh[c]);
                    }
                }
                pcol[c] = col;
                pslot[c] = sl[c];
                pval[c] = widen(cur.val[c]);
            }
            // ---- alpha_i <-> new (consumed next iteration)
            double rep = 0.0;
            if (lane == 0) rep = atomic_exch(alpha + cur.i, nw);
            pnw = nw;
            prep = rep;
            if (a.H > 0 && --until_flush == 0) {
                hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit, lead}, a.H, dirty, lane, true);
                until_flush = a.period;
            }
            // progress counter, bumped every PROGRESS_BATCH updates (the workers'
            // counter_batch, asynchronous.py:155-162): a host monitor reads it
            // (per CTA in shared memory first: one global atomic per CTA_PROGRESS
            // updates of the CTA instead of per PROGRESS_BATCH of a warp -- the
            // same reporting granularity, 148 x 512 vs 4736 x 16 updates, and no
            // same-address atomic stream from every warp into one L2 line)
            if (lane == 0 && (slot - first) % PROGRESS_BATCH == 0) {
                const unsigned long long o = atomicAdd(&cta_prog, (unsigned long long)PROGRESS_BATCH);
                if ((o + PROGRESS_BATCH) / CTA_PROGRESS != o / CTA_PROGRESS)
                    atomicAdd(a.counter, (unsigned long long)CTA_PROGRESS);
            }
            if (!more) break;
            cur = nxt;
        }
        // last credit
        const double t = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
#pragma unroll
        for (int c = 0; c < NC; c++) {
            if (pcol[c] >= 0) {
                if (pslot[c] >= 0) {
                    atomicAdd(pab + pslot[c], t * pval[c]);
                    mark_dirty(dirty, pslot[c]);
                } else {
                    red_add(coord + 4 * (int64_t)pcol[c] + 1, t * pval[c]);
                }
            }
        }
    }
    if (lane == 0) {
        const int64_t mine = q + (gw < rr ? 1 : 0);
        if (mine % PROGRESS_BATCH) atomicAdd(a.counter, (unsigned long long)(mine % PROGRESS_BATCH));
    }
    __syncthreads();  // every warp's CTA progress is in
    if (threadIdx.x == 0 && cta_prog % CTA_PROGRESS) atomicAdd(a.counter, cta_prog % CTA_PROGRESS);
    if (a.cluster > 1)  // the leader's staging area stays alive until every member stops reading it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (a.H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            dirty[lane] = HOT_PER_LANE >= 32 ? 0xffffffffu : (0xffffffffu >> (32 - HOT_PER_LANE));
            __syncwarp();
            hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit}, a.H, dirty, lane, false);
        }
        hot_async_drain();
    }
}

}  // namespace ps
#include "fast2.cuh"
namespace ps {

// ---------------------------------------------------------------------------
// Fast async kernel for group lasso on contiguous blocks of G <= 16
// coordinates (BASELINE config 5), rows of <= 32 nonzeros.
//   * the row's distinct blocks (T_i) come from __match_any_sync on col / G,
//     so rows need not be sorted; block rank = popc of the leader mask;
//   * the extended support (g blocks x G coordinates) is processed in passes
//     of 32/G blocks, G lanes per block; x^, abar^, D and the row values per
//     ext slot are staged in per-warp shared memory between the margin pass
//     and the prox pass (one read of x^ per coordinate, as worker_iteration);
//   * block norms by segmented shuffle over the G lanes (penalties.py:103-108);
//   * hot blocks (all G coordinates) staged per CTA exactly like hot columns.
template <typename VT, typename PT, int LOSS, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) sps_group_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    const int G = a.G;
    const int bpc = 32 / G;
    const bool store_zero = !(a.diag & PS_FLAG_DELTA_ZERO);
    HotView h = hot_view(smem_dyn, a.H);
    unsigned *dirty = reinterpret_cast<unsigned *>(smem_dyn + a.hot_doubles);
    double *px = h.pend + (2 * (wib % NCOPY)) * a.H, *pab = px + a.H;
    const int HB = a.H / max(G, 1);
    int *bcnt = reinterpret_cast<int *>(smem_dyn + a.hot_doubles + HDR_DOUBLES);
    const int hdr = a.H > 0 ? a.hot_doubles + HDR_DOUBLES + (HB + 1) / 2 : 0;
    // per-warp staging: row value / x^ / abar^ / D per ext slot (32 * G each)
    double *wa = smem_dyn + hdr + (int64_t)wib * (4 * 32 * G);
    double *wx = wa + 32 * G, *wab = wx + 32 * G, *wd = wab + 32 * G;
    if (a.H > 0) {
        for (int s = threadIdx.x; s < a.H; s += blockDim.x) {
            const double *g = a.coord + 4 * hot_coord(a, s);
            reinterpret_cast<double2 *>(h.xab)[s] = ld_cg2(g);
            h.d[s] = __ldg(g + 2);
        }
        for (int s = threadIdx.x; s < 2 * NCOPY * a.H; s += blockDim.x) h.pend[s] = 0.0;
        if (threadIdx.x < 2 * HDR_DOUBLES) dirty[threadIdx.x] = 0u;
        for (int r = threadIdx.x; r < HB; r += blockDim.x) bcnt[r] = 0;
        __syncthreads();
    }
    const int64_t nwarps = (int64_t)gridDim.x * nwib;
    const int64_t q0 = a.count / nwarps, rr = a.count % nwarps;
    uint64_t slot = (uint64_t)(gw * q0 + min(gw, rr));
    int64_t prog = 0;  // this warp's updates (progress counter)
    const uint64_t slot_end = slot + (uint64_t)(q0 + (gw < rr ? 1 : 0));
    const int S = 1 << a.hot_shift;
    const int hbl = (a.H / max(G, 1)) * S;  // hot block indices are multiples of S below this
    const double inv_n = 1.0 / a.n_d;
    int until_flush = a.H > 0 ? 1 + (wib * a.period) / max(1, nwib) : 0;
    const int qd = lane % G, tb = lane / G;

    if (slot < slot_end) {
        RowRegs<VT> cur = fetch_row<VT, PT>(a, sample_row(a.seed, a.slot_base + slot, (uint64_t)a.n), lane);
        while (true) {
            const int col = cur.col;
            const bool act = col >= 0;
            const int blk = act ? col / G : -1 - lane;
            const unsigned peers = __match_any_sync(FULL, blk);
            const int lead = __ffs(peers) - 1;
            const unsigned leaders = __ballot_sync(FULL, act && lead == lane);
            const int g = __popc(leaders);
            const int myrank = __popc(leaders & ((1u << lead) - 1u));
            double old = 0.0;
            if (lane == 0) old = ld_cg(a.alpha + cur.i);
            // row values into their ext slots
            for (int s2 = lane; s2 < g * G; s2 += 32) wa[s2] = 0.0;
            __syncwarp();
            const double cval = widen(cur.val);
            if (act) wa[myrank * G + (col - blk * G)] = cval;
            __syncwarp();
            // ---- pass 1: gather x^, abar^, D on T_i; partial margin
            double part = 0.0;
            for (int t0 = 0; t0 < g; t0 += bpc) {
                const int t = t0 + tb;
                const bool on0 = tb < bpc && t < g;
                const int src = on0 ? (int)__fns(leaders, 0, t + 1) : 0;
                const int B = __shfl_sync(FULL, blk, src);
                if (on0) {
                    wx[t * G + qd] = wab[t * G + qd] = wd[t * G + qd] = 0.0;
                }
                const bool on = on0 && (int64_t)B * G + qd < a.p;  // ragged last block
                if (on) {
                    const int s2 = t * G + qd;
                    const int64_t c = (int64_t)B * G + qd;
                    double xh, ab, d;
                    if (B < hbl && (B & (S - 1)) == 0) {
                        const int hs = (B / S) * G + qd;
                        double2 v = reinterpret_cast<const double2 *>(h.xab)[hs];
                        xh = v.x;
                        ab = v.y;
                        d = h.d[hs];
                    } else {
                        double2 v = ld_cg2(a.coord + 4 * c);
                        xh = v.x;
                        ab = v.y;
                        d = __ldg(a.coord + 4 * c + 2);
                    }
                    wx[s2] = xh;
                    wab[s2] = ab;
                    wd[s2] = d;
                    part += wa[s2] * xh;
                }
            }
            // ---- prefetch the next sample's row
            const bool more = slot + 1 < slot_end;
            slot++;
            int64_t ni = more ? sample_row(a.seed, a.slot_base + slot, (uint64_t)a.n) : cur.i;
            int64_t nlo = rp<PT>(a.row_ptr, ni);
            int nk = more ? (int)(rp<PT>(a.row_ptr, ni + 1) - nlo) : 0;
            const double margin = warp_sum(part);
            old = __shfl_sync(FULL, old, 0);
            const double nw = loss_deriv(LOSS, margin, widen(cur.y));
            const double ds = nw - old;
            RowRegs<VT> nxt;
            nxt.i = ni;
            nxt.k = nk;
            nxt.col = -1;
            nxt.val = VT(0);
            if (lane < nk) {
                nxt.col = __ldg(a.col + nlo + lane);
                nxt.val = __ldg(reinterpret_cast<const VT *>(a.val) + nlo + lane);
            }
            nxt.y = more ? __ldg(reinterpret_cast<const VT *>(a.y) + ni) : VT(0);
            __syncwarp();
            // ---- pass 2: u, block norms, group shrinkage, commit x on T_i
            for (int t0 = 0; t0 < g; t0 += bpc) {
                const int t = t0 + tb;
                const bool on0 = tb < bpc && t < g;
                const int src = on0 ? (int)__fns(leaders, 0, t + 1) : 0;
                const int B = __shfl_sync(FULL, blk, src);
                const bool on = on0 && (int64_t)B * G + qd < a.p;
                const int s2 = t * G + qd;
                double xh = 0.0, u = 0.0, d = 0.0;
                const bool hot = B < hbl && (B & (S - 1)) == 0;
                if (on) {
                    xh = wx[s2];
                    d = wd[s2];
                    const double gB = a.gamma * fmin(1.0, (hot ? a.kappa_hot : a.kappa) * d);
                    double v = d * (wab[s2] + a.lambda1 * xh);
                    v += ds * wa[s2];
                    u = xh - gB * v;
                }
                double sq = u * u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    double r = __shfl_down_sync(FULL, sq, o);
                    if (qd + o < G && lane + o < 32) sq += r;
                }
                const double ss = __shfl_sync(FULL, sq, lane - qd);
                if (on) {
                    if (hot) {  // accumulate the gradient step; block prox at flush
                        const int hs = (B / S) * G + qd;
                        atomicAdd(px + hs, u - xh);
                        if (qd == 0) atomicAdd(bcnt + B / S, 1);
                    } else {
                        const double gB = a.gamma * fmin(1.0, a.kappa * d);
                        const double f = group_factor(sqrt(ss), gB * d, a.lam2);
                        if (f == 0.0 && store_zero) atomic_exch(a.coord + 4 * ((int64_t)B * G + qd), 0.0);
                        else red_add(a.coord + 4 * ((int64_t)B * G + qd), u * f - xh);
                    }
                }
            }
            // ---- alpha swap, abar credit on S_i
            double rep = 0.0;
            if (lane == 0) rep = atomic_exch(a.alpha + cur.i, nw);
            rep = __shfl_sync(FULL, rep, 0);
            const double tt = (nw - rep) * inv_n;
            if (act) {
                const bool hot = blk < hbl && (blk & (S - 1)) == 0;
                if (hot) {
                    const int hs = (blk / S) * G + (col - blk * G);
                    atomicAdd(pab + hs, tt * cval);
                } else {
                    red_add(a.coord + 4 * (int64_t)col + 1, tt * cval);
                }
            }
            if (a.H > 0 && --until_flush == 0) {
                hot_flush_group(a, h, bcnt, lane, true);
                until_flush = a.period;
            }
            if (lane == 0 && ++prog % PROGRESS_BATCH == 0) atomicAdd(a.counter, (unsigned long long)PROGRESS_BATCH);
            __syncwarp();
            if (!more) break;
            cur = nxt;
        }
    }
    if (lane == 0 && prog % PROGRESS_BATCH) atomicAdd(a.counter, (unsigned long long)(prog % PROGRESS_BATCH));
    if (a.H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) hot_flush_group(a, h, bcnt, lane, false);
        hot_async_drain();
    }
}

}  // namespace ps

using namespace ps;

static int scratch_layout(const ps_csr_t *csr, const ps_part_t *part, int *M, int *GB)
{
    // max_slots from ps_prepare; GB bounded by the longest row
    *M = std::max(1, (int)part->max_slots);
    *GB = 1;
    if (part->kind != PS_PART_SINGLETON) *GB = std::max(1, (int)std::min<int64_t>(part->max_slots, csr->n_cols));
    int ints = *M + 2 * (*GB) + 2;
    return 4 * (*M) + (ints + 1) / 2;  // doubles per warp
}

static bool needs_scratch(const ps_csr_t *csr, const ps_part_t *part, bool big = false)
{
    if (part->kind != PS_PART_SINGLETON) return true;
    return !big && part->max_slots > NCH_MAX * 32;
}

extern "C" int64_t ps_scratch_bytes(const ps_csr_t *csr, const ps_part_t *part, int32_t warps)
{
    if (!csr || !part || !needs_scratch(csr, part)) return 0;
    int M, GB;
    int stride = scratch_layout(csr, part, &M, &GB);
    return (int64_t)stride * 8 * std::max(warps, 1);
}

template <typename VT, typename PT, int PART> static void *kernel_ptr()
{
    return (void *)sps_kernel<VT, PT, PART, 256>;
}
template <typename VT, typename PT> static void *kernel_ptr_big()
{
    return (void *)sps_kernel<VT, PT, PS_PART_SINGLETON, 1024>;
}
// fast kernel CTA sizes: 32 warps (default) or 24 warps (warps_per_cta = 24)
constexpr int FAST_T = 1024, FAST_T_SMALL = 768;
template <typename VT, typename PT, int NC, int T> static void *kernel_ptr_fast_t(int loss, int pen)
{
    if (loss == PS_LOSS_LOGISTIC) {
        if (pen == PS_PEN_L1) return (void *)sps_fast_kernel<VT, PT, PS_LOSS_LOGISTIC, PS_PEN_L1, NC, T>;
        return (void *)sps_fast_kernel<VT, PT, PS_LOSS_LOGISTIC, PS_PEN_ZERO, NC, T>;
    }
    if (pen == PS_PEN_L1) return (void *)sps_fast_kernel<VT, PT, PS_LOSS_SQUARED, PS_PEN_L1, NC, T>;
    return (void *)sps_fast_kernel<VT, PT, PS_LOSS_SQUARED, PS_PEN_ZERO, NC, T>;
}
template <typename VT, typename PT, int NC> static void *kernel_ptr_fast(int loss, int pen, bool small)
{
    return small ? kernel_ptr_fast_t<VT, PT, NC, FAST_T_SMALL>(loss, pen) : kernel_ptr_fast_t<VT, PT, NC, FAST_T>(loss, pen);
}
template <typename VT, typename PT, bool LIT, int NC> static void *kernel_ptr_hot_l(int loss, int pen)
{
    if (loss == PS_LOSS_LOGISTIC) {
        if (pen == PS_PEN_L1) return (void *)sps_hot_kernel<VT, PT, PS_LOSS_LOGISTIC, PS_PEN_L1, LIT, NC>;
        return (void *)sps_hot_kernel<VT, PT, PS_LOSS_LOGISTIC, PS_PEN_ZERO, LIT, NC>;
    }
    if (pen == PS_PEN_L1) return (void *)sps_hot_kernel<VT, PT, PS_LOSS_SQUARED, PS_PEN_L1, LIT, NC>;
    return (void *)sps_hot_kernel<VT, PT, PS_LOSS_SQUARED, PS_PEN_ZERO, LIT, NC>;
}
template <typename VT, typename PT> static void *kernel_ptr_hot(int loss, int pen, bool literal, int nc)
{
    if (nc == 2)
        return literal ? kernel_ptr_hot_l<VT, PT, true, 2>(loss, pen) : kernel_ptr_hot_l<VT, PT, false, 2>(loss, pen);
    return literal ? kernel_ptr_hot_l<VT, PT, true, 1>(loss, pen) : kernel_ptr_hot_l<VT, PT, false, 1>(loss, pen);
}
static void *pick_hot(const ps_csr_t *csr, int loss, int pen, bool literal, int nc)
{
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (f64 && i64) return kernel_ptr_hot<double, long long>(loss, pen, literal, nc);
    if (f64) return kernel_ptr_hot<double, int>(loss, pen, literal, nc);
    if (i64) return kernel_ptr_hot<float, long long>(loss, pen, literal, nc);
    return kernel_ptr_hot<float, int>(loss, pen, literal, nc);
}
// ---------------------------------------------------------------------------
// Group lasso, lane per block (contiguous blocks of G in {2,4,5,8,10,16},
// rows of <= 32 nonzeros; BASELINE config 5).  The leader lane of each of the
// row's distinct blocks (__match_any_sync on col / G) owns the whole block:
// it issues the G coordinate loads back to back, computes u on the block,
// its squared norm in registers, the group shrinkage (penalties.py:103-108)
// and commits the G coordinates; no shuffles inside a block.  The row
// values reach their block owner through per-warp shared memory.  Pipelined
// like sps_fast_kernel (next row prefetched, abar credit deferred one update).
template <typename VT, typename PT, int LOSS, int G, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) sps_group_lane_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    // shared memory: [hot staging area | dirty words] then per-warp row values
    HotView h = hot_view(smem_dyn, a.H);
    unsigned *dirty = reinterpret_cast<unsigned *>(smem_dyn + a.hot_doubles);
    double *px = h.pend + (2 * (wib % NCOPY)) * a.H, *pab = px + a.H;
    const int hdr = a.H > 0 ? a.hot_doubles + HDR_DOUBLES : 0;
    double *wa = smem_dyn + hdr + (int64_t)wib * (32 * G);  // row value per (leader lane, q)
    if (a.H > 0) {
        for (int s = threadIdx.x; s < a.H; s += blockDim.x) {
            const double *g = a.coord + 4 * hot_coord(a, s);
            reinterpret_cast<double2 *>(h.xab)[s] = ld_cg2(g);
            h.d[s] = __ldg(g + 2);
        }
        for (int s = threadIdx.x; s < 2 * NCOPY * a.H; s += blockDim.x) h.pend[s] = 0.0;
        if (threadIdx.x < 2 * HDR_DOUBLES) dirty[threadIdx.x] = 0u;
        __syncthreads();
    }
    double *const coord = a.coord;
    double *const alpha = a.alpha;
    const double gamma = a.gamma, lambda1 = a.lambda1, kappa = a.kappa, kappa_hot = a.kappa_hot, lam2 = a.lam2;
    const bool skip_zero = (a.diag & PS_FLAG_GROUP_STORE_ZEROS) == 0;
    const bool store_zero = !(a.diag & PS_FLAG_DELTA_ZERO);
    const uint64_t seed = a.seed, base = a.slot_base, nrows = (uint64_t)a.n;
    const double inv_n = 1.0 / a.n_d;
    const int64_t p = a.p;
    const int shift = a.hot_shift;
    const int hbl = (a.H / G) << shift;  // hot blocks: multiples of 2^shift below this
    const int64_t nwarps = (int64_t)gridDim.x * nwib;
    const int64_t q0 = a.count / nwarps, rr = a.count % nwarps;
    uint64_t slot = (uint64_t)(gw * q0 + min(gw, rr));
    int64_t prog = 0;  // this warp's updates (progress counter)
    const uint64_t slot_end = slot + (uint64_t)(q0 + (gw < rr ? 1 : 0));
    int until_flush = a.H > 0 ? 1 + (wib * a.period) / max(1, nwib) : 0;

    int pcol = -1, pslot = -1;
    double pval = 0.0, pnw = 0.0, prep = 0.0;
    if (slot < slot_end) {
        Row<VT, 1> cur;
        fetch_rowc<VT, PT, 1>(a, sample_row(seed, base + slot, nrows), lane, cur, true);
        while (true) {
            const int col = cur.col[0];
            const bool act = col >= 0;
            const int blk = act ? col / G : -1 - lane;
            const unsigned peers = __match_any_sync(FULL, blk);
            const bool leader = act && (__ffs(peers) - 1) == lane;
            const int lead = __ffs(peers) - 1;
            // staged block: its G slots start at sb
            const int sb = (act && blk < hbl && (blk & ((1 << shift) - 1)) == 0) ? (blk >> shift) * G : -1;
            // ---- leaders: the block's G records (x^, abar^) and its weight D
            double xh[G], ab[G], d = 0.0;
            const int64_t c0 = (int64_t)blk * G;
            const int nq = leader ? (int)min((int64_t)G, p - c0) : 0;  // ragged last block
            if (leader) {
                if (sb >= 0) {
#pragma unroll
                    for (int q = 0; q < G; q++) {
                        double2 v = reinterpret_cast<const double2 *>(h.xab)[sb + q];
                        xh[q] = v.x;
                        ab[q] = v.y;
                    }
                    d = h.d[sb];
                } else {
#pragma unroll
                    for (int q = 0; q < G; q++) {
                        double2 v = q < nq ? ld_cg2(coord + 4 * (c0 + q)) : make_double2(0.0, 0.0);
                        xh[q] = v.x;
                        ab[q] = v.y;
                    }
                    d = __ldg(coord + 4 * c0 + 2);
                }
            }
            double old = 0.0;
            if (lane == 0) old = ld_cg(alpha + cur.i);
            // ---- abar credit of the previous update
            {
                const double t = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
                if (pcol >= 0) {
                    if (pslot >= 0) {
                        atomicAdd(pab + pslot, t * pval);
                        mark_dirty(dirty, pslot);
                    } else {
                        red_add(coord + 4 * (int64_t)pcol + 1, t * pval);
                    }
                }
            }
            // ---- prefetch the next row
            const bool more = slot + 1 < slot_end;
            slot++;
            Row<VT, 1> nxt;
            fetch_rowc<VT, PT, 1>(a, more ? sample_row(seed, base + slot, nrows) : cur.i, lane, nxt, more);
            // ---- row values to their block owner
            if (leader) {
#pragma unroll
                for (int q = 0; q < G; q++) wa[lane * G + q] = 0.0;
            }
            __syncwarp();
            const double cval = widen(cur.val[0]);
            if (act) wa[lead * G + (col - blk * G)] = cval;
            __syncwarp();
            double part = 0.0;
            if (leader) {
#pragma unroll
                for (int q = 0; q < G; q++) part += wa[lane * G + q] * xh[q];
            }
            const double margin = warp_sum(part);
            old = __shfl_sync(FULL, old, 0);
            const double nw = deriv_t<LOSS>(margin, widen(cur.y));
            const double ds = nw - old;
            if (leader) {
                const double gB = gamma * fmin(1.0, (sb >= 0 ? kappa_hot : kappa) * d);
                double ss = 0.0;
#pragma unroll
                for (int q = 0; q < G; q++) {
                    double v = d * (ab[q] + lambda1 * xh[q]);
                    v += ds * wa[lane * G + q];
                    const double u = xh[q] - gB * v;
                    ab[q] = u;  // reuse
                    ss += u * u;
                }
                const double f = group_factor(sqrt(ss), gB * d, lam2);
                bool was_zero = true;
#pragma unroll
                for (int q = 0; q < G; q++) was_zero = was_zero && xh[q] == 0.0;
                if (f == 0.0 && store_zero && was_zero && skip_zero && sb < 0) {
                    // a block read as zero that the prox keeps at zero: its delta is 0,
                    // so nothing is committed (the store would be a same-address atomic
                    // per coordinate on the hottest blocks; near lambda_max most of T_i)
                } else if (f == 0.0 && store_zero) {
                    // the prox zeroed the block: store it
#pragma unroll
                    for (int q = 0; q < G; q++) {
                        if (q < nq) {
                            if (sb >= 0) {
                                drop_pending_x(h, sb + q);
                                h.xab[2 * (sb + q)] = 0.0;  // this CTA sees its own store
                            }
                            atomic_exch(coord + 4 * (c0 + q), 0.0);
                        }
                    }
                } else if (sb >= 0) {
#pragma unroll
                    for (int q = 0; q < G; q++) {
                        atomicAdd(px + sb + q, ab[q] * f - xh[q]);
                        mark_dirty(dirty, sb + q);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < G; q++)
                        if (q < nq) red_add(coord + 4 * (c0 + q), ab[q] * f - xh[q]);
                }
            }
            double rep = 0.0;
            if (lane == 0) rep = atomic_exch(alpha + cur.i, nw);
            pnw = nw;
            prep = rep;
            pcol = col;
            pslot = sb >= 0 ? sb + (col - blk * G) : -1;
            pval = cval;
            if (a.H > 0 && --until_flush == 0) {
                hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit}, a.H, dirty, lane, true);
                until_flush = a.period;
            }
            if (lane == 0 && ++prog % PROGRESS_BATCH == 0) atomicAdd(a.counter, (unsigned long long)PROGRESS_BATCH);
            __syncwarp();
            if (!more) break;
            cur = nxt;
        }
        const double t = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
        if (pcol >= 0) {
            if (pslot >= 0) {
                atomicAdd(pab + pslot, t * pval);
                mark_dirty(dirty, pslot);
            } else {
                red_add(coord + 4 * (int64_t)pcol + 1, t * pval);
            }
        }
    }
    if (lane == 0 && prog % PROGRESS_BATCH) atomicAdd(a.counter, (unsigned long long)(prog % PROGRESS_BATCH));
    if (a.H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            dirty[lane] = HOT_PER_LANE >= 32 ? 0xffffffffu : (0xffffffffu >> (32 - HOT_PER_LANE));
            __syncwarp();
            hot_flush(FlushArgs{a.coord, a.hot_shift, a.hot_unit}, a.H, dirty, lane, false);
        }
        hot_async_drain();
    }
}

// 768 threads (85 registers) while the block's 2G doubles fit, else 512
static constexpr int glane_threads(int G) { return G <= 5 ? 768 : 512; }
template <typename VT, typename PT, int G> static void *kernel_ptr_glane(int loss)
{
    if (loss == PS_LOSS_LOGISTIC)
        return (void *)sps_group_lane_kernel<VT, PT, PS_LOSS_LOGISTIC, G, glane_threads(G)>;
    return (void *)sps_group_lane_kernel<VT, PT, PS_LOSS_SQUARED, G, glane_threads(G)>;
}
template <int G> static void *pick_glane_g(const ps_csr_t *csr, int loss)
{
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (f64 && i64) return kernel_ptr_glane<double, long long, G>(loss);
    if (f64) return kernel_ptr_glane<double, int, G>(loss);
    if (i64) return kernel_ptr_glane<float, long long, G>(loss);
    return kernel_ptr_glane<float, int, G>(loss);
}
static bool glane_ok(int G) { return G == 2 || G == 4 || G == 5 || G == 8 || G == 10 || G == 16; }
static void *pick_glane(const ps_csr_t *csr, int loss, int G)
{
    switch (G) {
    case 2: return pick_glane_g<2>(csr, loss);
    case 4: return pick_glane_g<4>(csr, loss);
    case 5: return pick_glane_g<5>(csr, loss);
    case 8: return pick_glane_g<8>(csr, loss);
    case 10: return pick_glane_g<10>(csr, loss);
    default: return pick_glane_g<16>(csr, loss);
    }
}

constexpr int GROUP_T = 512;
template <typename VT, typename PT> static void *kernel_ptr_group(int loss)
{
    if (loss == PS_LOSS_LOGISTIC) return (void *)sps_group_kernel<VT, PT, PS_LOSS_LOGISTIC, GROUP_T>;
    return (void *)sps_group_kernel<VT, PT, PS_LOSS_SQUARED, GROUP_T>;
}
static void *pick_group(const ps_csr_t *csr, int loss)
{
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (f64 && i64) return kernel_ptr_group<double, long long>(loss);
    if (f64) return kernel_ptr_group<double, int>(loss);
    if (i64) return kernel_ptr_group<float, long long>(loss);
    return kernel_ptr_group<float, int>(loss);
}
static void *pick_fast(const ps_csr_t *csr, int loss, int pen, int nc, bool small)
{
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (nc == 1) {
        if (f64 && i64) return kernel_ptr_fast<double, long long, 1>(loss, pen, small);
        if (f64) return kernel_ptr_fast<double, int, 1>(loss, pen, small);
        if (i64) return kernel_ptr_fast<float, long long, 1>(loss, pen, small);
        return kernel_ptr_fast<float, int, 1>(loss, pen, small);
    }
    if (f64 && i64) return kernel_ptr_fast<double, long long, 2>(loss, pen, small);
    if (f64) return kernel_ptr_fast<double, int, 2>(loss, pen, small);
    if (i64) return kernel_ptr_fast<float, long long, 2>(loss, pen, small);
    return kernel_ptr_fast<float, int, 2>(loss, pen, small);
}

static void *pick_kernel(const ps_csr_t *csr, int kind, bool big)
{
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    if (big) {
        if (f64 && i64) return kernel_ptr_big<double, long long>();
        if (f64) return kernel_ptr_big<double, int>();
        if (i64) return kernel_ptr_big<float, long long>();
        return kernel_ptr_big<float, int>();
    }
#define PICK(VT, PT)                                                                 \
    switch (kind) {                                                                  \
    case PS_PART_SINGLETON: return kernel_ptr<VT, PT, PS_PART_SINGLETON>();          \
    case PS_PART_CONTIG: return kernel_ptr<VT, PT, PS_PART_CONTIG>();                \
    default: return kernel_ptr<VT, PT, PS_PART_GENERAL>();                           \
    }
    if (f64 && i64) { PICK(double, long long) }
    if (f64) { PICK(double, int) }
    if (i64) { PICK(float, long long) }
    PICK(float, int)
#undef PICK
}

// Launch-geometry queries cached per (kernel, device, block, smem): the
// occupancy and cluster-residency queries and the dynamic-smem attribute cost
// tens of microseconds each in the driver and ran on every call (three
// launch_config evaluations per run_async: ~0.2 ms of a 2.8 ms end-to-end call)
namespace {
std::mutex g_geo_mu;
std::map<std::tuple<void *, int, int, size_t>, int> g_occ, g_clusters;
std::map<std::pair<void *, int>, size_t> g_smem_set;
cudaError_t cached_set_smem(void *k, int dev, size_t smem)
{
    std::lock_guard<std::mutex> g(g_geo_mu);
    size_t &have = g_smem_set[{k, dev}];
    if (have >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}
cudaError_t cached_occupancy(int *per_sm, void *k, int dev, int threads, size_t smem)
{
    std::lock_guard<std::mutex> g(g_geo_mu);
    auto key = std::make_tuple(k, dev, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
        *per_sm = it->second;
        return cudaSuccess;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k, threads, smem);
    if (e == cudaSuccess) g_occ[key] = *per_sm;
    return e;
}
// resident clusters of 2 for the kernel (-1: the query was refused)
int cached_pair_clusters(void *k, int dev, int threads, size_t smem, int ctas)
{
    std::lock_guard<std::mutex> g(g_geo_mu);
    auto key = std::make_tuple(k, dev, threads, smem);
    auto it = g_clusters.find(key);
    if (it != g_clusters.end()) return it->second;
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(ctas);
    q.blockDim = dim3(threads);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 2;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int resident = 0;
    if (cudaOccupancyMaxActiveClusters(&resident, k, &q) != cudaSuccess) resident = -1;
    cudaGetLastError();  // a refused query leaves no sticky error behind
    g_clusters[key] = resident;
    return resident;
}
}  // namespace

// pending-delta copies of sps_hot_kernel: flags bits 24..25 (0: default 1, else 1 << (v - 1))
static int hot2_ncopy(int flags)
{
    const int v = (flags >> 24) & 3;
    return v == 0 ? 1 : (1 << (v - 1));
}
struct LaunchCfg {
    int ncopy = 1;
    void *kernel;
    bool fast, hot2;
    int ctas, wpc, smem_flag, stride, M, GB, H, hot_doubles;
    size_t smem;
    int64_t gscratch_bytes;
};

static int launch_config(const ps_csr_t *csr, const ps_part_t *part, const ps_sched_t *sched, LaunchCfg *L,
                         const ps_params_t *prm = nullptr)
{
    const bool det = sched->samples != nullptr;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool diag_generic = (sched->flags & 16) != 0;
    const int pen = prm ? prm->penalty : PS_PEN_L1;
    // group-lasso fast kernel: contiguous blocks of G <= 16, rows <= 32 nonzeros
    const bool group_fast = !det && !diag_generic && part->kind == PS_PART_CONTIG && part->G <= 16 &&
                            part->max_row_nnz <= 32 && pen == PS_PEN_GROUP && sched->batch <= 0;
    // singleton rows of <= 32 (<= 64 for the fast kernel) nonzeros: one 24-warp
    // CTA per SM (fewest hot-flush agents, full register budget); else 8-warp CTAs
    const bool can_big = part->kind == PS_PART_SINGLETON && part->max_slots <= 32;
    const bool can_fast = part->kind == PS_PART_SINGLETON && part->max_slots <= 64 && !det && sched->batch <= 0 &&
                          !diag_generic && (sched->warps_per_cta <= 0 || sched->warps_per_cta == FAST_T / 32 ||
                                            sched->warps_per_cta == FAST_T_SMALL / 32);
    L->H = 0;
    L->hot2 = false;
    if (!det && (part->kind == PS_PART_SINGLETON || group_fast))
        L->H = std::min(HOT_MAX, std::max(0, (int)sched->hot_cols));
    int wpc;
    L->fast = false;
    if (group_fast && glane_ok(part->G) && (sched->hot_cols > 0 || (sched->flags & PS_FLAG_GROUP_LANE)) &&
        !(sched->flags & PS_FLAG_GROUP_WARP)) {
        // lane-per-block group kernel; hot blocks staged per CTA like hot columns
        // (opt-in: staging converges at small lambda but stalls near lambda_max,
        // see DESIGN.md; the default group path is the warp kernel, unstaged)
        L->wpc = wpc = (part->G <= 5 ? 768 : 512) / 32;
        const size_t warp_stage = (size_t)wpc * 32 * part->G * 8;
        L->H -= L->H % part->G;  // whole blocks
        while (L->H > 0 && warp_stage + (size_t)((3 + 2 * NCOPY) * L->H + HDR_DOUBLES) * 8 > 220 * 1024) L->H -= part->G;
        L->kernel = pick_glane(csr, prm ? prm->loss : PS_LOSS_LOGISTIC, part->G);
        L->hot_doubles = L->H > 0 ? (3 + 2 * NCOPY) * L->H : 0;
        L->smem = warp_stage + (L->H > 0 ? (size_t)(L->hot_doubles + HDR_DOUBLES) * 8 : 0);
        L->smem_flag = 0;
        L->stride = L->M = L->GB = 0;
        L->gscratch_bytes = 0;
        L->fast = true;
    } else if (group_fast) {
        wpc = GROUP_T / 32;
        const size_t warp_stage = (size_t)wpc * 4 * 32 * part->G * 8;
        // keep the CTA within the shared-memory budget: shrink the hot set (whole blocks)
        L->H -= L->H % part->G;  // whole blocks
        while (L->H > 0 && warp_stage + (size_t)((3 + 2 * NCOPY) * L->H + HDR_DOUBLES) * 8 > 220 * 1024) L->H -= part->G;
        L->kernel = pick_group(csr, prm ? prm->loss : PS_LOSS_LOGISTIC);
        L->wpc = wpc;
        L->hot_doubles = L->H > 0 ? (3 + 2 * NCOPY) * L->H : 0;
        L->smem = warp_stage + (L->H > 0 ? (size_t)(L->hot_doubles + HDR_DOUBLES) * 8 : 0);
        L->smem_flag = 0;
        L->stride = L->M = L->GB = 0;
        L->gscratch_bytes = 0;
        L->fast = true;
    } else {
        L->hot_doubles = L->H > 0 ? (3 + 2 * NCOPY) * L->H : 0;
        wpc = det ? 1 : (sched->warps_per_cta > 0 ? sched->warps_per_cta : (can_fast ? FAST_T / 32 : (can_big ? 24 : 8)));
        bool big = can_big && wpc > 8;
        // the pipelined fast kernel: static split, 768-thread CTAs (flags bit 4 forces the generic one)
        L->fast = can_fast && (wpc == FAST_T / 32 || wpc == FAST_T_SMALL / 32);
        if (L->fast) big = true;  // no per-warp scratch
        L->wpc = wpc = std::min(std::max(wpc, 1), big ? 32 : 8);
        L->kernel = pick_kernel(csr, part->kind, can_big && wpc > 8);
        if (L->fast)
            L->kernel = pick_fast(csr, prm ? prm->loss : PS_LOSS_LOGISTIC, pen, part->max_slots <= 32 ? 1 : 2,
                                  wpc == FAST_T_SMALL / 32);
        L->smem = L->H > 0 ? (size_t)(L->hot_doubles + HDR_DOUBLES) * 8 : 0;
        // second-generation hot kernel (fast2.cuh): rows <= 32 nonzeros, 32-warp CTAs
        L->hot2 = L->fast && part->max_slots <= 64 && wpc == FAST_T / 32 && !(sched->flags & PS_FLAG_FAST_V1) &&
                  ((sched->flags >> 8) & 0xff) == 0 && !(sched->flags & PS_FLAG_ZERO_IMMEDIATE) &&
                  csr->n_rows < (int64_t(1) << 32);
        if (L->hot2) {
            L->kernel = pick_hot(csr, prm ? prm->loss : PS_LOSS_LOGISTIC, pen, (sched->flags & PS_FLAG_DELTA_ZERO) != 0,
                                 part->max_slots <= 32 ? 1 : 2);
            L->ncopy = hot2_ncopy(sched->flags);
            L->hot_doubles = L->H > 0 ? hot2_doubles(L->H, L->ncopy) : 0;
            L->smem = (size_t)L->hot_doubles * 8 + (size_t)wpc * HOT2_BATCH_BYTES;  // + per-warp sample batches
        }
        L->smem_flag = 0;
        L->stride = L->M = L->GB = 0;
        L->gscratch_bytes = 0;
        if (needs_scratch(csr, part, big)) {
            L->stride = scratch_layout(csr, part, &L->M, &L->GB);
            size_t per_cta = (size_t)L->stride * 8 * wpc;
            if (per_cta + L->smem <= 96 * 1024) {
                L->smem_flag = 1;
                L->smem += per_cta;
            }
        }
    }
    if (L->smem > 48 * 1024) {
        cudaError_t e = cached_set_smem(L->kernel, dev, L->smem);
        if (e != cudaSuccess) return ps_cuda_fail(e, "ps_run smem attribute");
    }
    int per_sm = 1;
    cudaError_t e = cached_occupancy(&per_sm, L->kernel, dev, wpc * 32, L->smem);
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_run occupancy");
    per_sm = std::max(per_sm, 1);
    // default grid: one full wave, but no more than n/16 warps in flight so a
    // sample is rarely processed twice concurrently on small problems
    int64_t cap = std::max<int64_t>(1, csr->n_rows / (16 * (int64_t)wpc));
    L->ctas = det ? 1 : (sched->ctas > 0 ? sched->ctas : (int)std::min<int64_t>((int64_t)sms * per_sm, cap));
    if (L->stride > 0 && !L->smem_flag) L->gscratch_bytes = (int64_t)L->stride * 8 * wpc * L->ctas;
    return PS_OK;
}

extern "C" int ps_launch_config(const ps_csr_t *csr, const ps_part_t *part, const ps_sched_t *sched, int32_t *ctas,
                                int32_t *warps_per_cta, int64_t *scratch_bytes)
{
    if (!csr || !part || !sched) return ps_fail(PS_EINVAL, "null argument");
    LaunchCfg L;
    int r = launch_config(csr, part, sched, &L);
    if (r) return r;
    if (ctas) *ctas = L.ctas;
    if (warps_per_cta) *warps_per_cta = L.wpc;
    if (scratch_bytes) *scratch_bytes = L.gscratch_bytes;
    return PS_OK;
}

extern "C" int ps_run(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, double *coord,
                      double *alpha, const ps_sched_t *sched, void *scratch, void *stream)
{
    NvtxRange nvtx_range("K1/K2 ps_run");
    if (!csr || !part || !prm || !coord || !alpha || !sched) return ps_fail(PS_EINVAL, "null argument");
    if (csr->n_rows < 1) return ps_fail(PS_EINVAL, "dataset is empty");
    if (!(prm->gamma > 0)) return ps_fail(PS_EINVAL, "gamma must be positive");
    if (part->kind == PS_PART_CONTIG && (part->G < 1 || part->G > 32))
        return ps_fail(PS_EINVAL, "contiguous partition needs 1 <= G <= 32 (use GENERAL otherwise)");
    if (prm->penalty == PS_PEN_GROUP && part->kind == PS_PART_SINGLETON)
        return ps_fail(PS_EINVAL, "group penalty needs a CONTIG (G>=1) or GENERAL partition");
    if (sched->count < 0) return ps_fail(PS_EINVAL, "negative update count");
    if (sched->count == 0) return PS_OK;
    const bool det = sched->samples != nullptr;
    if (!det && !sched->counter) return ps_fail(PS_EINVAL, "async mode needs a device counter");

    KArgs a{};
    a.row_ptr = csr->row_ptr;
    a.col = csr->col_idx;
    a.val = csr->values;
    a.y = csr->labels;
    a.n = csr->n_rows;
    a.p = csr->n_cols;
    a.n_d = (double)csr->n_rows;
    a.G = part->G;
    a.blk_ptr = part->blk_ptr;
    a.blk_coords = part->blk_coords;
    a.row_blk = part->row_blk;
    a.row_g = part->row_g;
    a.spos = part->spos;
    a.blk_weight = part->blk_weight;
    a.coord = coord;
    a.alpha = alpha;
    a.loss = prm->loss;
    a.pen = prm->penalty;
    a.lambda1 = prm->lambda1;
    a.lam2 = prm->lam2;
    a.lo = prm->lo;
    a.hi = prm->hi;
    a.gamma = prm->gamma;
    a.samples = sched->samples;
    a.count = sched->count;
    {  // splitmix64(seed), host side
        uint64_t z = sched->seed + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        a.seed = z ^ (z >> 31);
    }
    a.slot_base = sched->slot_base;
    a.counter = sched->counter;
    if (det && (sched->trace_v != nullptr) != (sched->trace_dx != nullptr))
        return ps_fail(PS_EINVAL, "trace_v and trace_dx go together");
    a.trace_v = det ? sched->trace_v : nullptr;
    a.trace_dx = det ? sched->trace_dx : nullptr;
    a.batch = sched->batch;
    a.det = det ? 1 : 0;

    LaunchCfg L;
    int r = launch_config(csr, part, sched, &L, prm);
    if (r) return r;
    a.H = L.H;
    a.hot_doubles = L.hot_doubles;
    a.hot_shift = std::max(0, (int)sched->hot_shift);
    a.hot_unit = part->kind == PS_PART_CONTIG ? part->G : 1;
    a.scramble = 0;
    a.diag = sched->flags;
    if (sched->flags & 4) {  // diagnostics: permute the slot order within the call
        uint64_t m = 1000003ull;  // prime
        while ((uint64_t)sched->count % m == 0) m += 2;
        a.scramble = m % (uint64_t)sched->count ? m : 1;
    }
    // default flush period: 24 updates per warp for the singleton fast kernel
    // (32 warps per CTA), 16 elsewhere (tools/exp_floor2.py sweeps)
    a.period = sched->hot_period > 0 ? sched->hot_period : ((L.fast && part->kind == PS_PART_SINGLETON && L.wpc == FAST_T / 32) ? 24 : 16);
    // effective delay: in-flight warps + the staleness of the hot snapshot
    // (up to period * ctas updates between a CTA's refreshes)
    double tau = (double)((int64_t)L.ctas * L.wpc) + (a.H > 0 ? (double)a.period * L.ctas : 0.0);
    a.kappa = (!det && sched->contention > 0) ? sched->contention / tau : INFINITY;
    {  // diagnostics: flags bits 8..15 = extra divisor of the hot columns' kappa
        int div = (sched->flags >> 8) & 0xff;
        a.kappa_hot = a.kappa / (double)(div > 0 ? div : 1);
    }
    a.ncopy = L.ncopy;
    a.stride = L.stride;
    a.M = L.M;
    a.GB = L.GB;
    a.smem = L.smem_flag;
    if (L.gscratch_bytes > 0) {
        if (!scratch) return ps_fail(PS_EINVAL, "scratch buffer required (see ps_launch_config)");
        a.gscratch = (double *)scratch;
    }
    // fast singleton kernel with staging: CTA pairs (thread-block clusters of 2)
    // share the hot snapshot refresh -- the second CTA reads the first's
    // snapshot through distributed shared memory, halving the refresh reads of
    // the hot records at L2 (config 2: +15-20% updates/s, same epochs to 1e-6;
    // clusters of 4 do not all fit co-resident and run at 0.65x).  Used only
    // when every cluster of the grid can be resident at once.
    a.cluster = 1;
    // (sps_hot_kernel: only up to 512 staged columns -- with 1024 the members'
    // second-hand tier-2 refresh measured unstable on a config-3-like
    // instance, tools/gpu/dbg_knobs.py, and round 1 measured no gain there)
    if (L.fast && part->kind == PS_PART_SINGLETON && a.H > 0 && !(sched->flags & PS_FLAG_NO_CLUSTER) &&
        L.ctas % 2 == 0 && !(L.hot2 && a.H > 512)) {
        int dev = 0;
        cudaGetDevice(&dev);
        const int resident = cached_pair_clusters(L.kernel, dev, L.wpc * 32, L.smem, L.ctas);
        if (resident > 0 && 2 * resident >= L.ctas) a.cluster = 2;
    }
    void *args[] = {(void *)&a};
    cudaError_t e;
    // deterministic replay with the state on chip (sps_det_smem_kernel)
    const size_t det_smem = (size_t)(3 * csr->n_cols + csr->n_rows) * sizeof(double);
    if (det && part->kind == PS_PART_SINGLETON && part->max_slots <= 64 && prm->penalty != PS_PEN_GROUP &&
        det_smem <= 200 * 1024 && !(sched->flags & PS_FLAG_GENERIC)) {
        void *k = pick_det_smem(csr);
        int dev = 0;
        cudaGetDevice(&dev);
        if (det_smem > 48 * 1024) {
            e = cached_set_smem(k, dev, det_smem);
            if (e != cudaSuccess) return ps_cuda_fail(e, "ps_run det smem attribute");
        }
        e = cudaLaunchKernel(k, dim3(1), dim3(32), args, det_smem, (cudaStream_t)stream);
        if (e != cudaSuccess) return ps_cuda_fail(e, "ps_run launch");
        return PS_OK;
    }
    if (a.cluster > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(L.ctas);
        cfg.blockDim = dim3(L.wpc * 32);
        cfg.dynamicSmemBytes = L.smem;
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)a.cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelExC(&cfg, L.kernel, args);
    } else {
        e = cudaLaunchKernel(L.kernel, dim3(L.ctas), dim3(L.wpc * 32), args, L.smem, (cudaStream_t)stream);
    }
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_run launch");
    return PS_OK;
}

// x of the live coordinate records into a device snapshot (the monitor's
// device mode: a few CTAs beside the solve, which leaves them the SMs)
namespace ps {
constexpr int SNAP_CTAS = 8;
__global__ void __launch_bounds__(1024) k_snap_x(const double *coord, double *dst, int64_t p)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        dst[j] = __ldcg(coord + 4 * j);
}
}  // namespace ps

// ---------------------------------------------------------------------------
// ps_run_monitored: the reference's monitor (asynchronous.py:187-198) on the
// device.  One asynchronous launch runs the whole solve; this (host) thread
// polls the progress counter and, each time it crosses a checkpoint mark,
// snapshots the live coordinate records into (pinned) host memory on a copy
// stream -- a copy-engine DMA that runs beside the kernel (a device-to-device
// memcpy would need SMs and wait for the launch), i.e. an inconsistent
// snapshot taken while the warps keep updating, as snapshot_x
// (asynchronous.py:65-66) is -- and records an event after it.  The solve
// never stops for a checkpoint.  Objectives of the snapshots are evaluated by
// the caller afterwards (ps_objective, stride 4).
extern "C" int ps_run_monitored(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, double *coord,
                                double *alpha, const ps_sched_t *sched, void *scratch, void *stream, int64_t every,
                                int32_t max_snaps, double *snaps, int64_t *snap_counts, float *snap_ms,
                                int32_t *n_snaps)
{
    NvtxRange nvtx_range("K6 ps_run_monitored");
    if (!sched || !snaps || !snap_counts || !snap_ms || !n_snaps || every < 1 || max_snaps < 1)
        return ps_fail(PS_EINVAL, "bad monitor arguments");
    if (sched->samples) return ps_fail(PS_EINVAL, "the monitor is for asynchronous runs");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t p = csr->n_cols, total = sched->count;
    // per-device monitor resources, created once and kept: copy + poll streams,
    // a pinned counter mirror, a growing pool of events
    struct Mon {
        cudaStream_t cp = nullptr, poll = nullptr;
        unsigned long long *h_cnt = nullptr;
        cudaEvent_t ev0 = nullptr;
        std::vector<cudaEvent_t> evs;
    };
    static Mon mons[64];
    static std::mutex locks[64];  // one monitored run per device at a time (shared resources)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return ps_fail(PS_EINVAL, "device index out of range");
    std::lock_guard<std::mutex> guard(locks[dev]);
    Mon &m = mons[dev];
    int rc = PS_OK;
#define MCK(x, what)                                       \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) {                           \
            rc = ps_cuda_fail(e_, what);                   \
            return rc;                                     \
        }                                                  \
    } while (0)
    if (!m.cp) {
        MCK(cudaStreamCreateWithFlags(&m.cp, cudaStreamNonBlocking), "monitor stream");
        MCK(cudaStreamCreateWithFlags(&m.poll, cudaStreamNonBlocking), "monitor stream");
        MCK(cudaMallocHost((void **)&m.h_cnt, sizeof(unsigned long long)), "monitor pinned counter");
        MCK(cudaEventCreate(&m.ev0), "monitor event");
    }
    while ((int)m.evs.size() < max_snaps) {
        cudaEvent_t e;
        MCK(cudaEventCreate(&e), "monitor event");
        m.evs.push_back(e);
    }
    cudaStream_t cp = m.cp, poll = m.poll;
    cudaEvent_t ev0 = m.ev0;
    std::vector<cudaEvent_t> &evs = m.evs;
    unsigned long long *h_cnt = m.h_cnt;
    // device mode (PS_FLAG_MON_DEVICE_X): x-only snapshots into device memory by
    // k_snap_x on SNAP_CTAS SMs the solve leaves free (host snapshots of all the
    // records of a 3e7-coordinate problem cost more PCIe time than an epoch)
    const bool dev_x = (sched->flags & PS_FLAG_MON_DEVICE_X) != 0;
    if (dev_x) {
        // load k_snap_x now: a lazily loaded kernel's first launch waits for the
        // device to go idle, i.e. for the solve (measured: first snapshot at the end)
        cudaFuncAttributes fa;
        MCK(cudaFuncGetAttributes(&fa, k_snap_x), "monitor snapshot kernel");
    }
    ps_sched_t s2 = *sched;
    if (dev_x && s2.ctas <= 0) {
        int32_t c0 = 0, w0 = 0;
        int64_t sb = 0;
        int r0 = ps_launch_config(csr, part, sched, &c0, &w0, &sb);
        if (r0) return r0;
        s2.ctas = std::max(2, (c0 - SNAP_CTAS) & ~1);
    }
    const int64_t rec = dev_x ? 1 : 4;  // doubles per coordinate in a snapshot
    auto snapshot = [&](int k, cudaStream_t on) -> cudaError_t {
        if (dev_x) {
            k_snap_x<<<SNAP_CTAS, 1024, 0, on>>>(coord, snaps + (size_t)k * p, p);
            return cudaGetLastError();
        }
        return cudaMemcpyAsync(snaps + (size_t)k * 4 * p, coord, sizeof(double) * 4 * p, cudaMemcpyDeviceToHost, on);
    };
    (void)rec;
    MCK(cudaMemsetAsync(sched->counter, 0, sizeof(unsigned long long), st), "monitor counter reset");
    MCK(cudaEventRecord(ev0, st), "monitor event");
    const bool ends_in_place = (sched->flags & PS_FLAG_MON_ENDS_IN_PLACE) != 0;
    // checkpoint 0: the state before the first update (asynchronous.py:181)
    int ns = 0;
    if (ends_in_place) {
        MCK(cudaEventRecord(evs[0], st), "monitor event");
    } else {
        MCK(cudaStreamWaitEvent(cp, ev0, 0), "monitor wait");
        MCK(snapshot(0, cp), "monitor snapshot");
        MCK(cudaEventRecord(evs[0], cp), "monitor event");
        // the solve must not start before snapshot 0 is taken
        MCK(cudaStreamWaitEvent(st, evs[0], 0), "monitor wait");
    }
    snap_counts[0] = 0;
    ns = 1;
    int r = ps_run(csr, part, prm, coord, alpha, &s2, scratch, stream);
    if (r) return r;
    int64_t next_mark = every;
    while (true) {
        const bool done = cudaStreamQuery(st) == cudaSuccess;
        if (done) break;
        MCK(cudaMemcpyAsync(h_cnt, sched->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, poll),
            "monitor poll");
        MCK(cudaStreamSynchronize(poll), "monitor poll");
        const int64_t c = (int64_t)*h_cnt;
        if (c >= next_mark && next_mark < total && ns < max_snaps - 1) {
            MCK(snapshot(ns, cp), "monitor snapshot");
            MCK(cudaEventRecord(evs[ns], cp), "monitor event");
            snap_counts[ns++] = c;
            while (next_mark <= c) next_mark += every;
        }
    }
    // final checkpoint: after the launch (consistent)
    MCK(cudaStreamWaitEvent(cp, ev0, 0), "monitor wait");
    MCK(cudaStreamSynchronize(st), "monitor join");
    if (!ends_in_place) MCK(snapshot(ns, st), "monitor snapshot");
    MCK(cudaEventRecord(evs[ns], st), "monitor event");
    if (ends_in_place) {
        // the last checkpoint comes after the launch AND after every snapshot copy
        // still in flight on the copy stream (checkpoint times stay monotone)
        MCK(cudaStreamWaitEvent(cp, evs[ns], 0), "monitor wait");
        MCK(cudaEventRecord(evs[ns], cp), "monitor event");
    }
    snap_counts[ns++] = total;
    MCK(cudaStreamSynchronize(st), "monitor join");
    MCK(cudaStreamSynchronize(cp), "monitor join");
    for (int k = 0; k < ns; k++) MCK(cudaEventElapsedTime(snap_ms + k, ev0, evs[k]), "monitor timing");
    *n_snaps = ns;
#undef MCK
    return PS_OK;
}

// ps_loss_deriv: the kernels' loss derivative applied elementwise (test /
// inspection hook).  fast = 1 is the asynchronous kernels' deriv_t.
namespace ps {
__global__ void k_loss_deriv(int loss, int fast, const double *z, const double *b, int64_t m, double *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (!fast) out[i] = loss_deriv(loss, z[i], b[i]);
        else if (fast == 2) out[i] = loss == PS_LOSS_LOGISTIC ? deriv_t<PS_LOSS_LOGISTIC>(z[i], b[i])
                                                              : deriv_t<PS_LOSS_SQUARED>(z[i], b[i]);
        else out[i] = loss == PS_LOSS_LOGISTIC ? deriv2<PS_LOSS_LOGISTIC>(z[i], b[i])
                                               : deriv2<PS_LOSS_SQUARED>(z[i], b[i]);
    }
}
__global__ void k_loss_eval(int loss, const double *z, const double *b, int64_t m, double *val, double *der)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (val) val[i] = loss_value(loss, z[i], b[i]);
        if (der) der[i] = loss_deriv(loss, z[i], b[i]);
    }
}
}  // namespace ps

extern "C" int ps_loss_eval(int32_t loss, const double *z, const double *b, int64_t m, double *value, double *deriv,
                            void *stream)
{
    if (loss != PS_LOSS_LOGISTIC && loss != PS_LOSS_SQUARED) return ps_fail(PS_EINVAL, "unknown loss");
    if (m < 0 || (m > 0 && (!z || !b || (!value && !deriv)))) return ps_fail(PS_EINVAL, "bad loss_eval arguments");
    if (m == 0) return PS_OK;
    ps::k_loss_eval<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(loss, z, b, m,
                                                                                                      value, deriv);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_loss_eval launch");
    return PS_OK;
}

extern "C" int ps_loss_deriv(int32_t loss, int32_t fast, const double *z, const double *b, int64_t m, double *out,
                             void *stream)
{
    if (loss != PS_LOSS_LOGISTIC && loss != PS_LOSS_SQUARED) return ps_fail(PS_EINVAL, "unknown loss");
    if (m < 0 || (m > 0 && (!z || !b || !out))) return ps_fail(PS_EINVAL, "bad loss_deriv arguments");
    if (m == 0) return PS_OK;
    ps::k_loss_deriv<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(loss, fast, z,
                                                                                                       b, m, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_loss_deriv launch");
    return PS_OK;
}
