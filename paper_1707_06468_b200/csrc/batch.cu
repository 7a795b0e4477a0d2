// Lambda-batched group-lasso SPS (BASELINE config 5; SURVEY §8(e) "Option").
//
// B independent solves of the same problem that differ only in the penalty
// weight (a regularisation path) share every sampled row: one warp reads row
// i once -- the sample, the CSR extent, its columns / values / label, its
// distinct blocks T_i -- and applies the Sparse Proximal SAGA step
// (saga.py:150-185 / asynchronous.py:80-117, group prox penalties.py:103-108)
// to all B lambda-states.  The per-sample scalar work (margin reduction,
// logistic derivative, alpha exchange) runs once per lane for B states in
// parallel instead of once per warp per state.
//
// State layout (bidx below): states in groups of 2, each group its own
// region [block][q][2](x, abar) followed by a hot area where the most frequent
// blocks keep one coordinate per KB, x and abar in separate sectors (the L2
// serialises the atomics of a 128-B line); alpha[i*B + beta]; the block weights d_B come from ps_prepare
// (part->blk_weight).  The first block of T_i is loaded once per row (margin
// and prox share it), stored block 0 at most every hshare-th row per warp.
//
// Lane mapping: LPB = 32/B lanes per state; lane l works on state l % B and
// on the block coordinates q = l / B + LPB r.  Rows of <= 32 nonzeros,
// contiguous blocks of G <= 16.  Asynchronous mode: one warp per in-flight
// row, REDs on x / abar, atomicExch on alpha (asynchronous.py's atomics);
// deterministic mode (sched->samples): one warp, plain stores in sps_step's
// order (x = x^ + (z - x^), abar += ((new - alpha_i)/n) a_i, alpha_i = new).
#include <algorithm>
#include <cstdio>

#include "fastmath.cuh"
#include "internal.h"

namespace ps {

// state layout (bidx below)
struct BLay {
    int64_t body, region, hstride;  // doubles: nb*G*S*2; body + hot area + pad; per scattered coordinate
    int32_t G, S, hshift, nhot;
    int32_t hab;  // hot slots: doubles from the x sector to the abar sector (0: one packed (x, abar) sector)
};

struct BArgs {
    const int32_t *row_ptr;
    const int32_t *col;
    const void *val, *y;
    int64_t n, p;
    int32_t G;
    const double *bd;   // d_B per block
    double *state;      // see above
    double *alpha;      // [n][B]
    const double *lam2; // [B]
    int32_t loss;
    double lambda1, gamma, kappa, n_d;
    int64_t nb;  // blocks (ceil(p / G))
    // schedule
    const int64_t *samples;
    int64_t count;
    uint64_t seed, slot_base;
    unsigned long long *counter;
    int32_t det, skip_zero;
    // replicated x-delta accumulators of the hottest blocks (asynchronous mode):
    // stored block b with (b & hmask) == 0 and rank b >> hshift < nrb commits its
    // x deltas to replica (warp % nrep) of xrep[nrep][nrb][G][B]; a read of its x
    // is the state's x plus every replica; k_batch_fold folds them after the launch
    double *xrep;
    int32_t nrep, nrb, hshift;
    int64_t rpad, rstride;  // state region pad; doubles per (replica, hot block) chunk
    BLay L;                 // state layout (bidx)
    int32_t hshare;         // > 0: the CTA shares its loads of stored block 0 (see the kernel)
};

#ifndef BATCH_THREADS
#define BATCH_THREADS 512
#endif
constexpr int BATCH_T = BATCH_THREADS;  // threads per CTA (16 warps; A/B knob)
// A/B knob: -DBATCH_MINB=2 caps the kernel at 64 registers (two CTAs per SM)
#ifdef BATCH_MINB
#define BATCH_BOUNDS __launch_bounds__(BATCH_T, BATCH_MINB)
#else
#define BATCH_BOUNDS __launch_bounds__(BATCH_T)
#endif
// State layout: states are grouped S = 2 at a time (one 32-B sector per
// coordinate and group); group g of the B states is its own region
//   state[((g * NB*G + j) * S + beta % S) * 2 + {0: x, 1: abar}],  g = beta / S
// so a block's B states sit in B/S regions (hundreds of MB apart): the REDs
// of a hot block -- every row updates the Zipf head's blocks -- reach B/S
// times more L2 slices than one contiguous [b][q][beta] record (ncu: one
// slice's atomic unit 88% busy with the contiguous record, 20.5 M rows/s
// whatever the grid; 22.2 M with the groups), at the same sectors per warp
// access.  A region per (group, q) (G*B/S regions) spreads them further but
// measured slower (16.2 M rows/s: each lane's loads of a block land in
// different 2 MB pages).
constexpr int BATCH_S = 2;
constexpr int PROGRESS_BATCH_B = 16;           // rows per progress bump of a warp
constexpr int BATCH_SM_WARP = 32 + 32 * 16;    // per-warp shared doubles: block ids + row values [32][16]
constexpr int BATCH_SM_SHARE = 32 * 8 * 2;     // per-CTA shared doubles: stored block 0's (x, abar) per (lane, r)
// Region g of the state is [body | hot area | pad]: body = nb*G*S*2 doubles in
// [block][q][S](x, abar) order.  SCATTERED HOT BLOCKS: stored block b with
// (b & ((1 << hshift) - 1)) == 0 and rank r = b >> hshift < nhot (the most
// frequent blocks of ps_hot_layout's spread order; the first nhot blocks when
// hshift = 0) keeps its coordinates in the hot area instead, coordinate q at
// (r*G + q) * hstride doubles -- one 32-B sector (the S states' (x, abar)
// pairs) per hstride (1 KB).  Every row commits all G coordinates of the Zipf
// head's blocks in every state; in the contiguous record four coordinates
// share a line and the L2 serialises a line's atomics (measured, config 5,
// tools/gpu/exp_batch_scatter.py: B = 16 24.9 -> 39.8 M rows/s, B = 8 25.3 ->
// 63.3, B = 4 43.5 -> 84.5, B = 2 78.8 -> 115 -- more than the replica
// accumulators gave, which it replaces by default).  The pad (diagnostics)
// shifts the regions against each other.
__host__ __device__ __forceinline__ int64_t bidx(int64_t b, int q, int beta, int field, const BLay &L)
{
    const int slot = beta % L.S;
    const int64_t base = (int64_t)(beta / L.S) * L.region;
    const int64_t r = b >> L.hshift;
    if (r < L.nhot && (b & ((1ll << L.hshift) - 1)) == 0) {
        const int64_t hslot = base + L.body + (r * L.G + q) * L.hstride;
        return L.hab ? hslot + slot + (int64_t)field * L.hab : hslot + slot * 2 + field;
    }
    return base + ((b * L.G + q) * L.S + slot) * 2 + field;
}
// the same address split for the kernel's block loops: coordinate q of stored
// block b in this lane's state lives at lane_base + off + q * qs, with
// lane_base = bidx(0, 0, beta) fixed per lane -- one hot test per block
// instead of one per coordinate access
// (hot slots with separate x / abar sectors: off carries the lane's -slot, the
// abar of a coordinate sits da doubles after its x; da = 1 everywhere else)
__device__ __forceinline__ void bref(int64_t b, int slot, const BLay &L, int64_t &off, int &qs, int &da)
{
    const int64_t r = b >> L.hshift;
    const bool hot = r < L.nhot && (b & ((1ll << L.hshift) - 1)) == 0;
    off = hot ? L.body + r * (L.G * L.hstride) - (L.hab ? slot : 0) : b * (L.G * L.S * 2);
    qs = hot ? (int)L.hstride : L.S * 2;
    da = hot && L.hab ? L.hab : 1;
}
// an (x, abar) pair: one 16-B load where they are adjacent
__device__ __forceinline__ double2 ld_pair(const double *px, int da)
{
    if (da == 1) return ld_cg2(px);
    return make_double2(ld_cg(px), ld_cg(px + da));
}
// layout knobs (doubles): the region pad and the stride of one (replica, hot
// block) chunk of the replica accumulators; set by ps_batch_tune (diagnostics)
static int64_t g_rpad = 0, g_rstride = 128;  // 1 KB replica chunks (tools/gpu/exp_batch_pad.py)
static int64_t g_hstride = 128;  // scattered hot blocks: one sector per KB (adjacent lines measured slower below B = 16)
static int32_t g_last_ctas = 0, g_last_wpc = 0;  // grid of the last ps_batch_run launch (ps_batch_last_grid)
static int32_t g_hab = -1;       // hot slots: the abar sector this many doubles after the x sector (0: packed;
                                 // -1: 64 = 512 B from B = 4, packed below: tools/gpu/exp_batch_scatter.py); ps_batch_tune2
static int32_t g_hshare = 4;     // rows between a warp's own L2 loads of stored block 0 (0: every row); ps_batch_tune2
static int32_t g_nhot = -1;      // how many: -1 = by B (128 from B = 8, else 32: tools/gpu/exp_batch_scatter.py); ps_batch_tune2

// rank of a replicated hot block, or -1
template <bool REP> __device__ __forceinline__ int rep_rank(const BArgs &a, int64_t b)
{
    if (!REP) return -1;
    const int64_t r = b >> a.hshift;
    return ((b & ((1ll << a.hshift) - 1)) == 0 && r < a.nrb) ? (int)r : -1;
}
__device__ __forceinline__ double *rep_ptr(const BArgs &a, int rr, int rank, int q, int beta, int B, int G)
{
    return a.xrep + ((int64_t)rr * a.nrb + rank) * a.rstride + q * B + beta;
}

template <typename VT, int LOSS, int B, int GT, bool REP>
__global__ void BATCH_BOUNDS sps_group_batch_kernel(const BArgs a)
{
    constexpr int LPB = 32 / B;                                  // lanes per state
    constexpr int S = B < BATCH_S ? B : BATCH_S;                 // states per layout group
    constexpr int RMAX = ((GT > 0 ? GT : 16) + LPB - 1) / LPB;   // block coordinates per lane
    extern __shared__ double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    const int beta = lane % B, sub = lane / B;
    int *sblk = reinterpret_cast<int *>(smem_dyn + (size_t)wib * BATCH_SM_WARP);
    double *sa = smem_dyn + (size_t)wib * BATCH_SM_WARP + 32;  // [rank][16]
    const int G = GT > 0 ? GT : a.G;
    const int64_t p = a.p;
    double *const st = a.state + ((int64_t)(beta / a.L.S) * a.L.region + (beta % a.L.S) * 2);  // this lane's state (region, slot)
    const double lam2 = a.lam2[beta];
    // CTA-shared loads of stored block 0 (the most frequent block: in ~every row of a
    // Zipf-headed problem): every warp needs its G x B (x, abar) pairs at the start of
    // every row, and those loads queue behind everyone's REDs on the same lines.  Each
    // warp loads them from L2 on every hshare-th row only (staggered by warp) and
    // publishes them here; on its other rows it reads this copy, which another warp of
    // the CTA refreshed a fraction of a row time ago -- an inconsistent read like any
    // other here (the row takes ~16 block updates to commit, with thousands of rows in
    // flight).  Nothing is write-combined: every delta still goes to L2 at once, so
    // abar stays the exact average and the certified gaps are unchanged (K3b).
    double2 *const hs = reinterpret_cast<double2 *>(smem_dyn + (size_t)nwib * BATCH_SM_WARP) + lane * RMAX;
    const bool share = !REP && !a.det && a.hshare > 0 && a.nb > 1;
    if (share) {
        if (wib == 0) {
            int64_t o0;
            int q0, d0;
            bref(0, beta % S, a.L, o0, q0, d0);
#pragma unroll
            for (int r = 0; r < RMAX; r++) {
                const int q = sub + LPB * r;
                hs[r] = q < G ? ld_pair(st + o0 + q * q0, d0)
                              : make_double2(0.0, 0.0);
            }
        }
        __syncthreads();
    }
    const VT *valp = reinterpret_cast<const VT *>(a.val);
    const VT *yp = reinterpret_cast<const VT *>(a.y);

    const int64_t nwarps = (int64_t)gridDim.x * nwib;
    int64_t t0, t1;
    if (a.det) {
        if (gw != 0) return;
        t0 = 0;
        t1 = a.count;
    } else {
        const int64_t q = a.count / nwarps, r = a.count % nwarps;
        t0 = gw * q + min(gw, r);
        t1 = t0 + q + (gw < r ? 1 : 0);
    }
    int64_t done = 0;
    for (int64_t t = t0; t < t1; t++) {
        const int64_t i = a.det ? __ldg(a.samples + t) : sample_row(a.seed, a.slot_base + (uint64_t)t, (uint64_t)a.n);
        const int lo = __ldg(a.row_ptr + i), k = __ldg(a.row_ptr + i + 1) - lo;
        // ---- the row's nonzeros (lane e) and distinct blocks (ranks)
        int col = -1;
        double val = 0.0;
        if (lane < k) {
            col = __ldg(a.col + lo + lane);
            val = widen(__ldg(valp + lo + lane));
        }
        // this lane's nonzero: the offset of x[col] from any lane's state base (one
        // layout lookup per nonzero; the margin loads and the abar REDs take it by shuffle)
        int64_t eoff = 0;  // bit 0: a hot slot with separate x / abar sectors (the reader subtracts its slot)
        if (col >= 0) {
            const int be = col / G;
            int eqs, eda;
            bref(be, 0, a.L, eoff, eqs, eda);
            eoff += (col - be * G) * eqs + (eda != 1 ? 1 : 0);
        }
        const double yb = widen(__ldg(yp + i));
        double old = 0.0;  // alpha_i of this lane's state (lanes < B)
        if (sub == 0) old = a.det ? a.alpha[i * B + beta] : ld_cg(a.alpha + i * B + beta);
        const int blk = col >= 0 ? col / G : -1 - lane;
        const unsigned peers = __match_any_sync(FULL, blk);
        const int lead = __ffs(peers) - 1;
        const unsigned leaders = __ballot_sync(FULL, col >= 0 && lead == lane);
        const int g = __popc(leaders);
        const int rank = __popc(leaders & ((1u << lead) - 1u));
        for (int s = lane; s < g * 16; s += 32) sa[s] = 0.0;
        __syncwarp();
        if (col >= 0) {
            sa[rank * 16 + (col - blk * G)] = val;
            if (lead == lane) sblk[rank] = blk;
        }
        __syncwarp();
        auto load_blk = [&](int tb, double2 *v, int64_t &off, int &qs, int &da) {
            const int b = sblk[tb];
            const int nq = (int)min((int64_t)G, p - (int64_t)b * G);  // ragged last block
            const int rk = rep_rank<REP>(a, b);
            bref(b, beta % S, a.L, off, qs, da);
#pragma unroll
            for (int r = 0; r < RMAX; r++) {
                const int q = sub + LPB * r;
                v[r] = q < nq ? ld_pair(st + off + q * qs, da) : make_double2(0.0, 0.0);
                if (rk >= 0 && q < nq)
                    for (int rr = 0; rr < a.nrep; rr++) v[r].x += ld_cg(rep_ptr(a, rr, rk, q, beta, B, G));
            }
        };
        // the first block of T_i (the hottest one present: the smallest stored index) is
        // loaded once, ahead of the margin: its x values feed the margin AND the block
        // update below, so the hottest lines take one load per row instead of two
        // (sps_step gathers x_hat once, saga.py:169-172)
        double2 bufa[RMAX], bufb[RMAX];
        int64_t aoff = 0, boff = 0;
        int aqs = 0, bqs = 0, ada = 1, bda = 1;
        const bool hot0 = share && g > 0 && sblk[0] == 0;
        const bool fresh = !hot0 || (done + wib) % a.hshare == 0;
        if (g > 0 && fresh) load_blk(0, bufa, aoff, aqs, ada);
        if (hot0 && !fresh) {
            bref(0, beta % S, a.L, aoff, aqs, ada);
#pragma unroll
            for (int r = 0; r < RMAX; r++) bufa[r] = hs[r];
        }
        const unsigned first0 = __ballot_sync(FULL, col >= 0 && rank == 0);  // nonzeros in that block
        // margin loads: x[col_e][beta] for this lane's other nonzeros e = sub + LPB j
        double xm[(32 + LPB - 1) / LPB];
#pragma unroll
        for (int j = 0; j < (32 + LPB - 1) / LPB; j++) {
            const int e = sub + LPB * j;
            const int64_t mo = __shfl_sync(FULL, eoff, e & 31);
            const bool need = e < k && !((first0 >> (e & 31)) & 1u);
            xm[j] = need ? ld_cg(st + (mo & ~1ll) - ((mo & 1) ? beta % S : 0)) : 0.0;
            if (REP) {
                const int ce = __shfl_sync(FULL, col, e & 31);
                const int rk = need ? rep_rank<REP>(a, ce / G) : -1;
                if (rk >= 0)
                    for (int rr = 0; rr < a.nrep; rr++) xm[j] += ld_cg(rep_ptr(a, rr, rk, ce - (ce / G) * G, beta, B, G));
            }
        }
        // block weights of T_i: lane t holds d_B of rank t
        double dB = 0.0;
        if (lane < g) dB = __ldg(a.bd + sblk[lane]);
        // ---- margins
        double part = 0.0;
#pragma unroll
        for (int j = 0; j < (32 + LPB - 1) / LPB; j++) {
            const int e = sub + LPB * j;
            const double ve = __shfl_sync(FULL, val, e & 31);
            part = __fma_rn(ve, xm[j], part);  // xm = 0 past the row
        }
        if (g > 0) {  // the first block's nonzeros, from its loaded coordinates (sa = 0 where the row has none)
#pragma unroll
            for (int r = 0; r < RMAX; r++) {
                const int q = sub + LPB * r;
                if (q < G) part = __fma_rn(sa[q], bufa[r].x, part);
            }
            if (hot0 && fresh) {  // publish this warp's load of stored block 0
#pragma unroll
                for (int r = 0; r < RMAX; r++) hs[r] = bufa[r];
            }
        }
#pragma unroll
        for (int o = B; o < 32; o <<= 1) part += __shfl_xor_sync(FULL, part, o);
        old = __shfl_sync(FULL, old, beta);
        const double nw = LOSS == PS_LOSS_LOGISTIC ? deriv2<PS_LOSS_LOGISTIC>(part, yb) : part - yb;
        const double ds = nw - old;
        // alpha_i <- new now (the exchange returns while the blocks are updated)
        double rep = old;
        if (sub == 0) {
            if (a.det) a.alpha[i * B + beta] = nw;
            else rep = atomic_exch(a.alpha + i * B + beta, nw);
        }
        // ---- every block of T_i, all B states; the next block's state loads
        // are issued before the current block is computed
        // two buffers in turn (no register copies between blocks)
        auto process = [&](int tb, const double2 *cur, const int64_t coff, const int cqs, const int cda) {
            const int b = sblk[tb];
            const double d = __shfl_sync(FULL, dB, tb);
            const double kd = a.kappa * d;
            const double gB = a.gamma * (kd < 1.0 ? kd : 1.0);
            const int nq = (int)min((int64_t)G, p - (int64_t)b * G);
            double u[RMAX];
            double ss = 0.0;
            bool zero = true;
#pragma unroll
            for (int r = 0; r < RMAX; r++) {
                const int q = sub + LPB * r;
                u[r] = 0.0;
                if (q < nq) {
                    const double vv = __fma_rn(ds, sa[tb * 16 + q], d * __fma_rn(a.lambda1, cur[r].x, cur[r].y));
                    u[r] = __fma_rn(-gB, vv, cur[r].x);
                    ss = __fma_rn(u[r], u[r], ss);
                    zero = zero && cur[r].x == 0.0;
                }
            }
#pragma unroll
            for (int o = B; o < 32; o <<= 1) {
                ss += __shfl_xor_sync(FULL, ss, o);
                zero = (__shfl_xor_sync(FULL, (int)zero, o) != 0) && zero;
            }
            // deterministic mode: penalties.py:103-108's arithmetic (sqrt, divide); asynchronous:
            // one reciprocal square root (the objective-level parity of the async kernels)
            const double f = a.det ? group_factor(sqrt(ss), gB * d, lam2)
                                   : (ss > 0.0 ? fmax(0.0, __fma_rn(-(gB * d * lam2), rsqrt(ss), 1.0)) : 0.0);
            // zero block kept at zero: delta 0, nothing committed (the lane
            // kernel's skip); a zeroed block is stored (zero commits)
            if (!(f == 0.0 && zero && a.skip_zero)) {
                const int rk = a.det ? -1 : rep_rank<REP>(a, b);
#pragma unroll
                for (int r = 0; r < RMAX; r++) {
                    const int q = sub + LPB * r;
                    if (q < nq) {
                        double *px = st + coff + q * cqs;
                        const double z = u[r] * f;
                        if (a.det) {
                            *px = cur[r].x + (z - cur[r].x);
                        } else if (f == 0.0) {  // a zeroed block is stored: the state and every replica
                            atomic_exch(px, 0.0);
                            if (rk >= 0)
                                for (int rr = 0; rr < a.nrep; rr++) atomic_exch(rep_ptr(a, rr, rk, q, beta, B, G), 0.0);
                        } else {
                            red_add(rk >= 0 ? rep_ptr(a, (int)(gw % a.nrep), rk, q, beta, B, G) : px, z - cur[r].x);
                        }
                    }
                }
            }
        };
        for (int tb = 0; tb < g; tb += 2) {  // block 0 is in bufa already
            if (tb + 1 < g) load_blk(tb + 1, bufb, boff, bqs, bda);
            process(tb, bufa, aoff, aqs, ada);
            if (tb + 1 < g) {
                if (tb + 2 < g) load_blk(tb + 2, bufa, aoff, aqs, ada);
                process(tb + 1, bufb, boff, bqs, bda);
            }
        }
        // ---- abar on S_i: ((new - replaced)/n) a_i
        rep = __shfl_sync(FULL, rep, beta);
        const double tq = (nw - rep) / a.n_d;  // saga.py:182-184: (delta / n) * vals
        for (int e0 = 0; e0 < k; e0 += LPB) {
            const int e = e0 + sub;
            const int64_t ao = __shfl_sync(FULL, eoff, e & 31);
            const double ve = __shfl_sync(FULL, val, e & 31);
            if (e < k) {
                double *pab = (ao & 1) ? st + (ao & ~1ll) - beta % S + a.L.hab : st + ao + 1;
                if (a.det) *pab = *pab + tq * ve;
                else red_add(pab, tq * ve);
            }
        }
        if (a.det) {
            __threadfence();
        } else if (lane == 0 && ++done % PROGRESS_BATCH_B == 0) {
            atomicAdd(a.counter, (unsigned long long)PROGRESS_BATCH_B);
        }
        __syncwarp();
    }
    if (!a.det && lane == 0 && done % PROGRESS_BATCH_B) atomicAdd(a.counter, (unsigned long long)(done % PROGRESS_BATCH_B));
}

template <typename VT, int LOSS, int GT, bool REP> static void *pick_bgr(int B)
{
    switch (B) {
    case 1: return (void *)sps_group_batch_kernel<VT, LOSS, 1, GT, REP>;
    case 2: return (void *)sps_group_batch_kernel<VT, LOSS, 2, GT, REP>;
    case 4: return (void *)sps_group_batch_kernel<VT, LOSS, 4, GT, REP>;
    case 8: return (void *)sps_group_batch_kernel<VT, LOSS, 8, GT, REP>;
    default: return (void *)sps_group_batch_kernel<VT, LOSS, 16, GT, REP>;
    }
}
template <typename VT, int LOSS, int GT> static void *pick_bg(int B, bool rep)
{
    return rep ? pick_bgr<VT, LOSS, GT, true>(B) : pick_bgr<VT, LOSS, GT, false>(B);
}
// G = 10 (BASELINE config 5) specialised, other G <= 16 at runtime
template <typename VT, int LOSS> static void *pick_b(int B, int G, bool rep)
{
    return G == 10 ? pick_bg<VT, LOSS, 10>(B, rep) : pick_bg<VT, LOSS, 0>(B, rep);
}

__global__ void k_batch_field(const double *state, int64_t p, const BLay L, int beta, int field, double *out, int set)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = j / L.G;
        double *s = const_cast<double *>(state) + bidx(b, (int)(j - b * L.G), beta, field, L);
        if (set) *s = out[j];
        else out[j] = *s;
    }
}

// fold the replicated x deltas of the hot blocks into the state (after a launch)
__global__ void k_batch_fold(double *state, double *xrep, int nrep, int nrb, int hshift, const BLay L, int B,
                             int64_t p, int64_t rstride)
{
    const int G = L.G;
    const int64_t m = (int64_t)nrb * G * B;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int beta = (int)(t % B);
        const int64_t rq = t / B;
        const int q = (int)(rq % G), rank = (int)(rq / G);
        double sum = 0.0;
        for (int rr = 0; rr < nrep; rr++) {
            double *r = xrep + ((int64_t)rr * nrb + rank) * rstride + q * B + beta;
            sum += *r;
            *r = 0.0;
        }
        const int64_t b = (int64_t)rank << hshift;
        if (b * G + q < p) state[bidx(b, q, beta, 0, L)] += sum;
    }
}

}  // namespace ps

using namespace ps;

static BLay batch_layout(int64_t p, int G, int B, int hshift)
{
    BLay L{};
    L.G = G;
    L.S = B < BATCH_S ? B : BATCH_S;
    L.body = ((p + G - 1) / G) * G * L.S * 2;
    L.hstride = (std::max<int64_t>(g_hstride, 2 * L.S) + 1) & ~1ll;  // even: bit 0 of a shuffled offset is a flag
    L.nhot = g_hstride > 0 ? (g_nhot >= 0 ? g_nhot : (B >= 8 ? 128 : 32)) : 0;
    L.hshift = std::max(0, std::min(hshift, 30));
    const int hab = g_hab >= 0 ? g_hab : (B >= 4 ? 64 : 0);
    L.hab = (hab > 0 && L.hstride >= hab + L.S) ? hab : 0;
    L.region = L.body + (int64_t)L.nhot * G * L.hstride + g_rpad;
    return L;
}

extern "C" int ps_batch_run_rep(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm,
                                const double *lam2, int32_t B, double *state, double *alpha, const ps_sched_t *sched,
                                double *xrep, int32_t nrep, int32_t nrb, void *stream)
{
    NvtxRange nvtx_range("K2b ps_batch_run");
    if (!csr || !part || !prm || !lam2 || !state || !alpha || !sched) return ps_fail(PS_EINVAL, "null argument");
    if (B != 1 && B != 2 && B != 4 && B != 8 && B != 16) return ps_fail(PS_EINVAL, "B must be 1, 2, 4, 8 or 16");
    if (part->kind != PS_PART_CONTIG || part->G < 1 || part->G > 16 || !part->blk_weight)
        return ps_fail(PS_EINVAL, "batched path: contiguous blocks of G <= 16 with ps_prepare weights");
    if (part->max_row_nnz > 32) return ps_fail(PS_EINVAL, "batched path: rows of <= 32 nonzeros");
    if (csr->row_ptr_type != PS_I32) return ps_fail(PS_EINVAL, "batched path: int32 row pointers");
    if (prm->penalty != PS_PEN_GROUP) return ps_fail(PS_EINVAL, "batched path: group penalty");
    if (!(prm->gamma > 0)) return ps_fail(PS_EINVAL, "gamma must be positive");
    if (sched->count < 0) return ps_fail(PS_EINVAL, "negative update count");
    if (sched->count == 0) return PS_OK;
    const bool det = sched->samples != nullptr;
    if (!det && !sched->counter) return ps_fail(PS_EINVAL, "async mode needs a device counter");
    BArgs a{};
    a.row_ptr = static_cast<const int32_t *>(csr->row_ptr);
    a.col = csr->col_idx;
    a.val = csr->values;
    a.y = csr->labels;
    a.n = csr->n_rows;
    a.p = csr->n_cols;
    a.G = part->G;
    a.bd = part->blk_weight;
    a.state = state;
    a.alpha = alpha;
    a.lam2 = lam2;
    a.loss = prm->loss;
    a.lambda1 = prm->lambda1;
    a.gamma = prm->gamma;
    a.n_d = (double)csr->n_rows;
    a.nb = (csr->n_cols + part->G - 1) / part->G;
    a.samples = sched->samples;
    a.count = sched->count;
    {  // splitmix64(seed), host side (as ps_run)
        uint64_t z = sched->seed + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        a.seed = z ^ (z >> 31);
    }
    a.slot_base = sched->slot_base;
    a.counter = sched->counter;
    a.det = det ? 1 : 0;
    a.skip_zero = (sched->flags & PS_FLAG_GROUP_STORE_ZEROS) ? 0 : 1;
    a.xrep = xrep;
    a.nrep = (!det && xrep && nrep > 0 && nrb > 0) ? nrep : 0;
    a.nrb = nrb;
    a.hshift = std::max(0, (int)sched->hot_shift);
    a.rpad = g_rpad;
    a.L = batch_layout(csr->n_cols, part->G, B, a.hshift);
    a.hshare = g_hshare;
    a.rstride = std::max<int64_t>(g_rstride, (int64_t)part->G * B);
    void *kern;
    const bool f64 = csr->value_type == PS_F64, sq = prm->loss == PS_LOSS_SQUARED;
    const int G = part->G;
    const bool rep = a.nrep > 0;
    if (f64) kern = sq ? pick_b<double, PS_LOSS_SQUARED>(B, G, rep) : pick_b<double, PS_LOSS_LOGISTIC>(B, G, rep);
    else kern = sq ? pick_b<float, PS_LOSS_SQUARED>(B, G, rep) : pick_b<float, PS_LOSS_LOGISTIC>(B, G, rep);
    const int wpc = sched->warps_per_cta > 0 ? std::min(sched->warps_per_cta, BATCH_T / 32) : BATCH_T / 32;
    const size_t smem = ((size_t)wpc * BATCH_SM_WARP + BATCH_SM_SHARE) * 8;
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                             "ps_batch_run smem attribute");
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wpc * 32, smem), "ps_batch_run occupancy");
    // default grid: one full wave, but no more than n/16 rows in flight (as ps_run)
    const int64_t cap = std::max<int64_t>(1, csr->n_rows / (16 * (int64_t)wpc));
    const int ctas = det ? 1 : (sched->ctas > 0 ? sched->ctas
                                                : (int)std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), cap));
    // per-coordinate step damping as ps_run: tau = rows in flight (every state sees all of them)
    const double tau = (double)ctas * wpc;
    a.kappa = (!det && sched->contention > 0) ? sched->contention / tau : INFINITY;
    void *args[] = {(void *)&a};
    CK(cudaLaunchKernel(kern, dim3(ctas), dim3(wpc * 32), args, smem, (cudaStream_t)stream), "ps_batch_run launch");
    g_last_ctas = ctas;
    g_last_wpc = wpc;
    if (a.nrep > 0) {
        const int64_t m = (int64_t)nrb * G * B;
        k_batch_fold<<<(int)std::min<int64_t>((m + 255) / 256, 1024), 256, 0, (cudaStream_t)stream>>>(
            state, xrep, a.nrep, nrb, a.hshift, a.L, B, a.p, a.rstride);
        CK(cudaGetLastError(), "ps_batch_run fold");
    }
    return PS_OK;
}

extern "C" int ps_batch_run(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *lam2,
                            int32_t B, double *state, double *alpha, const ps_sched_t *sched, void *stream)
{
    return ps_batch_run_rep(csr, part, prm, lam2, B, state, alpha, sched, nullptr, 0, 0, stream);
}

extern "C" int ps_batch_field(double *state, int64_t p, int32_t G, int32_t B, int32_t hot_shift, int32_t beta,
                              int32_t field, double *vec, int32_t set, void *stream)
{
    if (!state || !vec || beta < 0 || beta >= B || field < 0 || field > 1 || G < 1) return ps_fail(PS_EINVAL, "bad argument");
    if (p <= 0) return PS_OK;
    k_batch_field<<<(int)std::min<int64_t>((p + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(
        state, p, batch_layout(p, G, B, hot_shift), beta, field, vec, set);
    CK(cudaGetLastError(), "ps_batch_field launch");
    return PS_OK;
}

extern "C" int ps_batch_tune(int64_t rpad, int64_t rstride)
{
    if (rpad < 0 || rstride < 0) return ps_fail(PS_EINVAL, "bad argument");
    g_rpad = rpad;
    g_rstride = rstride;
    return PS_OK;
}

extern "C" int ps_batch_last_grid(int32_t *ctas, int32_t *warps_per_cta)
{
    if (!ctas || !warps_per_cta) return ps_fail(PS_EINVAL, "null argument");
    *ctas = g_last_ctas;
    *warps_per_cta = g_last_wpc;
    return PS_OK;
}

extern "C" int ps_batch_tune2(int32_t nhot, int64_t hstride, int32_t hshare, int32_t hab)
{
    if (nhot < -1 || hstride < 0 || hshare < 0 || hab < -1) return ps_fail(PS_EINVAL, "bad argument");
    g_hab = hab;
    g_nhot = nhot;
    g_hstride = hstride;
    g_hshare = hshare;
    return PS_OK;
}

extern "C" int64_t ps_batch_state_doubles(int64_t p, int32_t G, int32_t B)
{
    if (p < 0 || G < 1 || B < 1) return -1;
    const BLay L = batch_layout(p, G, B, 0);
    return (int64_t)(B / L.S) * L.region;
}

extern "C" int64_t ps_batch_rep_doubles(int32_t nrep, int32_t nrb, int32_t G, int32_t B)
{
    if (nrep < 0 || nrb < 0 || G < 1 || B < 1) return -1;
    return (int64_t)nrep * nrb * std::max<int64_t>(g_rstride, (int64_t)G * B);
}
