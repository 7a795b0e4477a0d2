// sps_lane_kernel -- the asynchronous singleton path with ONE THREAD PER
// IN-FLIGHT SAMPLE (configs 2-4, rows of <= KMAX nonzeros).
//
// The warp-per-sample kernels (fast2.cuh) spend ~400 warp-instructions per
// update and are bound by each warp's dependent latency chain (row -> gather
// -> butterfly -> logistic -> prox -> shared CAS, ~4.7k cycles) with at most
// 32 warps, i.e. 32 samples, in flight per SM (64 registers per thread at 1024
// threads).  Here each lane owns a whole sample: the row's columns, values and
// (x^, abar) stay in the lane's registers, the margin is a private fp64 sum
// (no shuffles), the loss derivative is computed once per sample instead of
// once per lane, and one warp instruction advances 32 samples.  Low occupancy
// (128-256 threads per SM, ~200 registers each) keeps the number of samples
// in flight -- the staleness tau of the asynchronous analysis -- in the same
// range as the warp kernel's while the instruction count per update drops by
// an order of magnitude.
//
// Per sample (asynchronous.py:80-117, one inconsistent read of x^ per
// coordinate, reused by the margin and the prox):
//   1. row i (sampler), its columns / values / label; alpha_i read;
//   2. (x^, abar) of every nonzero: staged columns from the CTA snapshot,
//      others one 16-B L2 load of the coordinate record; margin = sum val x^;
//   3. l'(margin) (fastmath.cuh deriv2), alpha_i <-> new (exchange issued now,
//      its value needed only by the abar credit at the end);
//   4. per nonzero, D (read-only, L1-cacheable), the contention-scaled step,
//      the prox, and the commit: cold -> RED (or a zero store), staged -> the
//      CTA's pending accumulators (fast2.cuh semantics: zero stores, deferred
//      zero flags, dirty words), the lanes of a warp that hit the same staged
//      slot at the same position combined first (__match_any_sync + a
//      segmented tree) so one lane per slot CASes;
//   5. abar += ((new - replaced) / n) val on the row, the same way.
// Staging layout and flush are sps_hot_kernel's (one pending copy,
// hot_flush2); each warp flushes after every `period` rounds of 32 samples.
#pragma once

#include "fast2.cuh"

namespace ps {

// combine v over the lanes that share `key` (participating lanes pass part =
// true; every lane of the warp must call this); returns the group sum on the
// group's lowest lane (its `leader` flag set), 0 elsewhere
__device__ __forceinline__ double seg_sum(bool part, unsigned key, double v, int lane, bool &leader)
{
    const unsigned k = part ? key : (0x80000000u | (unsigned)lane);
    const unsigned peers = __match_any_sync(FULL, k);
    const int gsz = __popc(peers);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    double s = part ? v : 0.0;
    if (__any_sync(FULL, gsz > 1)) {
        for (int off = 1; off < 32; off <<= 1) {
            if (!__any_sync(FULL, off < gsz)) break;
            const int pr = rank + off;
            const int src = pr < gsz ? (int)__fns(peers, 0u, pr + 1) : lane;
            const double o = __shfl_sync(FULL, s, src);
            if ((rank & (2 * off - 1)) == 0 && pr < gsz) s += o;
        }
    }
    leader = part && rank == 0;
    return s;
}

template <typename VT, typename PT, int LOSS, int PEN, bool LITERAL, int KMAX>
__global__ void __launch_bounds__(256, 1) sps_lane_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    __shared__ unsigned cta_prog;
    if (threadIdx.x == 0) cta_prog = 0u;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int H = a.H;
    double2 *const snap = reinterpret_cast<double2 *>(smem_dyn);
    double *const sd = smem_dyn + 2 * H;
    double *const pend = smem_dyn + 3 * H;
    unsigned *const zf = reinterpret_cast<unsigned *>(pend + 2 * H);
    const unsigned a_snap = (unsigned)__cvta_generic_to_shared(smem_dyn);
    const unsigned a_d = a_snap + 16u * H, a_zf = a_snap + 40u * H;
    const unsigned d_px = 3u * H, d_pab = 4u * H;
    const unsigned a_dirty = a_snap + hot2_dirty_off(H, 1);
    double *const coord = a.coord;
    if (H > 0) {
        for (int s = threadIdx.x; s < H; s += blockDim.x) {
            double x, ab, d;
            ld_record(coord + 4 * ((int64_t)s << a.hot_shift), x, ab, d);
            snap[s] = make_double2(x, ab);
            sd[s] = d;
            pend[s] = 0.0;
            pend[H + s] = 0.0;
            zf[s] = 0u;
        }
        if (threadIdx.x == 0) zf[H] = 0u;
        for (int b = threadIdx.x; b < 1024; b += blockDim.x)
            reinterpret_cast<unsigned *>(reinterpret_cast<unsigned char *>(smem_dyn) + hot2_dirty_off(H, 1))[b] = 0u;
    }
    __syncthreads();
    double *const alpha = a.alpha;
    const double gamma = a.gamma, lambda1 = a.lambda1, kappa = a.kappa, lam2 = a.lam2;
    const double plo = a.lo, phi = a.hi;
    const int pen = a.pen;
    const int shift = a.hot_shift;
    const unsigned hmask = (1u << shift) - 1u, hlim = (unsigned)H << shift;
    const uint64_t seed = a.seed, nrows = (uint64_t)a.n;
    const double inv_n = 1.0 / a.n_d;
    // static split of the call's slots over the THREADS (split_iterations)
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t q = a.count / nthr, rr = a.count % nthr;
    const uint64_t first = a.slot_base + (uint64_t)(gt * q + min(gt, rr));
    const unsigned todo = (unsigned)(q + (gt < rr ? 1 : 0));
    const unsigned rounds = (unsigned)(q + (rr > 0 ? 1 : 0));  // warp-uniform loop count
    int until_flush = H > 0 ? 1 + (wib * a.period) / max(1, nwib) : 0;
    const int32_t *const colp = a.col;
    const VT *const valp = reinterpret_cast<const VT *>(a.val);
    const VT *const yp = reinterpret_cast<const VT *>(a.y);
    const PT *const rowp = reinterpret_cast<const PT *>(a.row_ptr);

    for (unsigned t = 0; t < rounds; t++) {
        const bool act = t < todo;
        // ---- 1. the row
        int64_t i = 0;
        PT lo = PT(0);
        int k = 0;
        double yb = 0.0, old = 0.0;
        if (act) {
            i = sample_row(seed, first + t, nrows);
            lo = __ldg(rowp + i);
            k = (int)(__ldg(rowp + i + 1) - lo);
            yb = widen(__ldg(yp + i));
            old = ld_cg(alpha + i);
        }
        int col[KMAX];
        VT val[KMAX];
#pragma unroll
        for (int e = 0; e < KMAX; e++) {
            col[e] = -1;
            val[e] = VT(0);
            if (e < k) {
                const size_t o = sizeof(PT) == 4 ? (size_t)(unsigned)(lo + e) : (size_t)(lo + e);
                col[e] = __ldg(colp + o);
                val[e] = __ldg(valp + o);
            }
        }
        // ---- 2. (x^, abar) and the margin
        double xh[KMAX], ab[KMAX];
#pragma unroll
        for (int e = 0; e < KMAX; e++) {
            const bool hot = (unsigned)col[e] < hlim && ((unsigned)col[e] & hmask) == 0u;
            xh[e] = ab[e] = 0.0;
            if (hot) {
                const double2 v = sh_ld2(a_snap + 16u * ((unsigned)col[e] >> shift));
                xh[e] = v.x;
                ab[e] = v.y;
            } else if (col[e] >= 0) {
                const double2 v = ld_cg2(coord + 4 * (int64_t)col[e]);
                xh[e] = v.x;
                ab[e] = v.y;
            }
        }
        double margin = 0.0;
#pragma unroll
        for (int e = 0; e < KMAX; e++) margin = __fma_rn(widen(val[e]), xh[e], margin);
        // ---- 3. derivative, alpha exchange
        const double nw = act ? deriv2<LOSS>(margin, yb) : 0.0;
        const double ds = nw - old;
        double rep = 0.0;
        if (act) rep = atomic_exch(alpha + i, nw);
        // ---- 4. D, step, prox, commit (nonzero e of every lane's row together)
#pragma unroll
        for (int e = 0; e < KMAX; e++) {
            const bool ok = col[e] >= 0;
            const bool hot = (unsigned)col[e] < hlim && ((unsigned)col[e] & hmask) == 0u;
            const unsigned sl = (unsigned)col[e] >> shift;
            double d = 0.0;
            if (hot) d = sh_ld(a_d + 8u * sl);
            else if (ok) d = __ldg(coord + 4 * (int64_t)col[e] + 2);
            const double cval = widen(val[e]);
            const double v = __fma_rn(ds, cval, d * __fma_rn(lambda1, xh[e], ab[e]));
            const double kd = kappa * d;
            const double g = gamma * (kd < 1.0 ? kd : 1.0);
            const double z = prox2<PEN>(__fma_rn(-g, v, xh[e]), g * d, lam2, pen, plo, phi);
            const bool z0 = !LITERAL && ok && z == 0.0;
            const bool defer = z0 && hot && xh[e] == 0.0;
            double *const gx = coord + 4 * (int64_t)col[e];
            if (ok && !hot && !z0) red_add(gx, z - xh[e]);
            if (z0 && !defer) atomic_exch(gx, 0.0);
            if (z0 && hot) {  // the coordinate is stored: drop the CTA's pending x delta of it
                const unsigned ap = a_snap + 8u * (d_px + sl);
                if (sh_ld(ap) != 0.0) sh_zero64(ap);
            }
            if (defer) sh_st32(a_zf + 4u * sl, 1u);
            if (z0 && hot) sh_st32(a_dirty + 4u * sl, 1u);
            // staged deltas of the lanes sharing a slot, combined; one CAS per slot
            if (__any_sync(FULL, hot && !z0 && ok)) {
                bool lead;
                const double sdx = seg_sum(hot && !z0 && ok, sl, z - xh[e], lane, lead);
                if (lead) {
                    sh_add(d_px + sl, sdx);
                    sh_st32(a_dirty + 4u * sl, 1u);
                }
            }
        }
        // ---- 5. abar credit ((new - replaced)/n) a_i
        const double tq = (nw - rep) * inv_n;
#pragma unroll
        for (int e = 0; e < KMAX; e++) {
            const bool ok = col[e] >= 0;
            const bool hot = (unsigned)col[e] < hlim && ((unsigned)col[e] & hmask) == 0u;
            const unsigned sl = (unsigned)col[e] >> shift;
            const double inc = tq * widen(val[e]);
            if (ok && !hot) red_add(coord + 4 * (int64_t)col[e] + 1, inc);
            if (__any_sync(FULL, hot && ok)) {
                bool lead;
                const double sab = seg_sum(hot && ok, sl, inc, lane, lead);
                if (lead) {
                    sh_add(d_pab + sl, sab);
                    sh_st32(a_dirty + 4u * sl, 1u);
                }
            }
        }
        __syncwarp();
        if (H > 0 && --until_flush == 0) {
            hot_flush2(coord, H, 1, shift, 0u, lane, true);
            until_flush = a.period;
        }
        // progress: a warp's 32 samples of the round into the CTA count, every
        // CTA_PROGRESS of the CTA into the global counter (asynchronous.py:155-162)
        const unsigned nact = (unsigned)__popc(__ballot_sync(FULL, act));
        if (lane == 0 && nact) {
            const unsigned o = atomicAdd(&cta_prog, nact);
            if ((o + nact) / CTA_PROGRESS != o / CTA_PROGRESS)
                atomicAdd(a.counter, (unsigned long long)(((o + nact) / CTA_PROGRESS - o / CTA_PROGRESS) * CTA_PROGRESS));
        }
    }
    __syncthreads();  // every warp's CTA progress is in
    if (threadIdx.x == 0 && cta_prog % CTA_PROGRESS) atomicAdd(a.counter, (unsigned long long)(cta_prog % CTA_PROGRESS));
    if (H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            for (int b = lane; b < 1024; b += 32)
                reinterpret_cast<unsigned *>(reinterpret_cast<unsigned char *>(smem_dyn) + hot2_dirty_off(H, 1))[b] = b < H;
            __syncwarp();
            hot_flush2(coord, H, 1, shift, 0u, lane, false);
        }
    }
}

}  // namespace ps
