// sps_hot_kernel -- the asynchronous hot path, second generation (configs 2-4).
//
// Same algorithm and semantics as sps_fast_kernel (one warp per in-flight
// sample, inconsistent reads, the worker_iteration of asynchronous.py:80-117
// with the contention-scaled steps and zero commits of DESIGN.md, hot columns
// staged per CTA, CTA pairs sharing the snapshot refresh), rebuilt for the
// instruction budget: round 1's kernel issued ~400 warp-instructions per
// update at 66% issue-active (profiles/ncu_sps_r01.md).  What changed:
//   * no dirty bitmasks: the flush scans its CTA's staged slots (16 per lane)
//     instead of every hot commit marking a bit with a shared atomicOr;
//   * one pending copy; a zero store of a staged column is a plain 32-bit
//     flag store (the flush exchanges the flags);
//   * commits are straight-line predicated code (one CAS loop, for a staged
//     column's pending delta, is the only divergent part);
//   * a cold coordinate's record (x, abar, D) is one 256-bit L2 load;
//   * the row extent, label and sample of the next 32 updates are read once
//     per 32 updates (one per lane) and handed out by 32-bit shuffles;
//   * the logistic derivative: exp by a 64-entry table of 2^(j/64) (constant
//     bank, warp-uniform index) and a degree-5 polynomial, one Newton step
//     for the reciprocal; FMAs allowed (the asynchronous kernels are checked
//     against the oracle on the objective; the deterministic replay keeps the
//     reference's operation order without contraction).
// Restricted to SINGLETON rows of <= 32 nonzeros and 32-warp CTAs; everything
// else keeps the round-1 kernels.
#pragma once

#include "fastmath.cuh"

namespace ps {

// explicit 32-bit shared-memory accesses (one address register, no generic
// pointer arithmetic in the update loop)
__device__ __forceinline__ double sh_ld(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ double2 sh_ld2(unsigned a)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sh_st32(unsigned a, unsigned v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sh_st8(unsigned a, unsigned v)
{
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sh_zero64(unsigned a)
{
    asm volatile("{\n\t.reg .b64 t;\n\tatom.shared.exch.b64 t, [%0], 0;\n\t}" ::"r"(a) : "memory");
}
// fp64 add into the staging area (double index d): the compiler's shared
// fp64 atomicAdd (an ATOMS.CAST.SPIN loop; no native fp64 shared atomic on sm_100)
__device__ __forceinline__ void sh_add(unsigned d, double v)
{
    extern __shared__ double smem_dyn[];
    atomicAdd(smem_dyn + d, v);
}

// staging area of sps_hot_kernel (dynamic shared memory, doubles):
//   [0, 2H)  snapshot (x, abar) pairs    [2H, 3H) D
//   [3H + 2cH, 4H + 2cH) pending x deltas, [4H + 2cH, 5H + 2cH) pending abar
//   deltas of copy c < NC (warp w adds into copy w % NC: fewer CAS retries on
//   the hottest slots), then H 32-bit zero-store flags and the rotation word
//   then (16-B aligned) 1024 dirty words, word s = slot s has something
//   pending (set with plain 32-bit stores after the pending update; natural
//   order keeps the hottest slots in different banks); the flush reads them
//   four per lane per 512-B row
__host__ __device__ constexpr unsigned hot2_dirty_off(int H, int nc)
{
    return (8u * (3u + 2u * (unsigned)nc) * (unsigned)H + 4u * ((unsigned)H + 2u) + 15u) & ~15u;
}
__host__ __device__ constexpr int hot2_doubles(int H, int nc) { return (int)((hot2_dirty_off(H, nc) + 4096u + 15u) & ~15u) / 8; }
constexpr int HOT2_BATCH_BYTES = 0;

__device__ __noinline__ void hot_flush2(double *coord, const int H, const int nc, const int shift, const unsigned lead,
                                        const int lane, const bool refresh)
{
    extern __shared__ double smem_dyn[];
    double *const pend = smem_dyn + 3 * H;
    unsigned *zf = reinterpret_cast<unsigned *>(pend + 2 * nc * H);
    const unsigned a_dirty = (unsigned)__cvta_generic_to_shared(smem_dyn) + hot2_dirty_off(H, nc);
    // lane l flushes slots 128 r + 4 l .. + 3 of each 128-slot row r (one
    // conflict-free 512-B read of dirty words per row)
    for (int r0 = 0; r0 < H; r0 += 128) {
        uint4 w;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(a_dirty + 4u * (unsigned)(r0 + 4 * lane)) : "memory");
        const unsigned ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (!ww[j]) continue;
            const int s = r0 + 4 * lane + j;
            sh_st32(a_dirty + 4u * (unsigned)s, 0u);  // cleared before the pending values are taken
            double dx = 0.0, dab = 0.0;
            for (int c = 0; c < nc; c++) {
                dx += smem_take(pend + 2 * c * H + s);
                dab += smem_take(pend + (2 * c + 1) * H + s);
            }
            double *g = coord + 4 * ((int64_t)s << shift);
            if (atomicExch(zf + s, 0u)) atomic_exch(g, 0.0);  // deferred zero store, then the deltas added since
            if (dx != 0.0) red_add(g, dx);
            if (dab != 0.0) red_add(g + 1, dab);
        }
    }
    const int kmax = (H + 31) >> 5;
    if (!refresh) return;
    // tiered refresh: the HOT_TIER0 hottest slots every flush, the others a
    // rotating quarter per flush
    unsigned rot = 0;
    if (lane == 0) rot = atomicAdd(zf + H, 1u);
    rot = __shfl_sync(FULL, rot, 0) & 3u;
    if (lead) {  // cluster member: from the leader CTA's snapshot (distributed shared memory)
        for (int k = 0; k < kmax; k++) {
            const int s = lane + 32 * k;
            if (s < H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
                double2 v;
                asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(lead + 16u * s));
                reinterpret_cast<double2 *>(smem_dyn)[s] = v;
            }
        }
        return;
    }
    for (int k = 0; k < kmax; k++) {
        const int s = lane + 32 * k;
        if (s < H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dyn + 2 * s);
            const double *src = coord + 4 * ((int64_t)s << shift);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// LITERAL: commit prox-zeroed coordinates as the delta -x_hat (PS_FLAG_DELTA_ZERO)
template <typename VT, typename PT, int LOSS, int PEN, bool LITERAL, int NC>
__global__ void __launch_bounds__(1024, 1) sps_hot_kernel(const KArgs a)
{
    extern __shared__ double smem_dyn[];
    __shared__ unsigned cta_prog;  // this CTA's updates reported so far
    if (threadIdx.x == 0) cta_prog = 0u;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    const int H = a.H;
    double2 *const snap = reinterpret_cast<double2 *>(smem_dyn);
    double *const sd = smem_dyn + 2 * H;
    const int nc = a.ncopy;
    const bool diag_nohot = (a.diag & (1 << 26)) != 0;  // measurement only: staged deltas are dropped
    const bool local_view = (a.diag & PS_FLAG_LOCAL_VIEW) != 0;  // opt-in: a staged commit also updates the CTA snapshot
    double *const pend = smem_dyn + 3 * H;
    unsigned *const zf = reinterpret_cast<unsigned *>(pend + 2 * nc * H);
    // 32-bit shared addresses of the staging arrays; this warp's pending copy
    const unsigned a_snap = (unsigned)__cvta_generic_to_shared(smem_dyn);
    const unsigned a_d = a_snap + 16u * H, a_zf = a_snap + 8u * (3 + 2 * nc) * H;
    const unsigned d_px = (unsigned)(3 + 2 * (wib % nc)) * H, d_pab = d_px + H;  // double indices
    const unsigned a_dirty = a_snap + hot2_dirty_off(H, nc);
    double *const coord = a.coord;
    if (H > 0) {
        for (int s = threadIdx.x; s < H; s += blockDim.x) {
            double x, ab, d;
            ld_record(coord + 4 * ((int64_t)s << a.hot_shift), x, ab, d);
            snap[s] = make_double2(x, ab);
            sd[s] = d;
            for (int c = 0; c < 2 * nc; c++) pend[c * H + s] = 0.0;
            zf[s] = 0u;
        }
        if (threadIdx.x == 0) zf[H] = 0u;
        for (int b = threadIdx.x; b < 1024; b += blockDim.x)
            reinterpret_cast<unsigned *>(reinterpret_cast<unsigned char *>(smem_dyn) + hot2_dirty_off(H, nc))[b] = 0u;
    }
    __syncthreads();
    unsigned lead = 0u;
    if (a.cluster > 1) {
        unsigned rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        if (rank != 0 && H > 0) {
            const unsigned mine = (unsigned)__cvta_generic_to_shared(smem_dyn);
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(mine));
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    double *const alpha = a.alpha;
    const double gamma = a.gamma, lambda1 = a.lambda1, kappa = a.kappa, lam2 = a.lam2;
    const double plo = a.lo, phi = a.hi;
    const int pen = a.pen;
    const int shift = a.hot_shift;
    const unsigned hmask = (1u << shift) - 1u, hlim = (unsigned)H << shift;
    const uint64_t seed = a.seed, nrows = (uint64_t)a.n;
    const double inv_n = 1.0 / a.n_d;
    const int64_t nwarps = (int64_t)gridDim.x * nwib;
    const int64_t q = a.count / nwarps, rr = a.count % nwarps;
    const uint64_t first = a.slot_base + (uint64_t)(gw * q + min(gw, rr));
    const unsigned todo = (unsigned)(q + (gw < rr ? 1 : 0));
    int until_flush = H > 0 ? 1 + (wib * a.period) / max(1, nwib) : 0;
    const int32_t *const colp = a.col;
    const VT *const valp = reinterpret_cast<const VT *>(a.val);
    const VT *const yp = reinterpret_cast<const VT *>(a.y);
    const PT *const rowp = reinterpret_cast<const PT *>(a.row_ptr);

    if (todo > 0) {
        // samples, row extents and labels of 32 updates at a time: lane L holds
        // update t0 + L of the batch (k = -1 past the warp's last update)
        auto load_batch = [&](unsigned t0, unsigned &bi_, PT &blo_, int &bk_, VT &by_) {
            const unsigned t = t0 + (unsigned)lane;
            bi_ = 0u;
            blo_ = PT(0);
            bk_ = -1;
            by_ = VT(0);
            if (t < todo) {
                const int64_t i = sample_row(seed, first + t, nrows);
                bi_ = (unsigned)i;
                blo_ = __ldg(rowp + i);
                bk_ = (int)(__ldg(rowp + i + 1) - blo_);
                by_ = __ldg(yp + i);
            }
        };
        unsigned bi, ni;
        PT blo, nlo;
        int bk, nk;
        VT by, ny;
        load_batch(0u, bi, blo, bk, by);
        load_batch(32u, ni, nlo, nk, ny);
        // the current update's row: lane L holds nonzeros L, L + 32, ... (NC per
        // lane, col = -1 past the row), the sample and the label
        int col[NC];
        VT val[NC];
        unsigned ci = __shfl_sync(FULL, bi, 0);
        VT cy = __shfl_sync(FULL, by, 0);
        {
            const PT lo0 = __shfl_sync(FULL, blo, 0);
            const int k0 = __shfl_sync(FULL, bk, 0);
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int e = lane + 32 * c;
                col[c] = -1;
                val[c] = VT(0);
                if (e < k0) {
                    const size_t o = sizeof(PT) == 4 ? (size_t)(unsigned)(lo0 + e) : (size_t)(lo0 + e);
                    col[c] = __ldg(colp + o);
                    val[c] = __ldg(valp + o);
                }
            }
        }
        // deferred abar credit of the previous update
        int pcol[NC];  // >= 0: cold column; <= -2: staged slot -2 - pcol; -1: none
        double pval[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            pcol[c] = -1;
            pval[c] = 0.0;
        }
        double pnw = 0.0, prep = 0.0;
        unsigned t = 0u;
        while (true) {
            // ---- state reads: staged columns from the CTA snapshot, others one
            // 256-bit L2 read of the record
            double xh[NC], ab[NC], d[NC];
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const bool hot = (unsigned)col[c] < hlim && ((unsigned)col[c] & hmask) == 0u;
                const unsigned sl = (unsigned)col[c] >> shift;
                xh[c] = ab[c] = d[c] = 0.0;
                if (hot) {
                    const double2 v = sh_ld2(a_snap + 16u * sl);
                    xh[c] = v.x;
                    ab[c] = v.y;
                    d[c] = sh_ld(a_d + 8u * sl);
                } else if (col[c] >= 0) {
                    ld_record(coord + 4 * (int64_t)col[c], xh[c], ab[c], d[c]);
                }
            }
            double old = 0.0;
            if (lane == 0) old = ld_cg(alpha + ci);
            // ---- abar credit of the previous update (its alpha exchange has returned)
            {
                const double tq = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const double inc = tq * pval[c];
                    if (pcol[c] <= -2) {
                        if (!diag_nohot) sh_add(d_pab + (unsigned)(-2 - pcol[c]), inc);
                        sh_st32(a_dirty + 4u * (unsigned)(-2 - pcol[c]), 1u);
                    } else if (pcol[c] >= 0) {
                        red_add(coord + 4 * (int64_t)pcol[c] + 1, inc);
                    }
                }
            }
            // ---- the next update's row (extent from the batch registers)
            t++;
            if ((t & 31u) == 0u) {
                bi = ni;
                blo = nlo;
                bk = nk;
                by = ny;
                load_batch(t + 32u, ni, nlo, nk, ny);
            }
            const int src = (int)(t & 31u);
            const unsigned nci = __shfl_sync(FULL, bi, src);
            const VT ncy = __shfl_sync(FULL, by, src);
            int ncol[NC];
            VT nval[NC];
            {
                const PT lo1 = __shfl_sync(FULL, blo, src);
                const int k1 = __shfl_sync(FULL, bk, src);
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const int e = lane + 32 * c;
                    ncol[c] = -1;
                    nval[c] = VT(0);
                    if (e < k1) {
                        const size_t o = sizeof(PT) == 4 ? (size_t)(unsigned)(lo1 + e) : (size_t)(lo1 + e);
                        ncol[c] = __ldg(colp + o);
                        nval[c] = __ldg(valp + o);
                    }
                }
            }
            // ---- margin -> derivative
            double part = 0.0;
#pragma unroll
            for (int c = 0; c < NC; c++) part = __fma_rn(widen(val[c]), xh[c], part);
            const double margin = warp_sum(part);
            old = __shfl_sync(FULL, old, 0);
            const double nw = deriv2<LOSS>(margin, widen(cy));
            const double ds = nw - old;
            // ---- v, step, prox, commit (asynchronous.py:97-107)
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const double cval = widen(val[c]);
                const double v = __fma_rn(ds, cval, d[c] * __fma_rn(lambda1, xh[c], ab[c]));
                const double kd = kappa * d[c];
                const double g = gamma * (kd < 1.0 ? kd : 1.0);
                const double z = prox2<PEN>(__fma_rn(-g, v, xh[c]), g * d[c], lam2, pen, plo, phi);
                // commit, straight-line: a zero is stored, not added as the delta
                // -x_hat; a staged column already read as
                // 0 is stored by the CTA's next flush (flag), its pending delta dropped
                const bool hot = (unsigned)col[c] < hlim && ((unsigned)col[c] & hmask) == 0u;
                const unsigned sl = (unsigned)col[c] >> shift;
                const bool act = col[c] >= 0;
                const bool z0 = !LITERAL && act && z == 0.0;
                const bool defer = z0 && hot && xh[c] == 0.0;
                double *const gx = coord + 4 * (int64_t)col[c];
                if (act && !hot && !z0) red_add(gx, z - xh[c]);
                if (z0 && !defer) atomic_exch(gx, 0.0);
                if (z0 && hot) {  // the coordinate is stored: drop the CTA's pending x deltas of it
                    for (int q = 0; q < nc; q++) {
                        const unsigned ap = a_snap + 8u * ((unsigned)(3 + 2 * q) * H + sl);
                        if (sh_ld(ap) != 0.0) sh_zero64(ap);
                    }
                }
                if (defer) sh_st32(a_zf + 4u * sl, 1u);
                if (hot && !z0 && !diag_nohot) sh_add(d_px + sl, z - xh[c]);
                if (hot) sh_st32(a_dirty + 4u * sl, 1u);  // after the pending add / zero flag (flush order)
                if (hot && local_view)  // the CTA reads its own commit at once (racy plain store; a refresh overwrites it)
                    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a_snap + 16u * sl), "d"(z) : "memory");
                pcol[c] = hot ? -2 - (int)sl : col[c];
                pval[c] = cval;
            }
            // ---- alpha_i <-> new (the abar credit is issued next iteration)
            double rep = 0.0;
            if (lane == 0) rep = atomic_exch(alpha + ci, nw);
            pnw = nw;
            prep = rep;
            if (H > 0 && --until_flush == 0) {
                hot_flush2(coord, H, nc, shift, lead, lane, true);
                until_flush = a.period;
            }
            // progress: PROGRESS_BATCH updates of a warp into the CTA count, every
            // CTA_PROGRESS of the CTA into the global counter (asynchronous.py:155-162)
            if (lane == 0 && (t % PROGRESS_BATCH) == 0u) {
                unsigned o;
                asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                             : "=r"(o)
                             : "r"((unsigned)__cvta_generic_to_shared(&cta_prog)), "r"((unsigned)PROGRESS_BATCH)
                             : "memory");
                if ((o + PROGRESS_BATCH) / CTA_PROGRESS != o / CTA_PROGRESS)
                    atomicAdd(a.counter, (unsigned long long)CTA_PROGRESS);
            }
            __syncwarp();
            if (t == todo) break;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                col[c] = ncol[c];
                val[c] = nval[c];
            }
            ci = nci;
            cy = ncy;
        }
        // last credit
        const double tq = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
#pragma unroll
        for (int c = 0; c < NC; c++) {
            if (pcol[c] <= -2) {
                sh_add(d_pab + (unsigned)(-2 - pcol[c]), tq * pval[c]);
                sh_st32(a_dirty + 4u * (unsigned)(-2 - pcol[c]), 1u);
            } else if (pcol[c] >= 0) {
                red_add(coord + 4 * (int64_t)pcol[c] + 1, tq * pval[c]);
            }
        }
    }
    if (lane == 0 && todo % PROGRESS_BATCH) atomicAdd(a.counter, (unsigned long long)(todo % PROGRESS_BATCH));
    __syncthreads();  // every warp's CTA progress is in
    if (threadIdx.x == 0 && cta_prog % CTA_PROGRESS) atomicAdd(a.counter, (unsigned long long)(cta_prog % CTA_PROGRESS));
    if (a.cluster > 1)  // the leader's staging area stays alive until every member stops reading it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            for (int b = lane; b < 1024; b += 32)
                reinterpret_cast<unsigned *>(reinterpret_cast<unsigned char *>(smem_dyn) + hot2_dirty_off(H, nc))[b] = b < H;
            __syncwarp();
            hot_flush2(coord, H, nc, shift, 0u, lane, false);
        }
    }
}

}  // namespace ps
