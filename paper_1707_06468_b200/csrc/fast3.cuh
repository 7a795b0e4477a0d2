// sps_hot3_kernel -- the asynchronous hot path, third generation (configs 2-4).
//
// Same algorithm and semantics as sps_hot_kernel (fast2.cuh): one warp per
// in-flight sample, inconsistent reads, the worker_iteration of
// asynchronous.py:80-117 with the contention-scaled steps and zero commits of
// DESIGN.md, hot columns staged per CTA (snapshot + pending deltas, one
// pending copy), CTA pairs sharing the snapshot refresh.  Rebuilt for the
// instruction count that ncu showed binding (profiles/ncu_sps_r02.md: 396
// warp-instructions per update at 67% issue-active, ~40 of them shared-address
// arithmetic rematerialised per use, 10 divergent regions, 50 in the flush):
//   * the staging capacity HM (512 or 1024 slots) is a template constant and
//     every staging array sits at a fixed offset from the dynamic shared base,
//     so a staged access is `base + slot * 8 + IMM` (the base is the .shared
//     symbol address, a link-time constant);
//   * the state gather is one predicated pair: snapshot (staged columns and the
//     row's padding lanes, which read slot 0 harmlessly) or one 256-bit L2 load;
//   * every commit except the staged CAS add is a single predicated
//     instruction (RED, exchange, plain shared store);
//   * the flush walks a per-lane bitmask of dirty slots (16 or 32 bits, built
//     from conflict-free 16-B reads of the dirty words) instead of testing
//     every slot in unrolled divergent blocks.
// Restricted to SINGLETON rows of <= 64 nonzeros and 32-warp CTAs.
#pragma once

#include "fastmath.cuh"

namespace ps {

// shared-memory layout of the hot3 staging area (bytes from the dynamic base)
template <int HM> struct Hot3 {
    static constexpr unsigned SNAP = 0;            // (x, abar) pairs, 16 B (cp.async target)
    static constexpr unsigned D = 16u * HM;        // D
    static constexpr unsigned PX = 24u * HM;       // pending x deltas
    static constexpr unsigned PAB = 32u * HM;      // pending abar deltas
    static constexpr unsigned ZF = 40u * HM;       // deferred zero-store flags (u32)
    static constexpr unsigned DIRTY = 44u * HM;    // dirty words (u32): slot has something pending
    static constexpr unsigned ROT = 48u * HM;      // refresh rotation counter
    static constexpr unsigned PROG = 48u * HM + 4; // this CTA's updates reported so far
    static constexpr unsigned BYTES = 48u * HM + 16;
};

__device__ __forceinline__ unsigned smem_base()
{
    extern __shared__ double smem_dyn[];
    return (unsigned)__cvta_generic_to_shared(smem_dyn);
}
__device__ __forceinline__ double lds64(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32_if(bool p, unsigned a, unsigned v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u32 [%1], %2;\n\t}" ::"r"((unsigned)p), "r"(a),
                 "r"(v)
                 : "memory");
}
__device__ __forceinline__ void sts64z_if(bool p, unsigned a)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u64 [%1], 0;\n\t}" ::"r"((unsigned)p), "r"(a)
                 : "memory");
}
// zero a staged pending accumulator atomically and return what it held.  The
// returned value must be consumed: an exchange whose result is discarded
// (ATOMS.EXCH RZ) does not fail another warp's in-flight ATOMS.CAST.SPIN add,
// so the stale deltas being dropped come back (measured: one CTA of 32 warps
// ends 2-7% above the optimum, configs 2/3 limit-cycle or diverge)
__device__ __forceinline__ double atoms_take64_if(bool p, unsigned a)
{
    double t = 0.0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q atom.shared.exch.b64 %0, [%2], 0;\n\t}"
                 : "+d"(t)
                 : "r"((unsigned)p), "r"(a)
                 : "memory");
    return t;
}
__device__ __forceinline__ void red_add_if(bool p, double *g, double v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.relaxed.gpu.global.add.f64 [%1], %2;\n\t}" ::"r"(
                     (unsigned)p),
                 "l"(g), "d"(v)
                 : "memory");
}
__device__ __forceinline__ void exch0_if(bool p, double *g)
{
    asm volatile("{\n\t.reg .pred q;\n\t.reg .b64 t;\n\tsetp.ne.u32 q, %0, 0;\n\t@q atom.relaxed.gpu.global.exch.b64 t, [%1], "
                 "0;\n\t}" ::"r"((unsigned)p),
                 "l"(g)
                 : "memory");
}
// fp64 add into a staged pending accumulator at byte offset `off` of the
// staging area (no native fp64 shared atomic on sm_100: the compiler's
// ATOMS.CAST.SPIN loop, which reconverges; the only divergent part of a commit)
__device__ __forceinline__ void sh_add_if(bool p, unsigned off, double v)
{
    extern __shared__ double smem_dyn[];
    if (p) atomicAdd(smem_dyn + (off >> 3), v);
}
__device__ __forceinline__ void sh_add_cas_if(bool p, unsigned a, double v)
{
    if (p) {
        unsigned long long old;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(old) : "r"(a) : "memory");
        while (true) {
            const unsigned long long nw = (unsigned long long)__double_as_longlong(__longlong_as_double((long long)old) + v);
            unsigned long long got;
            asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(got) : "r"(a), "l"(old), "l"(nw) : "memory");
            if (got == old) break;
            old = got;
        }
    }
    __syncwarp();
}
__device__ __forceinline__ double lds_take64(unsigned a)
{
    double v;
    asm volatile("atom.shared.exch.b64 %0, [%1], 0;" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned lds_take32(unsigned a)
{
    unsigned v;
    asm volatile("atom.shared.exch.b32 %0, [%1], 0;" : "=r"(v) : "r"(a) : "memory");
    return v;
}

// state of one nonzero: staged -> snapshot (x, abar) + D; else the 256-bit
// record (x, abar, D, reserved) from L2
__device__ __forceinline__ void gather3(bool staged, unsigned a_snap, unsigned a_d, const double *rec, double &x, double &ab,
                                        double &d)
{
    double r3;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
                 "@q ld.shared.v2.f64 {%0, %1}, [%5];\n\t"
                 "@q ld.shared.f64 %2, [%6];\n\t"
                 "@!q ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%7];\n\t}"
                 : "=&d"(x), "=&d"(ab), "=&d"(d), "=&d"(r3)  // early clobber: written before %6/%7 are read
                 : "r"((unsigned)staged), "r"(a_snap), "r"(a_d), "l"(rec)
                 : "memory");
}

// per-warp flush of the CTA's dirty staged slots (one RED per dirty (slot,
// field); deferred zero stores first), then the snapshot refresh: the
// HOT_TIER0 hottest slots every flush, the rest a rotating quarter; a cluster
// member refreshes from the leader CTA's snapshot (distributed shared memory)
template <int HM>
__device__ __noinline__ void hot3_flush(double *coord, const int H, const int shift, const unsigned lead, const int lane,
                                        const bool refresh, const bool variant = false)
{
    using L = Hot3<HM>;
    const unsigned base = smem_base();
    // lane l owns slots 128 r + 4 l + j (j < 4): bit 4 r + j of m
    unsigned m = 0u;
#pragma unroll
    for (int r = 0; r < HM / 128; r++) {
        uint4 w;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(base + L::DIRTY + 16u * (unsigned)(32 * r + lane))
                     : "memory");
        m |= ((w.x != 0u) | ((w.y != 0u) << 1) | ((w.z != 0u) << 2) | ((w.w != 0u) << 3)) << (4 * r);
    }
    if (variant) {
        for (int r0 = 0; r0 < HM; r0 += 128) {
            uint4 w;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(base + L::DIRTY + 4u * (unsigned)(r0 + 4 * lane))
                         : "memory");
            const unsigned ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (!ww[j]) continue;
                const unsigned s = (unsigned)(r0 + 4 * lane + j);
                sts32_if(true, base + L::DIRTY + 4u * s, 0u);
                const double dx = lds_take64(base + L::PX + 8u * s);
                const double dab = lds_take64(base + L::PAB + 8u * s);
                double *const g = coord + 4 * ((int64_t)s << shift);
                if (lds_take32(base + L::ZF + 4u * s)) atomic_exch(g, 0.0);
                if (dx != 0.0) red_add(g, dx);
                if (dab != 0.0) red_add(g + 1, dab);
            }
        }
        m = 0u;
    }
    while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1u;
        const unsigned s = 128u * (unsigned)(b >> 2) + 4u * (unsigned)lane + (unsigned)(b & 3);
        sts32_if(true, base + L::DIRTY + 4u * s, 0u);  // cleared before the pending values are taken
        const double dx = lds_take64(base + L::PX + 8u * s);
        const double dab = lds_take64(base + L::PAB + 8u * s);
        const unsigned zf = lds_take32(base + L::ZF + 4u * s);
        double *const g = coord + 4 * ((int64_t)s << shift);
        exch0_if(zf != 0u, g);  // deferred zero store, then the deltas added since
        red_add_if(dx != 0.0, g, dx);
        red_add_if(dab != 0.0, g + 1, dab);
    }
    if (!refresh) return;
    // the refresh must see this warp's REDs: lanes flush and refresh different
    // slots, and a cp.async read can overtake the thread's own fire-and-forget
    // REDs -- a snapshot missing the CTA's own flushed deltas makes its next
    // updates recompute them (measured without the fence: configs 2/3
    // limit-cycle or diverge)
    __threadfence();
    __syncwarp();
    unsigned rot = 0u;
    if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(rot) : "r"(base + L::ROT) : "memory");
    rot = __shfl_sync(FULL, rot, 0) & 3u;
    const int kmax = (H + 31) >> 5;
    if (lead) {
        for (int k = 0; k < kmax; k++) {
            const unsigned s = (unsigned)(lane + 32 * k);
            if (s < (unsigned)H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
                double2 v;
                asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(lead + L::SNAP + 16u * s));
                asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(base + L::SNAP + 16u * s), "d"(v.x), "d"(v.y) : "memory");
            }
        }
        return;
    }
    for (int k = 0; k < kmax; k++) {
        const unsigned s = (unsigned)(lane + 32 * k);
        if (s < (unsigned)H && (k < HOT_TIER0 / 32 || (k & 3) == (int)rot)) {
            const double *src = coord + 4 * ((int64_t)s << shift);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + L::SNAP + 16u * s), "l"(src) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// LITERAL: commit prox-zeroed coordinates as the delta -x_hat (PS_FLAG_DELTA_ZERO)
template <typename VT, typename PT, int LOSS, int PEN, bool LITERAL, int NC, int HM>
__global__ void __launch_bounds__(1024, 1) sps_hot3_kernel(const KArgs a)
{
    using L = Hot3<HM>;
    const unsigned base = smem_base();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int nwib = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * nwib + wib;
    const int H = a.H;
    double *const coord = a.coord;
    if (threadIdx.x == 0) {
        sts32_if(true, base + L::ROT, 0u);
        sts32_if(true, base + L::PROG, 0u);
    }
    if (H > 0) {
        for (int s = threadIdx.x; s < HM; s += blockDim.x) {
            double x = 0.0, ab = 0.0, d = 0.0;
            if (s < H) ld_record(coord + 4 * ((int64_t)s << a.hot_shift), x, ab, d);
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(base + L::SNAP + 16u * s), "d"(x), "d"(ab) : "memory");
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(base + L::D + 8u * s), "d"(d) : "memory");
            sts64z_if(true, base + L::PX + 8u * s);
            sts64z_if(true, base + L::PAB + 8u * s);
            sts32_if(true, base + L::ZF + 4u * s, 0u);
            sts32_if(true, base + L::DIRTY + 4u * s, 0u);
        }
    }
    __syncthreads();
    unsigned lead = 0u;
    if (a.cluster > 1) {
        unsigned rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        if (rank != 0 && H > 0) asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(base));
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    double *const alpha = a.alpha;
    const double gamma = a.gamma, lambda1 = a.lambda1, kappa = a.kappa, lam2 = a.lam2;
    const double plo = a.lo, phi = a.hi;
    const int pen = a.pen;
    const bool dcas = (a.diag & (1 << 27)) != 0;  // diagnostics: asm CAS loop instead of atomicAdd
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
        // deferred abar credit of the previous update: >= 0 cold column,
        // <= -2 staged slot -2 - pcol, -1 none
        int pcol[NC];
        double pval[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            pcol[c] = -1;
            pval[c] = 0.0;
        }
        double pnw = 0.0, prep = 0.0;
        unsigned t = 0u;
        while (true) {
            // ---- state reads (padding lanes read staged slot 0: finite, times a zero value)
            double xh[NC], ab[NC], d[NC];
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const bool act = col[c] >= 0;
                const bool hot = (unsigned)col[c] < hlim && ((unsigned)col[c] & hmask) == 0u;
                const unsigned sl = act ? (unsigned)col[c] >> shift : 0u;
                gather3(hot || !act, base + L::SNAP + 16u * sl, base + L::D + 8u * sl, coord + 4 * (int64_t)col[c], xh[c],
                        ab[c], d[c]);
            }
            double old = 0.0;
            if (lane == 0) old = ld_cg(alpha + ci);
            // ---- abar credit of the previous update (its alpha exchange has returned)
            {
                const double tq = (pnw - __shfl_sync(FULL, prep, 0)) * inv_n;
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    const double inc = tq * pval[c];
                    const bool stg = pcol[c] <= -2;
                    const unsigned ps = (unsigned)(-2 - pcol[c]);
                    red_add_if(pcol[c] >= 0, coord + 4 * (int64_t)pcol[c] + 1, inc);
                    if (dcas || (a.diag & (1 << 28))) sh_add_cas_if(stg, base + L::PAB + 8u * ps, inc);
                    else sh_add_if(stg, L::PAB + 8u * ps, inc);
                    sts32_if(stg, base + L::DIRTY + 4u * ps, 1u);
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
                // commit: a zero is stored, not added as the delta -x_hat (DESIGN.md
                // "zero commits"); a staged column already read as 0 is stored by
                // the CTA's next flush (flag), its pending delta dropped
                const bool act = col[c] >= 0;
                const bool hot = (unsigned)col[c] < hlim && ((unsigned)col[c] & hmask) == 0u;
                const unsigned sl = (unsigned)col[c] >> shift;
                const bool z0 = !LITERAL && act && z == 0.0;
                const bool defer = z0 && hot && xh[c] == 0.0;
                double *const gx = coord + 4 * (int64_t)col[c];
                const double dz = z - xh[c];
                red_add_if(act && !hot && !z0, gx, dz);
                exch0_if(z0 && !defer, gx);
                // a staged coordinate stored to 0: the CTA's snapshot shows the 0 at
                // once, so the CTA's next updates compute their deltas against it
                if (!(a.diag & (1 << 31))) sts64z_if(z0 && hot && !defer, base + L::SNAP + 16u * sl);
                // the coordinate is stored: drop the pending x delta (the dropped
                // value feeds a never-taken branch so the exchange keeps its result)
                if (z0 && hot && lds64(base + L::PX + 8u * sl) != 0.0) atoms_take64_if(true, base + L::PX + 8u * sl);
                if (a.diag & (1 << 30)) __threadfence_block();  // diagnostics: order the drop before the flags
                sts32_if(defer, base + L::ZF + 4u * sl, 1u);
                if (dcas || (a.diag & (1 << 29))) sh_add_cas_if(hot && !z0, base + L::PX + 8u * sl, dz);
                else sh_add_if(hot && !z0, L::PX + 8u * sl, dz);
                if (a.diag & (1 << 30)) __threadfence_block();
                sts32_if(hot, base + L::DIRTY + 4u * sl, 1u);  // after the pending update / zero flag (flush order)
                pcol[c] = hot ? -2 - (int)sl : col[c];
                pval[c] = cval;
            }
            // ---- alpha_i <-> new (the abar credit is issued next iteration)
            double rep = 0.0;
            if (lane == 0) rep = atomic_exch(alpha + ci, nw);
            pnw = nw;
            prep = rep;
            if (H > 0 && --until_flush == 0) {
                __syncwarp();
                hot3_flush<HM>(coord, H, shift, lead, lane, true, (a.diag & (1 << 30)) != 0);
                until_flush = a.period;
            }
            // progress: PROGRESS_BATCH updates of a warp into the CTA count, every
            // CTA_PROGRESS of the CTA into the global counter (asynchronous.py:155-162)
            if (lane == 0 && (t % PROGRESS_BATCH) == 0u) {
                unsigned o;
                asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(base + L::PROG), "r"((unsigned)PROGRESS_BATCH) : "memory");
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
            const bool stg = pcol[c] <= -2;
            const unsigned ps = (unsigned)(-2 - pcol[c]);
            red_add_if(pcol[c] >= 0, coord + 4 * (int64_t)pcol[c] + 1, tq * pval[c]);
            sh_add_if(stg, L::PAB + 8u * ps, tq * pval[c]);
            sts32_if(stg, base + L::DIRTY + 4u * ps, 1u);
        }
    }
    if (lane == 0 && todo % PROGRESS_BATCH) atomicAdd(a.counter, (unsigned long long)(todo % PROGRESS_BATCH));
    __syncthreads();  // every warp's CTA progress is in
    if (threadIdx.x == 0) {
        const unsigned prog = (unsigned)lds_take32(base + L::PROG);
        if (prog % CTA_PROGRESS) atomicAdd(a.counter, (unsigned long long)(prog % CTA_PROGRESS));
    }
    if (a.cluster > 1)  // the leader's staging area stays alive until every member stops reading it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (H > 0) {
        hot_async_drain();
        __syncthreads();
        if (wib == 0) {
            for (int s = lane; s < HM; s += 32) sts32_if(true, base + L::DIRTY + 4u * s, s < H ? 1u : 0u);
            __syncwarp();
            hot3_flush<HM>(coord, H, shift, 0u, lane, false);
        }
    }
}

}  // namespace ps
