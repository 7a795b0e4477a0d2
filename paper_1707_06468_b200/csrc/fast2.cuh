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

namespace ps {

// 2^(j/64), j = 0..63, correctly rounded (tools/gen_exptab.py)
__constant__ double c_exp2_64[64] = {
    0x1.0000000000000p+0,
    0x1.02c9a3e778061p+0,
    0x1.059b0d3158574p+0,
    0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0,
    0x1.0e3ec32d3d1a2p+0,
    0x1.11301d0125b51p+0,
    0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0,
    0x1.1a35beb6fcb75p+0,
    0x1.1d4873168b9aap+0,
    0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0,
    0x1.26b4565e27cddp+0,
    0x1.29e9df51fdee1p+0,
    0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0,
    0x1.33c08b26416ffp+0,
    0x1.371a7373aa9cbp+0,
    0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0,
    0x1.4160a21f72e2ap+0,
    0x1.44e086061892dp+0,
    0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0,
    0x1.4f9b2769d2ca7p+0,
    0x1.5342b569d4f82p+0,
    0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0,
    0x1.5e76f15ad2148p+0,
    0x1.6247eb03a5585p+0,
    0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0,
    0x1.6dfb23c651a2fp+0,
    0x1.71f75e8ec5f74p+0,
    0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0,
    0x1.7e2f336cf4e62p+0,
    0x1.82589994cce13p+0,
    0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0,
    0x1.8f1ae99157736p+0,
    0x1.93737b0cdc5e5p+0,
    0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0,
    0x1.a0c667b5de565p+0,
    0x1.a5503b23e255dp+0,
    0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0,
    0x1.b33a2b84f15fbp+0,
    0x1.b7f76f2fb5e47p+0,
    0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0,
    0x1.c67f12e57d14bp+0,
    0x1.cb720dcef9069p+0,
    0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0,
    0x1.da9e603db3285p+0,
    0x1.dfc97337b9b5fp+0,
    0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0,
    0x1.efa1bee615a27p+0,
    0x1.f50765b6e4540p+0,
    0x1.fa7c1819e90d8p+0
};

// polynomial / reduction constants (constant bank operands, not UMOV pairs)
__constant__ double c_exp_k[8] = {
    0x1.71547652b82fep+6,   // 64 / ln2
    -0x1.62e42fefa0000p-7,  // -ln2_hi / 64 (36 significant bits: kd * it is exact for |kd| < 2^17)
    -0x1.cf79abc9e3b3ap-46, // -ln2_lo / 64
    0x1.1111111111111p-7,   // 1/120
    0x1.5555555555555p-5,   // 1/24
    0x1.5555555555555p-3,   // 1/6
    0x1.8p52,               // round-to-integer shifter
    -746.0};

// exp(x) for x <= 0 (or NaN): x = (64 m + j) ln2/64 + r, |r| <= ln2/128;
// exp(r) - 1 = r (1 + r/2 + r^2/6 + r^3/24 + r^4/120) (truncation < 4e-17);
// 2^m applied as two exact power-of-two factors (subnormal results round once).
__device__ __forceinline__ double exp_nonpos2(double x)
{
    x = x < c_exp_k[7] ? c_exp_k[7] : x;
    double kd = __fma_rn(x, c_exp_k[0], c_exp_k[6]);
    const int n = __double2loint(kd);
    kd = __dsub_rn(kd, c_exp_k[6]);
    double r = __fma_rn(kd, c_exp_k[1], x);
    r = __fma_rn(kd, c_exp_k[2], r);
    double q = __fma_rn(r, c_exp_k[3], c_exp_k[4]);
    q = __fma_rn(q, r, c_exp_k[5]);
    q = __fma_rn(q, r, 0.5);
    q = __fma_rn(q, r, 1.0);
    const double s = __dmul_rn(r, q);  // exp(r) - 1
    const double T = c_exp2_64[n & 63];
    double y = __fma_rn(T, s, T);
    const int m = n >> 6, m1 = m >> 1, m2 = m - m1;  // m in [-1077, 0]
    y = __dmul_rn(y, __hiloint2double((m1 + 1023) << 20, 0));
    return __dmul_rn(y, __hiloint2double((m2 + 1023) << 20, 0));
}

// num / den for den in [1, 2]: reciprocal estimate, one Newton step, one
// residual correction of the quotient
__device__ __forceinline__ double div_1to2b(double num, double den)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
    y = __fma_rn(y, __fma_rn(-den, y, 1.0), y);
    const double q = __dmul_rn(num, y);
    return __fma_rn(__fma_rn(-den, q, num), y, q);
}

// losses.py:73-86: et = exp(-|t|), sig = (t > 0 ? 1 : et) / (1 + et), l' = -b sig
template <int LOSS> __device__ __forceinline__ double deriv2(double z, double b)
{
    if (LOSS == PS_LOSS_LOGISTIC) {
        const double t = -b * z;
        const double et = exp_nonpos2(-fabs(t));
        return -b * div_1to2b(t > 0 ? 1.0 : et, 1.0 + et);
    }
    return z - b;
}

// 256-bit L2 load of a coordinate record (x, abar, D, reserved)
__device__ __forceinline__ void ld_record(const double *p, double &x, double &ab, double &d)
{
    double r3;
    asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(x), "=d"(ab), "=d"(d), "=d"(r3) : "l"(p));
}

// separable prox with effective step eff (penalties.py:78-81 / :134-135 / :60-61);
// L1 as copysign(max(|u| - thr, 0), u) (the sign of a zero result is irrelevant:
// a zero is committed as a store of +0)
template <int PEN>
__device__ __forceinline__ double prox2(double u, double eff, double lam2, int pen, double lo, double hi)
{
    if (PEN == PS_PEN_L1) {
        const double m = fabs(u) - eff * lam2;
        return copysign(m > 0.0 ? m : 0.0, u);
    }
    return prox_sep(pen, u, eff, lam2, lo, hi);
}

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
