// Arithmetic of the asynchronous kernels (sps_hot_kernel, the batched group
// kernel): the logistic derivative of losses.py:73-86 with a table exp and a
// one-Newton reciprocal division (<= 4 ulp from the deterministic kernels'
// libdevice arithmetic, tests/test_gpu_fast.py), the separable prox, and the
// 256-bit record load.  Included by several translation units (static tables).
#pragma once

#include "common.cuh"

namespace ps {

// 2^(j/64), j = 0..63, correctly rounded (tools/gen_exptab.py)
static __constant__ double c_exp2_64[64] = {
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
static __constant__ double c_exp_k[8] = {
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

}  // namespace ps
