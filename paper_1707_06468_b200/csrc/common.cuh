// Device helpers shared by the SPS kernels and the auxiliary kernels.
// Arithmetic restates the reference's scalar formulas (cited per function)
// in fp64; data values stored as fp32 are widened exactly before use.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/proxsaga.h"

namespace ps {

constexpr unsigned FULL = 0xffffffffu;

// L2-coherent loads for shared mutable state (x, abar, alpha): bypass L1 so a
// warp never reuses a stale L1 line of a cell other warps update atomically
// (the "inconsistent read" of asynchronous.py:92-96 is a read of L2).
__device__ __forceinline__ double ld_cg(const double *p) { return __ldcg(p); }
__device__ __forceinline__ double2 ld_cg2(const double *p)
{
    return __ldcg(reinterpret_cast<const double2 *>(p));
}
// Fire-and-forget fp64 add resolved at L2 (REDG.E.ADD.F64), the device form of
// _atomics.c:59-75 atomic_add_f64 / py_scatter_add.
__device__ __forceinline__ void red_add(double *p, double v)
{
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// _atomics.c:260-283 py_exchange.
__device__ __forceinline__ double atomic_exch(double *p, double v)
{
    return __longlong_as_double(
        (long long)atomicExch(reinterpret_cast<unsigned long long *>(p),
                              (unsigned long long)__double_as_longlong(v)));
}

template <typename T> __device__ __forceinline__ double widen(T v) { return (double)v; }

// Butterfly all-reduce: every lane ends with the bitwise-identical sum
// (a+b == b+a exactly, so both partners of each exchange agree).
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// losses.py:73-86 loss_scalar (derivative part): branchy overflow-safe sigmoid.
__device__ __forceinline__ double loss_deriv(int loss, double z, double b)
{
    if (loss == PS_LOSS_LOGISTIC) {
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

// losses.py:53-59 (_log1pexp) / :34-36 (squared).
__device__ __forceinline__ double loss_value(int loss, double z, double b)
{
    if (loss == PS_LOSS_LOGISTIC) {
        double t = -b * z;
        if (t > 0) return t + log1p(exp(-t));
        return log1p(exp(t));
    }
    double d = z - b;
    return 0.5 * d * d;
}

// Separable prox with effective step eff (= gamma * d):
// penalties.py:78-81 (L1 soft threshold, threshold = eff*lam2),
// :134-135 (box clamp), :60-61 (identity).
__device__ __forceinline__ double prox_sep(int pen, double u, double eff, double lam2, double lo,
                                           double hi)
{
    if (pen == PS_PEN_L1) {
        double thr = eff * lam2;
        double a = fmax(fabs(u) - thr, 0.0);
        return u > 0 ? a : (u < 0 ? -a : 0.0);
    }
    if (pen == PS_PEN_BOX) return u < lo ? lo : (u > hi ? hi : u);
    return u;
}

// penalties.py:103-108 GroupL2Penalty.prox_block scale factor for a block
// with norm `norm` and effective step eff: z = u * f (z = 0 when norm == 0).
__device__ __forceinline__ double group_factor(double norm, double eff, double lam2)
{
    if (norm == 0.0) return 0.0;
    return fmax(0.0, 1.0 - eff * lam2 / norm);
}

// Counter-based sampler for the asynchronous mode: slot s of stream `seed`
// maps to a uniform row in [0, n) (splitmix64 + Lemire multiply-high).  The
// reference draws PCG64 per worker (asynchronous.py:120-122); async parity is
// on the objective, so the stream only needs to be uniform and reproducible.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ int64_t sample_row(uint64_t seed_mix, uint64_t slot, uint64_t n)
{
    // seed_mix = splitmix64(seed) precomputed on the host side of the launch
    uint64_t h = splitmix64(seed_mix + slot * 0x9E3779B97F4A7C15ull);
    return (int64_t)__umul64hi(h, n);
}

}  // namespace ps
