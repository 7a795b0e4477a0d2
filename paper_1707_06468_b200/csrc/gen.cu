// K7: on-device generator for the large BASELINE configs (3 and 4), which
// host numpy cannot build in reasonable time (6e8 / 1.6e9 nonzeros).
// One warp per row: each lane draws one column from a Zipf(s) law by
// inverse-CDF binary search (the CDF table is built on the host), the warp
// bitonic-sorts its draws and redraws duplicates until the k columns are
// distinct (resample-until-distinct); values are binary or
// lognormal(0,1), then the row is l2-normalised.  Config 4's 13 "dense"
// columns [0, 13) are in every row; its 22 Zipf columns are drawn over
// [13, p).  Counter-based RNG: splitmix64(seed, row, round, lane).
#include <climits>
#include <cmath>

#include "common.cuh"
#include "internal.h"

using namespace ps;

namespace {

__device__ __forceinline__ uint64_t rng(uint64_t seed, uint64_t a, uint64_t b)
{
    return splitmix64(splitmix64(seed ^ (a * 0x9E3779B97F4A7C15ull)) + b);
}

__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

// first index with cdf[idx] > u  (cdf increasing, cdf[m-1] == 1)
__device__ __forceinline__ int64_t cdf_search(const double *cdf, int64_t m, double u)
{
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(cdf + mid) > u) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ void bitonic32(int &c, int lane)
{
    for (int size = 2; size <= 32; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            int oc = __shfl_xor_sync(FULL, c, stride);
            bool up = (lane & size) == 0, lower = (lane & stride) == 0;
            if (lower ? (up ? oc < c : oc > c) : (up ? oc > c : oc < c)) c = oc;
        }
}

// rows with k_dense fixed columns [0, k_dense) + k_zipf distinct Zipf draws over
// [k_dense, k_dense + m) (m = CDF length); k = k_dense + k_zipf <= 32
__global__ void k_gen_rows(int64_t n, int k_dense, int k_zipf, const double *cdf, int64_t m, uint64_t seed,
                           int lognormal, int32_t *col, float *val)
{
    const int lane = threadIdx.x & 31;
    const int k = k_dense + k_zipf;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        // zipf part: lanes [0, k_zipf) hold draws; others +inf
        int c = INT_MAX;
        if (lane < k_zipf) c = k_dense + (int)cdf_search(cdf, m, u01(rng(seed, (uint64_t)i, (uint64_t)lane)));
        bitonic32(c, lane);
        for (int round = 1; round < 64; round++) {
            int prev = __shfl_up_sync(FULL, c, 1);
            bool dup = lane > 0 && lane < k_zipf && c == prev;
            if (!__any_sync(FULL, dup)) break;
            if (dup)
                c = k_dense + (int)cdf_search(cdf, m, u01(rng(seed, (uint64_t)i, (uint64_t)(lane + 32 * round))));
            bitonic32(c, lane);
        }
        // dense columns first (they are the smallest ids), then the sorted draws;
        // up to two 32-wide output chunks (k <= 64)
        double v[2], sq = 0.0;
        int oc[2];
#pragma unroll
        for (int ch = 0; ch < 2; ch++) {
            const int e = lane + 32 * ch;
            const int src = (e - k_dense) & 31;
            const int zc = __shfl_sync(FULL, c, src);
            oc[ch] = e < k_dense ? e : zc;
            v[ch] = 1.0;
            if (lognormal) {  // exp(N(0,1)) by Box-Muller
                uint64_t h = rng(seed ^ 0x5bd1e995ull, (uint64_t)i, (uint64_t)e);
                double u1 = fmax(u01(h), 1e-300), u2 = u01(splitmix64(h));
                v[ch] = exp(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
            }
            if (e < k) sq += v[ch] * v[ch];
        }
        sq = warp_sum(sq);
        const double inv = 1.0 / sqrt(sq);
#pragma unroll
        for (int ch = 0; ch < 2; ch++) {
            const int e = lane + 32 * ch;
            if (e < k) {
                const int64_t idx = i * (int64_t)k + e;
                col[idx] = oc[ch];
                val[idx] = (float)(v[ch] * inv);
            }
        }
    }
}

__global__ void k_row_ptr_uniform(int64_t n, int k, int64_t *row_ptr)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
        row_ptr[i] = i * (int64_t)k;
}

// labels y_i = sign(a_i . w + noise * N(0,1)) with sign(0) = +1 (problems.py:42)
__global__ void k_labels(int64_t n, int k, const int32_t *col, const float *val, const double *w, double noise,
                         uint64_t seed, float *y)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double z = 0.0;
        for (int e = 0; e < k; e++) z += (double)val[i * k + e] * w[col[i * k + e]];
        uint64_t h = rng(seed ^ 0x27d4eb2dull, (uint64_t)i, 7);
        double u1 = fmax(u01(h), 1e-300), u2 = u01(splitmix64(h));
        z += noise * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        y[i] = z >= 0 ? 1.0f : -1.0f;
    }
}

}  // namespace

extern "C" int ps_gen_zipf_csr(int64_t n, int32_t k_dense, int32_t k_zipf, const double *cdf, int64_t m,
                               uint64_t seed, int32_t lognormal, int64_t *row_ptr, int32_t *col, float *val,
                               void *stream)
{
    if (n < 1 || k_dense < 0 || k_zipf < 0 || k_dense + k_zipf < 1 || k_zipf > 32 || k_dense + k_zipf > 64 || !cdf ||
        m < k_zipf || !row_ptr || !col || !val)
        return ps_fail(PS_EINVAL, "bad generator arguments (k_zipf <= 32, k <= 64, m >= k_zipf)");
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_row_ptr_uniform<<<sms * 8, 256, 0, st>>>(n, k_dense + k_zipf, row_ptr);
    k_gen_rows<<<sms * 16, 256, 0, st>>>(n, k_dense, k_zipf, cdf, m, seed, lognormal, col, val);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_gen_zipf_csr");
    return PS_OK;
}

extern "C" int ps_gen_labels(int64_t n, int32_t k, const int32_t *col, const float *val, const double *w,
                             double noise, uint64_t seed, float *y, void *stream)
{
    if (n < 1 || k < 1 || !col || !val || !w || !y) return ps_fail(PS_EINVAL, "bad label arguments");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_labels<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(n, k, col, val, w, noise, seed, y);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ps_cuda_fail(e, "ps_gen_labels");
    return PS_OK;
}
