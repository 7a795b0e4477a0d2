// Auxiliary device kernels around the SPS loop:
//   ps_prepare            K5/K6: block counts n_B, weights d_B, delta, dead
//                         blocks, max ||a_i||^2, per-row T_i (GENERAL)
//   ps_objective          K3: full objective (SpMV + loss + ||x||^2 + h(x))
//   ps_smooth_gradient    K4: A^T l'(Ax)/n + lambda1 x
//   ps_fixed_point_residual, ps_resync_average, ps_prox, coord get/set,
//   and the device forms of the reference's _atomics primitives.
// Reductions are deterministic: per-CTA partials, then one CTA sums them in
// CTA order.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

using namespace ps;

// ---------------------------------------------------------------------------
// error state
static thread_local std::string g_err;

int ps_fail(int code, const char *msg)
{
    g_err = msg ? msg : "";
    return code;
}

int ps_cuda_fail(cudaError_t e, const char *where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return PS_ECUDA;
}

extern "C" int ps_abi_version(void) { return PS_ABI_VERSION; }
extern "C" const char *ps_last_error(void) { return g_err.c_str(); }
extern "C" int ps_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}


// Scratch of the aux entry points comes from the device's default stream-
// ordered pool.  Its release threshold defaults to 0, i.e. every synchronize
// hands freed pages back and the next cudaMallocAsync maps them again (about a
// millisecond, measured on ps_objective); keep them instead.
static cudaError_t pool_alloc(void **ptr, size_t bytes, cudaStream_t st)
{
    static bool kept[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !kept[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        kept[dev] = true;
    }
    return cudaMallocAsync(ptr, bytes, st);
}

static int sm_count()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

template <typename PT> __device__ __forceinline__ int64_t rpx(const void *p, int64_t i)
{
    return (int64_t)reinterpret_cast<const PT *>(p)[i];
}
template <typename VT> __device__ __forceinline__ double rvx(const void *p, int64_t e)
{
    return widen(reinterpret_cast<const VT *>(p)[e]);
}

// Block-level sum of one double per thread into out[blockIdx.x] (blockDim 256).
__device__ __forceinline__ void block_sum_store(double v, double *out)
{
    __shared__ double red[8];
    v = warp_sum(v);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        double s = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
        s = warp_sum(s);
        if (l == 0) out[blockIdx.x] = s;
    }
    __syncthreads();
}

// Final ordered sum of `nparts` partials (single CTA of 256 threads).
__global__ void k_finish_sum(const double *parts, int nparts, int ncols, double *out, double scale0)
{
    // parts laid out [col][nparts]; out[col] = sum (col 0 scaled by scale0)
    for (int c = 0; c < ncols; c++) {
        double v = 0.0;
        for (int q = threadIdx.x; q < nparts; q += blockDim.x) v += parts[(int64_t)c * nparts + q];
        __shared__ double red[8];
        v = warp_sum(v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
            out[c] = c == 0 ? s * scale0 : s;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// ps_prepare kernels

// per row: ||a_i||^2 (losses.py:99-105 via data.py:74-80), nnz; maxima
// reduced per warp first (one atomic per warp, not per row: a per-row atomic
// on one address serialises ~n L2 operations).
template <typename VT, typename PT>
__global__ void k_rowstats(const void *row_ptr, const void *val, int64_t n, unsigned long long *max_sq,
                           int *max_nnz)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    int k = 0;
    if (i < n) {
        int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
        for (int64_t e = lo; e < hi; e++) {
            double v = rvx<VT>(val, e);
            s += v * v;
        }
        k = (int)(hi - lo);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    k = __reduce_max_sync(0xffffffffu, k);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(max_sq, (unsigned long long)__double_as_longlong(s));  // s >= 0: bit order == value order
        atomicMax(max_nnz, k);
    }
}

// singleton: n_j = #rows containing column j (columns distinct within a row).
// The leading CNT_HEAD columns are counted per CTA in shared memory first: a
// Zipf head column sits in almost every row, and a global atomic per nonzero
// queues ~n operations on its L2 line (config 2: 0.25 ms -> ~10 us).  Hot
// columns are in the head both in original order (Zipf rank = index) and
// after ps_hot_layout (hot rank r at index r * stride).
constexpr int CNT_HEAD = 8192;
__global__ void __launch_bounds__(512) k_count_cols(const int32_t *col, int64_t nnz, int64_t p, int32_t *counts)
{
    __shared__ int32_t bins[CNT_HEAD];
    const int hb = p < (int64_t)CNT_HEAD ? (int)p : CNT_HEAD;
    for (int j = threadIdx.x; j < hb; j += blockDim.x) bins[j] = 0;
    __syncthreads();
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = col[e];
        if (c < hb) atomicAdd(bins + c, 1);
        else atomicAdd(counts + c, 1);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < hb; j += blockDim.x)
        if (bins[j]) atomicAdd(counts + j, bins[j]);
}
static void count_cols(const int32_t *col, int64_t nnz, int64_t p, int32_t *counts, int sms, cudaStream_t st)
{
    // enough nonzeros per CTA that the head flush (CNT_HEAD bins) stays small
    int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 4, (nnz + 4095) / 4096));
    k_count_cols<<<(int)ctas, 512, 0, st>>>(col, nnz, p, counts);
}

// contiguous groups: count each distinct block of a row once; max slots.
template <typename PT>
__global__ void k_count_contig(const void *row_ptr, const int32_t *col, int64_t n, int G, int32_t *counts,
                               int *max_slots)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
    int prev = -1, g = 0;
    for (int64_t e = lo; e < hi; e++) {
        int b = col[e] / G;
        if (b != prev) {
            atomicAdd(counts + b, 1);
            prev = b;
            g++;
        }
    }
    atomicMax(max_slots, g * G);
}

// general partition: per row, sorted unique blocks -> row_blk[lo..lo+g),
// counts, slot of each nonzero (block offset + rank within the block).
template <typename PT>
__global__ void k_index_general(const void *row_ptr, const int32_t *col, int64_t n, const int32_t *block_of,
                                const int32_t *blk_ptr, const int32_t *blk_coords, int32_t *counts,
                                int32_t *row_blk, int32_t *row_g, int32_t *spos, int *max_slots)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
    int g = 0;
    for (int64_t e = lo; e < hi; e++) {  // insertion into a sorted unique list
        int b = block_of[col[e]];
        int q = g;
        while (q > 0 && row_blk[lo + q - 1] > b) q--;
        if (q > 0 && row_blk[lo + q - 1] == b) continue;
        for (int r = g; r > q; r--) row_blk[lo + r] = row_blk[lo + r - 1];
        row_blk[lo + q] = b;
        g++;
    }
    row_g[i] = g;
    int slots = 0;
    for (int t = 0; t < g; t++) {
        int b = row_blk[lo + t];
        atomicAdd(counts + b, 1);
        slots += blk_ptr[b + 1] - blk_ptr[b];
    }
    atomicMax(max_slots, slots);
    for (int64_t e = lo; e < hi; e++) {
        int c = col[e], b = block_of[c];
        int off = 0, t = 0;
        while (row_blk[lo + t] != b) {  // blocks sorted: offset = sizes of smaller ones
            off += blk_ptr[row_blk[lo + t] + 1] - blk_ptr[row_blk[lo + t]];
            t++;
        }
        int a0 = blk_ptr[b], a1 = blk_ptr[b + 1];  // rank of c inside its block
        while (a0 < a1) {
            int mid = (a0 + a1) >> 1;
            if (blk_coords[mid] < c) a0 = mid + 1;
            else a1 = mid;
        }
        spos[e] = off + (a0 - blk_ptr[b]);
    }
}

// data.py:259-262: d_B = n / n_B (0 for dead), max n_B, dead count (warp
// reductions, one atomic per warp).
__global__ void k_weights(const int32_t *counts, int64_t nb, int64_t n, double *w, unsigned long long *maxc,
                          unsigned long long *dead)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t end = (nb + 31) / 32 * 32;  // whole warps stay in the loop
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < end; b += stride) {
        int c = 0;
        unsigned nd = 0;
        if (b < nb) {
            c = counts[b];
            w[b] = c > 0 ? (double)n / (double)c : 0.0;
            nd = c == 0;
        }
        c = __reduce_max_sync(0xffffffffu, c);
        nd = __reduce_add_sync(0xffffffffu, nd);
        if ((threadIdx.x & 31) == 0) {
            if (nd) atomicAdd(dead, (unsigned long long)nd);
            atomicMax(maxc, (unsigned long long)c);
        }
    }
}

// coord_weights (data.py:228-233): D_j = d_{B(j)} into coord[4j+2].
__global__ void k_coord_weights(double *coord, int64_t p, int kind, int G, const int32_t *block_of,
                                const double *w)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = kind == PS_PART_SINGLETON ? j : (kind == PS_PART_CONTIG ? j / G : block_of[j]);
        coord[4 * j + 2] = w[b];
    }
}

extern "C" int ps_prepare(const ps_csr_t *csr, ps_part_t *part, double *coord, ps_stats_t *stats, void *stream)
{
    NvtxRange nvtx_range("K5 ps_prepare");
    if (!csr || !part || !coord || !stats) return ps_fail(PS_EINVAL, "null argument");
    if (csr->n_rows < 1) return ps_fail(PS_EINVAL, "dataset is empty");
    if (!part->blk_count || !part->blk_weight) return ps_fail(PS_EINVAL, "blk_count / blk_weight required");
    if (part->kind == PS_PART_CONTIG && part->G < 1) return ps_fail(PS_EINVAL, "G must be >= 1");
    if (part->kind == PS_PART_GENERAL &&
        (!part->block_of || !part->blk_ptr || !part->blk_coords || !part->row_blk || !part->row_g || !part->spos))
        return ps_fail(PS_EINVAL, "general partition needs block_of/blk_ptr/blk_coords/row_blk/row_g/spos");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t n = csr->n_rows, p = csr->n_cols, nb = part->n_blocks;
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;

    // tmp: [max_sq u64][maxc u64][dead u64][max_nnz i32][max_slots i32]
    void *tmp = nullptr;
    CK(pool_alloc(&tmp, 64, st), "ps_prepare alloc");
    CK(cudaMemsetAsync(tmp, 0, 64, st), "ps_prepare memset");
    unsigned long long *max_sq = (unsigned long long *)tmp;
    unsigned long long *maxc = max_sq + 1, *dead = max_sq + 2;
    int *max_nnz = (int *)(max_sq + 3), *max_slots = max_nnz + 1;
    CK(cudaMemsetAsync(part->blk_count, 0, sizeof(int32_t) * nb, st), "ps_prepare memset counts");

    int tb = 256;
    int rows_grid = (int)((n + tb - 1) / tb);
    if (f64 && i64) k_rowstats<double, long long><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->values, n, max_sq, max_nnz);
    else if (f64) k_rowstats<double, int><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->values, n, max_sq, max_nnz);
    else if (i64) k_rowstats<float, long long><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->values, n, max_sq, max_nnz);
    else k_rowstats<float, int><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->values, n, max_sq, max_nnz);

    int grid = sm_count() * 8;
    if (part->kind == PS_PART_SINGLETON) {
        if (csr->nnz > 0) count_cols(csr->col_idx, csr->nnz, p, part->blk_count, sm_count(), st);
    } else if (part->kind == PS_PART_CONTIG) {
        if (i64) k_count_contig<long long><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->col_idx, n, part->G, part->blk_count, max_slots);
        else k_count_contig<int><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->col_idx, n, part->G, part->blk_count, max_slots);
    } else {
        if (i64)
            k_index_general<long long><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->col_idx, n, part->block_of, part->blk_ptr,
                                                                  part->blk_coords, part->blk_count, part->row_blk,
                                                                  part->row_g, part->spos, max_slots);
        else
            k_index_general<int><<<rows_grid, tb, 0, st>>>(csr->row_ptr, csr->col_idx, n, part->block_of, part->blk_ptr,
                                                            part->blk_coords, part->blk_count, part->row_blk,
                                                            part->row_g, part->spos, max_slots);
    }
    k_weights<<<grid, tb, 0, st>>>(part->blk_count, nb, n, part->blk_weight, maxc, dead);
    k_coord_weights<<<grid, tb, 0, st>>>(coord, p, part->kind, part->G, part->block_of, part->blk_weight);
    CK(cudaGetLastError(), "ps_prepare launch");

    unsigned long long h[8];
    CK(cudaMemcpyAsync(h, tmp, 64, cudaMemcpyDeviceToHost, st), "ps_prepare readback");
    CK(cudaFreeAsync(tmp, st), "ps_prepare free");
    CK(cudaStreamSynchronize(st), "ps_prepare sync");
    int *hi32 = (int *)(h + 3);
    double msq;
    std::memcpy(&msq, &h[0], 8);
    stats->max_row_sqnorm = msq;
    stats->max_count = (int64_t)h[1];
    stats->n_dead = (int64_t)h[2];
    stats->max_row_nnz = hi32[0];
    stats->max_slots = part->kind == PS_PART_SINGLETON ? hi32[0] : hi32[1];
    part->max_slots = stats->max_slots;
    part->max_row_nnz = stats->max_row_nnz;
    return PS_OK;
}

// ---------------------------------------------------------------------------
// ps_objective (losses.py:134-136: mean loss + lambda1/2 ||x||^2 + penalty) in
// one launch (checkpoints evaluate it every epoch; separate launches for the
// loss pass, the coordinate terms, the final sum and the combine cost more
// than the work): per-CTA partials of the loss (thread per row for short rows,
// warp per row otherwise), of ||x||^2 and of the penalty (|x|, box violations,
// or sum_B ||x_B|| for the group penalty, penalties.py:97-101), then the last
// CTA to finish sums them in a fixed order (deterministic) and combines.
template <typename VT, typename PT, bool TROW>
__global__ void __launch_bounds__(256) k_objective_fused(const void *row_ptr, const int32_t *col, const void *val,
                                                         const void *y, int64_t n, int loss, const double *x, int xs,
                                                         int64_t p, int pen, double lo, double hi, int kind, int G,
                                                         int64_t nb, const int32_t *blk_ptr, const int32_t *blk_coords,
                                                         double lambda1, double lam2, double *parts, unsigned *done,
                                                         double *out)
{
    const int G1 = gridDim.x;
    double acc = 0.0;
    if (TROW) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            int64_t lo_ = rpx<PT>(row_ptr, i), hi_ = rpx<PT>(row_ptr, i + 1);
            double z = 0.0;
#pragma unroll 8
            for (int64_t e = lo_; e < hi_; e++) z += rvx<VT>(val, e) * x[(int64_t)col[e] * xs];
            acc += loss_value(loss, z, rvx<VT>(y, i));
        }
    } else {
        const int lane = threadIdx.x & 31;
        const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t i = w; i < n; i += nw) {
            int64_t lo_ = rpx<PT>(row_ptr, i), hi_ = rpx<PT>(row_ptr, i + 1);
            double z = 0.0;
            for (int64_t e = lo_ + lane; e < hi_; e += 32) z += rvx<VT>(val, e) * x[(int64_t)col[e] * xs];
            z = warp_sum(z);
            if (lane == 0) acc += loss_value(loss, z, rvx<VT>(y, i));
        }
    }
    block_sum_store(acc, parts);
    double xx = 0.0, pv = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        double v = x[j * xs];
        xx += v * v;
        if (pen == PS_PEN_L1) pv += fabs(v);
        else if (pen == PS_PEN_BOX && !(v >= lo && v <= hi)) pv += 1.0;
    }
    block_sum_store(xx, parts + G1);
    if (pen == PS_PEN_GROUP) {
        double gv = 0.0;
        for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
            double ss = 0.0;
            if (kind == PS_PART_GENERAL) {
                for (int q = blk_ptr[b]; q < blk_ptr[b + 1]; q++) {
                    double v = x[(int64_t)blk_coords[q] * xs];
                    ss += v * v;
                }
            } else {
                int64_t g = kind == PS_PART_SINGLETON ? 1 : G;
                for (int64_t j = b * g; j < min((b + 1) * g, p); j++) {
                    double v = x[j * xs];
                    ss += v * v;
                }
            }
            gv += sqrt(ss);
        }
        block_sum_store(gv, parts + 2 * G1);
    } else {
        block_sum_store(pv, parts + 2 * G1);
    }
    // last CTA: fixed-order final sums + combine
    __shared__ bool last;
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == (unsigned)gridDim.x - 1u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ double sums[3];
    for (int c = 0; c < 3; c++) {
        double v = 0.0;
        for (int q = threadIdx.x; q < G1; q += blockDim.x) v += ld_cg(parts + (int64_t)c * G1 + q);
        __shared__ double red[8];
        v = warp_sum(v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
            sums[c] = c == 0 ? t * (1.0 / (double)n) : t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sums[0];
        out[1] = 0.5 * lambda1 * sums[1];
        if (pen == PS_PEN_L1 || pen == PS_PEN_GROUP) out[2] = lam2 * sums[2];
        else if (pen == PS_PEN_BOX) out[2] = sums[2] > 0 ? INFINITY : 0.0;
        else out[2] = 0.0;
    }
}

extern "C" int ps_objective(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *x,
                            int32_t x_stride, double *out, void *stream)
{
    NvtxRange nvtx_range("K3 ps_objective");
    if (!csr || !part || !prm || !x || !out) return ps_fail(PS_EINVAL, "null argument");
    if (csr->n_rows < 1) return ps_fail(PS_EINVAL, "dataset is empty");
    cudaStream_t st = (cudaStream_t)stream;
    const int G1 = std::max(1, sm_count() * 4);  // CTAs per partial pass (fixed -> deterministic)
    double *parts = nullptr;
    CK(pool_alloc((void **)&parts, sizeof(double) * (3 * G1 + 1), st), "ps_objective alloc");
    unsigned *done = reinterpret_cast<unsigned *>(parts + 3 * G1);
    CK(cudaMemsetAsync(done, 0, sizeof(unsigned), st), "ps_objective memset");
    const int64_t n = csr->n_rows, p = csr->n_cols;
    const bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    const bool trow = part->max_row_nnz > 0 && part->max_row_nnz <= 64;  // short rows: thread per row
    const int64_t nb = part->kind == PS_PART_SINGLETON ? p : part->n_blocks;
#define OBJ_FUSED(V, P, T)                                                                                           \
    k_objective_fused<V, P, T><<<G1, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, n,        \
                                                   prm->loss, x, x_stride, p, prm->penalty, prm->lo, prm->hi,      \
                                                   part->kind, part->G, nb, part->blk_ptr, part->blk_coords,       \
                                                   prm->lambda1, prm->lam2, parts, done, out)
    if (trow) {
        if (f64 && i64) OBJ_FUSED(double, long long, true);
        else if (f64) OBJ_FUSED(double, int, true);
        else if (i64) OBJ_FUSED(float, long long, true);
        else OBJ_FUSED(float, int, true);
    } else {
        if (f64 && i64) OBJ_FUSED(double, long long, false);
        else if (f64) OBJ_FUSED(double, int, false);
        else if (i64) OBJ_FUSED(float, long long, false);
        else OBJ_FUSED(float, int, false);
    }
#undef OBJ_FUSED
    CK(cudaGetLastError(), "ps_objective launch");
    CK(cudaFreeAsync(parts, st), "ps_objective free");
    return PS_OK;
}

// ---------------------------------------------------------------------------
// smooth gradient / resync: A^T s via atomic scatter (warp per row).
template <typename VT, typename PT>
__global__ void __launch_bounds__(256) k_rmatvec_deriv(const void *row_ptr, const int32_t *col, const void *val,
                                                       const void *y, int64_t n, int loss, const double *x, int xs,
                                                       const double *s, double *out, int os)
{
    int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
        int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
        double d;
        if (s) {
            d = s[i];
        } else {
            double z = 0.0;
            for (int64_t e = lo + lane; e < hi; e += 32) z += rvx<VT>(val, e) * x[(int64_t)col[e] * xs];
            z = warp_sum(z);
            d = loss_deriv(loss, z, rvx<VT>(y, i));
        }
        for (int64_t e = lo + lane; e < hi; e += 32) atomicAdd(out + (int64_t)col[e] * os, d * rvx<VT>(val, e));
    }
}

__global__ void k_fill(double *out, int os, int64_t p, double v)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        out[j * os] = v;
}

// out = out / n + lambda1 * x   (losses.py:122)
__global__ void k_grad_finish(double *out, int os, const double *x, int xs, int64_t p, double n, double lambda1)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        double g = out[j * os] / n;
        out[j * os] = x ? g + lambda1 * x[j * xs] : g;
    }
}

static int rmatvec(const ps_csr_t *csr, int loss, const double *x, int xs, const double *s, double *out, int os,
                   cudaStream_t st)
{
    int grid = sm_count() * 8;
    k_fill<<<grid, 256, 0, st>>>(out, os, csr->n_cols, 0.0);
    bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
    int64_t n = csr->n_rows;
    if (f64 && i64) k_rmatvec_deriv<double, long long><<<grid, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, n, loss, x, xs, s, out, os);
    else if (f64) k_rmatvec_deriv<double, int><<<grid, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, n, loss, x, xs, s, out, os);
    else if (i64) k_rmatvec_deriv<float, long long><<<grid, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, n, loss, x, xs, s, out, os);
    else k_rmatvec_deriv<float, int><<<grid, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, n, loss, x, xs, s, out, os);
    CK(cudaGetLastError(), "rmatvec launch");
    return PS_OK;
}

extern "C" int ps_smooth_gradient(const ps_csr_t *csr, const ps_params_t *prm, const double *x, int32_t x_stride,
                                  double *grad, void *stream)
{
    NvtxRange nvtx_range("K4 ps_smooth_gradient");
    if (!csr || !prm || !x || !grad) return ps_fail(PS_EINVAL, "null argument");
    if (csr->n_rows < 1) return ps_fail(PS_EINVAL, "dataset is empty");
    cudaStream_t st = (cudaStream_t)stream;
    int r = rmatvec(csr, prm->loss, x, x_stride, nullptr, grad, 1, st);
    if (r) return r;
    k_grad_finish<<<sm_count() * 8, 256, 0, st>>>(grad, 1, x, x_stride, csr->n_cols, (double)csr->n_rows, prm->lambda1);
    CK(cudaGetLastError(), "ps_smooth_gradient launch");
    return PS_OK;
}

extern "C" int ps_resync_average(const ps_csr_t *csr, const double *alpha, double *coord, void *stream)
{
    NvtxRange nvtx_range("K4 ps_resync_average");
    if (!csr || !alpha || !coord) return ps_fail(PS_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    int r = rmatvec(csr, 0, nullptr, 0, alpha, coord + 1, 4, st);
    if (r) return r;
    k_grad_finish<<<sm_count() * 8, 256, 0, st>>>(coord + 1, 4, nullptr, 0, csr->n_cols, (double)csr->n_rows, 0.0);
    CK(cudaGetLastError(), "ps_resync_average launch");
    return PS_OK;
}

// fixed-point residual (saga.py:299-317)
__global__ void __launch_bounds__(256) k_fp_sep(const double *coord, const double *grad, int64_t p, int pen,
                                                double gamma, double lam2, double lo, double hi, double *parts)
{
    double acc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        double x = coord[4 * j], d = coord[4 * j + 2];
        double inner = x - gamma * d * grad[j];
        double z = prox_sep(pen, inner, gamma * d, lam2, lo, hi);
        double r = x - z;
        acc += r * r;
    }
    block_sum_store(acc, parts);
}

__global__ void __launch_bounds__(256) k_fp_group(const double *coord, const double *grad, int64_t p, int kind,
                                                  int G, int64_t nb, const int32_t *blk_ptr,
                                                  const int32_t *blk_coords, const double *bw, double gamma,
                                                  double lam2, double *parts)
{
    double acc = 0.0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int64_t q0, q1;
        if (kind == PS_PART_GENERAL) {
            q0 = blk_ptr[b];
            q1 = blk_ptr[b + 1];
        } else {
            int64_t g = kind == PS_PART_SINGLETON ? 1 : G;
            q0 = b * g;
            q1 = min((b + 1) * g, p);
        }
        double ss = 0.0;
        for (int64_t q = q0; q < q1; q++) {
            int64_t j = kind == PS_PART_GENERAL ? blk_coords[q] : q;
            double u = coord[4 * j] - gamma * coord[4 * j + 2] * grad[j];
            ss += u * u;
        }
        double f = group_factor(sqrt(ss), gamma * bw[b], lam2);
        for (int64_t q = q0; q < q1; q++) {
            int64_t j = kind == PS_PART_GENERAL ? blk_coords[q] : q;
            double x = coord[4 * j];
            double u = x - gamma * coord[4 * j + 2] * grad[j];
            double r = x - u * f;
            acc += r * r;
        }
    }
    block_sum_store(acc, parts);
}

// ---------------------------------------------------------------------------
// Fenchel dual objective (duality gap = primal - dual, SURVEY §8 "on-device
// objective and duality-gap evaluation").  No reference counterpart (parity
// unpinned; the oracle restates the same formulas in numpy).
//   P(x) = (1/n) sum_i l(a_i.x, b_i) + (lambda1/2)||x||^2 + h(x)
//   D(theta) = -(1/n) sum_i l*(-theta_i) - g*((1/n) A^T theta),  g = lambda1/2||.||^2 + h
// at the dual point induced by x: theta_i = -l'(a_i.x, b_i) (= -s_i), so
// v = (1/n) A^T theta = -(1/n) A^T s.  Conjugates:
//   logistic l*(s) = t log t + (1 - t) log(1 - t), t = -b s in [0, 1]; squared l*(s) = s^2/2 + s b;
//   lambda1 > 0: L1 sum (|v_j| - lam2)_+^2 / (2 lambda1); group sum_B (||v_B|| - lam2)_+^2 / (2 lambda1);
//                box sum v c - lambda1 c^2 / 2, c = clip(v / lambda1, lo, hi); zero sum v^2 / (2 lambda1);
//   lambda1 = 0: L1 / group: theta scaled by c = min(1, lam2 / max |v_j| (max ||v_B||)), g* = 0;
//                box: sum max(v lo, v hi); zero: 0 if v = 0 else +inf.
__device__ __forceinline__ double loss_conj(int loss, double s, double b)
{
    if (loss == PS_LOSS_LOGISTIC) {
        const double t = -b * s;
        double r = 0.0;
        if (t > 0.0) r += t * log(t);
        if (t < 1.0) r += (1.0 - t) * log1p(-t);
        return r;
    }
    return 0.5 * s * s + s * b;
}

__device__ __forceinline__ void atomic_max_nonneg(double *p, double v)
{
    atomicMax(reinterpret_cast<unsigned long long *>(p), (unsigned long long)__double_as_longlong(v));
}

// s_i = l'(a_i.x, b_i) into s[], sum of l*(s_i) per CTA (thread per row)
template <typename VT, typename PT>
__global__ void __launch_bounds__(256) k_dual_rows(const void *row_ptr, const int32_t *col, const void *val,
                                                   const void *y, int64_t n, int loss, const double *x, int xs,
                                                   double *s_out, double *parts)
{
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
        double z = 0.0;
        for (int64_t e = lo; e < hi; e++) z += rvx<VT>(val, e) * x[(int64_t)col[e] * xs];
        const double b = rvx<VT>(y, i);
        const double si = loss_deriv(loss, z, b);
        s_out[i] = si;
        acc += loss_conj(loss, si, b);
    }
    block_sum_store(acc, parts);
}

// w = A^T s (warp per row).  Columns below `head` (the Zipf head, where the
// hot layout also puts the staged columns) are summed in a per-CTA shared
// array first and flushed once per CTA: a plain global atomic scatter would
// queue ~n atomics on column 0's sector.
constexpr int DUAL_HEAD = 12288;  // 96 KB of shared memory
template <typename VT, typename PT>
__global__ void __launch_bounds__(512) k_dual_scatter(const void *row_ptr, const int32_t *col, const void *val,
                                                      int64_t n, int head, const double *s, double *w)
{
    extern __shared__ double acc_head[];
    for (int j = threadIdx.x; j < head; j += blockDim.x) acc_head[j] = 0.0;
    __syncthreads();
    int lane = threadIdx.x & 31;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
        const double si = s[i];
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int c = col[e];
            const double v = rvx<VT>(val, e) * si;
            if (c < head) atomicAdd(acc_head + c, v);
            else atomicAdd(w + c, v);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < head; j += blockDim.x)
        if (acc_head[j] != 0.0) atomicAdd(w + j, acc_head[j]);
}

__device__ __forceinline__ double gstar_sep(int pen, double v, double lambda1, double lam2, double lo, double hi)
{
    if (lambda1 > 0.0) {
        if (pen == PS_PEN_L1) {
            const double m = fmax(fabs(v) - lam2, 0.0);
            return m * m / (2.0 * lambda1);
        }
        if (pen == PS_PEN_BOX) {
            const double c = fmin(fmax(v / lambda1, lo), hi);
            return v * c - 0.5 * lambda1 * c * c;
        }
        return v * v / (2.0 * lambda1);  // zero penalty
    }
    if (pen == PS_PEN_BOX) return fmax(v * lo, v * hi);
    return 0.0;  // L1 (after scaling) / zero (checked through the max)
}

// separable penalties: g* partial sums and max |v_j|, v = -w / n
__global__ void __launch_bounds__(256) k_dual_coords(const double *w, int64_t p, double inv_n, int pen,
                                                     double lambda1, double lam2, double lo, double hi,
                                                     double *parts, double *vmax)
{
    double acc = 0.0, m = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        const double v = -w[j] * inv_n;
        acc += gstar_sep(pen, v, lambda1, lam2, lo, hi);
        m = fmax(m, fabs(v));
    }
    block_sum_store(acc, parts);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(vmax, m);
}

// group penalty: per block ||v_B||, g* partial sums and the max block norm
__global__ void __launch_bounds__(256) k_dual_blocks(const double *w, int64_t p, double inv_n, int kind, int G,
                                                     int64_t nb, const int32_t *blk_ptr, const int32_t *blk_coords,
                                                     double lambda1, double lam2, double *parts, double *vmax)
{
    double acc = 0.0, m = 0.0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        double ss = 0.0;
        if (kind == PS_PART_GENERAL) {
            for (int q = blk_ptr[b]; q < blk_ptr[b + 1]; q++) {
                const double v = w[blk_coords[q]] * inv_n;
                ss += v * v;
            }
        } else {
            const int64_t g = kind == PS_PART_SINGLETON ? 1 : G;
            for (int64_t j = b * g; j < min((b + 1) * g, p); j++) {
                const double v = w[j] * inv_n;
                ss += v * v;
            }
        }
        const double nrm = sqrt(ss);
        if (lambda1 > 0.0) {
            const double e = fmax(nrm - lam2, 0.0);
            acc += e * e / (2.0 * lambda1);
        }
        m = fmax(m, nrm);
    }
    block_sum_store(acc, parts);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(vmax, m);
}

// lambda1 = 0 with L1 / group: conjugate sum at the scaled point c s
template <typename VT>
__global__ void __launch_bounds__(256) k_dual_rows_scaled(const double *s, const void *y, int64_t n, int loss,
                                                          const double *vmax, double lam2, double *parts)
{
    const double c = vmax[0] > lam2 ? lam2 / vmax[0] : 1.0;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += loss_conj(loss, c * s[i], rvx<VT>(y, i));
    block_sum_store(acc, parts);
}

// out[0] = dual value, out[1] = the dual scaling c
__global__ void k_dual_combine(const double *sums, const double *vmax, double inv_n, double lambda1, int pen,
                               double lam2, double *out)
{
    double c = 1.0;
    if (lambda1 <= 0.0 && (pen == PS_PEN_L1 || pen == PS_PEN_GROUP) && vmax[0] > lam2) c = lam2 / vmax[0];
    double d = -inv_n * sums[0] - sums[1];
    if (lambda1 <= 0.0 && pen == PS_PEN_ZERO && vmax[0] > 0.0) d = -INFINITY;
    out[0] = d;
    out[1] = c;
}

extern "C" int ps_dual_objective(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm, const double *x,
                                 int32_t x_stride, double *out, void *stream)
{
    NvtxRange nvtx_range("K8 ps_dual_objective");
    if (!csr || !part || !prm || !x || !out) return ps_fail(PS_EINVAL, "null argument");
    if (csr->n_rows < 1) return ps_fail(PS_EINVAL, "dataset is empty");
    cudaStream_t st = (cudaStream_t)stream;
    const int G1 = std::max(1, sm_count() * 4);
    const int64_t n = csr->n_rows, p = csr->n_cols;
    double *buf = nullptr;
    const size_t nd = (size_t)n + (size_t)p + 2 * (size_t)G1 + 4;
    CK(pool_alloc((void **)&buf, sizeof(double) * nd, st), "ps_dual_objective alloc");
    double *s = buf, *w = buf + n, *parts = w + p, *sums = parts + 2 * G1, *vmax = sums + 2;
    CK(cudaMemsetAsync(w, 0, sizeof(double) * p, st), "ps_dual_objective memset");
    CK(cudaMemsetAsync(vmax, 0, sizeof(double), st), "ps_dual_objective memset");
    const bool f64 = csr->value_type == PS_F64, i64 = csr->row_ptr_type == PS_I64;
#define DUAL_ROWS(V, P) k_dual_rows<V, P><<<G1, 256, 0, st>>>(csr->row_ptr, csr->col_idx, csr->values, csr->labels, \
                                                             n, prm->loss, x, x_stride, s, parts)
    const int head = (int)std::min<int64_t>(p, DUAL_HEAD);
    const int Gs = sm_count();  // one 512-thread CTA per SM (96 KB of head accumulators each)
#define DUAL_SCATTER(V, P)                                                                                         \
    do {                                                                                                         \
        cudaFuncSetAttribute(k_dual_scatter<V, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, DUAL_HEAD * 8); \
        k_dual_scatter<V, P><<<Gs, 512, head * 8, st>>>(csr->row_ptr, csr->col_idx, csr->values, n, head, s, w); \
    } while (0)
    if (f64 && i64) { DUAL_ROWS(double, long long); DUAL_SCATTER(double, long long); }
    else if (f64) { DUAL_ROWS(double, int); DUAL_SCATTER(double, int); }
    else if (i64) { DUAL_ROWS(float, long long); DUAL_SCATTER(float, long long); }
    else { DUAL_ROWS(float, int); DUAL_SCATTER(float, int); }
#undef DUAL_ROWS
#undef DUAL_SCATTER
    const double inv_n = 1.0 / (double)n;
    if (prm->penalty == PS_PEN_GROUP) {
        const int64_t nb = part->kind == PS_PART_SINGLETON ? p : part->n_blocks;
        k_dual_blocks<<<G1, 256, 0, st>>>(w, p, inv_n, part->kind, part->G, nb, part->blk_ptr, part->blk_coords,
                                         prm->lambda1, prm->lam2, parts + G1, vmax);
    } else {
        k_dual_coords<<<G1, 256, 0, st>>>(w, p, inv_n, prm->penalty, prm->lambda1, prm->lam2, prm->lo, prm->hi,
                                         parts + G1, vmax);
    }
    if (prm->lambda1 <= 0.0 && (prm->penalty == PS_PEN_L1 || prm->penalty == PS_PEN_GROUP)) {
        if (f64) k_dual_rows_scaled<double><<<G1, 256, 0, st>>>(s, csr->labels, n, prm->loss, vmax, prm->lam2, parts);
        else k_dual_rows_scaled<float><<<G1, 256, 0, st>>>(s, csr->labels, n, prm->loss, vmax, prm->lam2, parts);
    }
    k_finish_sum<<<1, 256, 0, st>>>(parts, G1, 2, sums, 1.0);
    k_dual_combine<<<1, 1, 0, st>>>(sums, vmax, inv_n, prm->lambda1, prm->penalty, prm->lam2, out);
    CK(cudaGetLastError(), "ps_dual_objective launch");
    CK(cudaFreeAsync(buf, st), "ps_dual_objective free");
    return PS_OK;
}

__global__ void k_sqrt(double *v) { v[0] = sqrt(v[0]); }

extern "C" int ps_fixed_point_residual(const ps_csr_t *csr, const ps_part_t *part, const ps_params_t *prm,
                                       const double *coord, double *grad, double *out, void *stream)
{
    NvtxRange nvtx_range("K4 ps_fixed_point_residual");
    if (!csr || !part || !prm || !coord || !grad || !out) return ps_fail(PS_EINVAL, "null argument");
    if (!(prm->gamma > 0)) return ps_fail(PS_EINVAL, "gamma must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    int r = ps_smooth_gradient(csr, prm, coord, 4, grad, stream);
    if (r) return r;
    const int G1 = std::max(1, sm_count() * 4);
    double *parts = nullptr;
    CK(pool_alloc((void **)&parts, sizeof(double) * G1, st), "ps_fixed_point_residual alloc");
    if (prm->penalty == PS_PEN_GROUP) {
        int64_t nb = part->kind == PS_PART_SINGLETON ? csr->n_cols : part->n_blocks;
        k_fp_group<<<G1, 256, 0, st>>>(coord, grad, csr->n_cols, part->kind, part->G, nb, part->blk_ptr,
                                       part->blk_coords, part->blk_weight, prm->gamma, prm->lam2, parts);
    } else {
        k_fp_sep<<<G1, 256, 0, st>>>(coord, grad, csr->n_cols, prm->penalty, prm->gamma, prm->lam2, prm->lo, prm->hi,
                                     parts);
    }
    k_finish_sum<<<1, 256, 0, st>>>(parts, G1, 1, out, 1.0);
    k_sqrt<<<1, 1, 0, st>>>(out);
    CK(cudaGetLastError(), "ps_fixed_point_residual launch");
    CK(cudaFreeAsync(parts, st), "ps_fixed_point_residual free");
    return PS_OK;
}

// ---------------------------------------------------------------------------
// standalone prox (penalty API)
__global__ void k_prox_sep(int pen, const double *v, const double *eff, int64_t m, double lam2, double lo, double hi,
                           double *out)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = prox_sep(pen, v[q], eff[q], lam2, lo, hi);
}

__global__ void __launch_bounds__(256) k_prox_group(const double *v, const double *eff, int64_t m, double lam2,
                                                    double *out)
{
    double ss = 0.0;
    for (int64_t q = threadIdx.x; q < m; q += blockDim.x) ss += v[q] * v[q];
    __shared__ double red[8];
    __shared__ double tot;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
        tot = s;
    }
    __syncthreads();
    double f = group_factor(sqrt(tot), eff[0], lam2);
    for (int64_t q = threadIdx.x; q < m; q += blockDim.x) out[q] = v[q] * f;
}

// ---------------------------------------------------------------------------
// FISTA (fista.py:38-58): the prox-gradient trial point
// x+ = prox_{h/L}(y - grad/L) over the whole vector (separable penalties per
// coordinate, the group penalty per block of the partition) together with
// grad.(x+ - y) and ||x+ - y||^2 for the backtracking test (per-CTA partials,
// last CTA sums in a fixed order); and the extrapolation y' = x+ + beta (x+ - x).
__global__ void __launch_bounds__(256) k_fista_prox(int kind, int G, int64_t nb, const int32_t *blk_ptr,
                                                    const int32_t *blk_coords, int pen, double lam2, double lo,
                                                    double hi, const double *y, const double *grad, double inv_L,
                                                    int64_t p, double *xn, double *parts, unsigned *done,
                                                    double *sums)
{
    double gd = 0.0, dd = 0.0;
    if (pen != PS_PEN_GROUP) {
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
            const double u = y[j] - grad[j] * inv_L;
            const double z = prox_sep(pen, u, inv_L, lam2, lo, hi);
            const double df = z - y[j];
            xn[j] = z;
            gd += grad[j] * df;
            dd += df * df;
        }
    } else {
        for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
            int64_t q0, q1, g = 1;
            if (kind == PS_PART_GENERAL) {
                q0 = blk_ptr[b];
                q1 = blk_ptr[b + 1];
            } else {
                g = kind == PS_PART_SINGLETON ? 1 : G;
                q0 = b * g;
                q1 = min((b + 1) * g, p);
            }
            double ss = 0.0;
            for (int64_t q = q0; q < q1; q++) {
                const int64_t j = kind == PS_PART_GENERAL ? blk_coords[q] : q;
                const double u = y[j] - grad[j] * inv_L;
                ss += u * u;
            }
            const double f = group_factor(sqrt(ss), inv_L, lam2);
            for (int64_t q = q0; q < q1; q++) {
                const int64_t j = kind == PS_PART_GENERAL ? blk_coords[q] : q;
                const double z = (y[j] - grad[j] * inv_L) * f;
                const double df = z - y[j];
                xn[j] = z;
                gd += grad[j] * df;
                dd += df * df;
            }
        }
    }
    const int G1 = gridDim.x;
    block_sum_store(gd, parts);
    block_sum_store(dd, parts + G1);
    __shared__ bool last;
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == (unsigned)gridDim.x - 1u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int c = 0; c < 2; c++) {
        double v = 0.0;
        for (int q = threadIdx.x; q < G1; q += blockDim.x) v += ld_cg(parts + (int64_t)c * G1 + q);
        __shared__ double red[8];
        v = warp_sum(v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
            sums[c] = t;
        }
        __syncthreads();
    }
}

__global__ void k_fista_extrapolate(const double *xn, const double *x, double beta, int64_t p, double *y)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        y[j] = xn[j] + beta * (xn[j] - x[j]);
}

extern "C" int ps_fista_prox(const ps_part_t *part, const ps_params_t *prm, const double *y, const double *grad,
                             double inv_L, int64_t p, double *x_new, double *sums, void *stream)
{
    if (!part || !prm || !y || !grad || !x_new || !sums || p < 1) return ps_fail(PS_EINVAL, "bad fista arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int G1 = std::max(1, sm_count() * 4);
    double *parts = nullptr;
    CK(pool_alloc((void **)&parts, sizeof(double) * (2 * G1 + 1), st), "ps_fista_prox alloc");
    unsigned *done = reinterpret_cast<unsigned *>(parts + 2 * G1);
    CK(cudaMemsetAsync(done, 0, sizeof(unsigned), st), "ps_fista_prox memset");
    const int64_t nb = part->kind == PS_PART_SINGLETON ? p : part->n_blocks;
    k_fista_prox<<<G1, 256, 0, st>>>(part->kind, part->G, nb, part->blk_ptr, part->blk_coords, prm->penalty,
                                     prm->lam2, prm->lo, prm->hi, y, grad, inv_L, p, x_new, parts, done, sums);
    CK(cudaGetLastError(), "ps_fista_prox launch");
    CK(cudaFreeAsync(parts, st), "ps_fista_prox free");
    return PS_OK;
}

extern "C" int ps_fista_extrapolate(const double *x_new, const double *x, double beta, int64_t p, double *y,
                                    void *stream)
{
    if (!x_new || !x || !y || p < 1) return ps_fail(PS_EINVAL, "bad fista arguments");
    k_fista_extrapolate<<<(int)std::min<int64_t>((p + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(x_new, x,
                                                                                                          beta, p, y);
    CK(cudaGetLastError(), "ps_fista_extrapolate launch");
    return PS_OK;
}

extern "C" int ps_prox(const ps_params_t *prm, const double *v, const double *eff, int64_t m, double *out,
                       void *stream)
{
    if (!prm || !v || !eff || !out) return ps_fail(PS_EINVAL, "null argument");
    if (m <= 0) return PS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (prm->penalty == PS_PEN_GROUP) k_prox_group<<<1, 256, 0, st>>>(v, eff, m, prm->lam2, out);
    else k_prox_sep<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(prm->penalty, v, eff, m, prm->lam2,
                                                                                     prm->lo, prm->hi, out);
    CK(cudaGetLastError(), "ps_prox launch");
    return PS_OK;
}

// ---------------------------------------------------------------------------
__global__ void k_coord_get(const double *coord, int64_t p, int f, double *out)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = coord[4 * j + f];
}
__global__ void k_coord_set(double *coord, int64_t p, int f, const double *in)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        coord[4 * j + f] = in ? in[j] : 0.0;
}

extern "C" int ps_coord_get(const double *coord, int64_t p, int32_t field, double *out, void *stream)
{
    if (!coord || !out || field < 0 || field > 3) return ps_fail(PS_EINVAL, "bad argument");
    if (p <= 0) return PS_OK;
    k_coord_get<<<(int)std::min<int64_t>((p + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(coord, p, field, out);
    CK(cudaGetLastError(), "ps_coord_get launch");
    return PS_OK;
}

extern "C" int ps_coord_set(double *coord, int64_t p, int32_t field, const double *in, void *stream)
{
    if (!coord || field < 0 || field > 3) return ps_fail(PS_EINVAL, "bad argument");
    if (p <= 0) return PS_OK;
    k_coord_set<<<(int)std::min<int64_t>((p + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(coord, p, field, in);
    CK(cudaGetLastError(), "ps_coord_set launch");
    return PS_OK;
}

// x0 = 0, abar = 0 (D kept), alpha = 0, counter = 0 in one launch
// (saga.py:231-232 / PAPER.md:1195-1199).
__global__ void k_state_reset(double *coord, int64_t p, double *alpha, int64_t n, unsigned long long *counter)
{
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t j = t0; j < p; j += stride) {
        double2 z = make_double2(0.0, 0.0);
        *reinterpret_cast<double2 *>(coord + 4 * j) = z;
    }
    for (int64_t i = t0; i < n; i += stride) alpha[i] = 0.0;
    if (t0 == 0 && counter) *counter = 0ull;
}

extern "C" int ps_state_reset(double *coord, int64_t p, double *alpha, int64_t n, unsigned long long *counter,
                              void *stream)
{
    if (!coord || !alpha) return ps_fail(PS_EINVAL, "null argument");
    int64_t m = std::max(p, n);
    k_state_reset<<<(int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, sm_count() * 8)), 256, 0,
                    (cudaStream_t)stream>>>(coord, p, alpha, n, counter);
    CK(cudaGetLastError(), "ps_state_reset launch");
    return PS_OK;
}

// device timestamp (%globaltimer, ns) into *dst: stream-ordered and capturable,
// so checkpoint times can be taken inside a CUDA graph (events recorded during
// capture cannot be used for elapsed-time queries)
__global__ void k_timestamp(unsigned long long *dst)
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
}

extern "C" int ps_timestamp(unsigned long long *dst, void *stream)
{
    if (!dst) return ps_fail(PS_EINVAL, "null argument");
    k_timestamp<<<1, 1, 0, (cudaStream_t)stream>>>(dst);
    CK(cudaGetLastError(), "ps_timestamp launch");
    return PS_OK;
}

// ---------------------------------------------------------------------------
// Hot-column layout (singleton partitions): the columns appearing in at least
// max(min_frac * n, theta) rows, theta chosen so at most hot_max qualify, are
// renumbered [0, H) (in original order), the rest [H, p) (in original order),
// and the CSR column indices are remapped in place.  The SPS kernel then
// recognises a hot column by `col < H` without any load and stages it in
// shared memory (SURVEY.md §7.3 "hot-column atomic contention").

__global__ void k_count_ge(const int32_t *counts, int64_t p, int theta, unsigned long long *out)
{
    unsigned long long c = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        c += counts[j] >= theta;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// append the counts >= lo (candidate hot units) to out[0..*m)
__global__ void k_collect_ge(const int32_t *counts, int64_t nu, int lo, int32_t *out, unsigned long long *m,
                             int64_t cap)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nu; j += (int64_t)gridDim.x * blockDim.x) {
        int c = counts[j];
        if (c >= lo) {
            unsigned long long s = atomicAdd(m, 1ull);
            if ((int64_t)s < cap) out[s] = c;
        }
    }
}

// chunked exclusive scan of hot flags: pass 1 per-CTA sums
__global__ void k_flag_sums(const int32_t *counts, int64_t p, int theta, int64_t chunk, int64_t *sums)
{
    int64_t lo = blockIdx.x * chunk, hi = min(lo + chunk, p);
    int64_t c = 0;
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) c += counts[j] >= theta;
    __shared__ int64_t red[32];
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
        sums[blockIdx.x] = t;
    }
}

// exclusive scan of nb per-chunk sums, one CTA (warp-shuffle scan per 1024 block)
__global__ void k_scan_small(int64_t *sums, int nb)
{
    __shared__ int64_t wsum[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += blockDim.x) {
        int b = base + threadIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int64_t v = b < nb ? sums[b] : 0, x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(FULL, t, o);
                if (lane >= o) t += y;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        int64_t incl = x + (w > 0 ? wsum[w - 1] : 0);
        if (b < nb) sums[b] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += incl;
        __syncthreads();
    }
}

// stored index of the c-th cold column when hot ranks r sit at r * S
__device__ __forceinline__ int64_t cold_pos(int64_t c, int64_t H, int64_t S)
{
    if (S == 1) return H + c;
    int64_t gaps = (S - 1) * H;
    if (c < gaps) return (c / (S - 1)) * S + 1 + (c % (S - 1));
    return S * H + (c - gaps);
}

// pass 3: serial-within-CTA rescan (one warp ballot per 32 columns) -> perm
__global__ void k_perm(const int32_t *counts, int64_t p, int theta, int64_t chunk, const int64_t *offs, int H,
                       int S, int32_t *perm, int32_t *inv)
{
    if (threadIdx.x >= 32) return;
    int lane = threadIdx.x;
    int64_t lo = blockIdx.x * chunk, hi = min(lo + chunk, p);
    int64_t hot_before = offs[blockIdx.x];
    for (int64_t base = lo; base < hi; base += 32) {
        int64_t j = base + lane;
        bool hot = j < hi && counts[j] >= theta;
        unsigned bal = __ballot_sync(FULL, hot);
        int64_t r = hot_before + __popc(bal & ((1u << lane) - 1u));
        if (j < hi) {
            int64_t nj = hot ? r * S : cold_pos(j - r, H, S);
            perm[j] = (int32_t)nj;
            inv[nj] = (int32_t)j;
        }
        hot_before += __popc(bal);
    }
}

__global__ void k_remap_cols(int32_t *col, int64_t nnz, const int32_t *perm)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        col[e] = perm[col[e]];
}

// distinct rows per unit (unit = 1: column counts; unit = G: block counts n_B).
// Rows may be unsorted: a unit is counted at its first occurrence in the row.
template <typename PT>
__global__ void k_count_units(const void *row_ptr, const int32_t *col, int64_t n, int unit, int32_t *counts)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
    for (int64_t e = lo; e < hi; e++) {
        int u = col[e] / unit;
        bool first = true;
        if (unit > 1)
            for (int64_t f = lo; f < e && first; f++) first = (col[f] / unit) != u;
        if (first) atomicAdd(counts + u, 1);
    }
}

// coordinate permutation from the unit permutation: c -> perm_u[c / unit] * unit + c % unit
__global__ void k_coord_perm(const int32_t *perm_u, int64_t p, int unit, int32_t *perm)
{
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < p; c += (int64_t)gridDim.x * blockDim.x)
        perm[c] = (int32_t)((int64_t)perm_u[c / unit] * unit + c % unit);
}

// restore strictly increasing columns per row after the remap (values move along):
// warp bitonic sort for rows of <= 32 nonzeros, one-lane insertion sort otherwise
template <typename VT, typename PT>
__global__ void k_sort_rows(const void *row_ptr, int32_t *col, void *valp, int64_t n)
{
    VT *val = reinterpret_cast<VT *>(valp);
    int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
        int64_t lo = rpx<PT>(row_ptr, i), hi = rpx<PT>(row_ptr, i + 1);
        int k = (int)(hi - lo);
        if (k <= 1) continue;
        if (k <= 32) {
            int c = lane < k ? col[lo + lane] : INT_MAX;
            VT v = lane < k ? val[lo + lane] : VT(0);
            for (int size = 2; size <= 32; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    int oc = __shfl_xor_sync(FULL, c, stride);
                    VT ov = __shfl_xor_sync(FULL, v, stride);
                    bool up = ((lane & size) == 0);
                    bool lower = (lane & stride) == 0;
                    bool take = lower ? (up ? oc < c : oc > c) : (up ? oc > c : oc < c);
                    if (take) {
                        c = oc;
                        v = ov;
                    }
                }
            }
            if (lane < k) {
                col[lo + lane] = c;
                val[lo + lane] = v;
            }
        } else if (lane == 0) {
            for (int64_t e = lo + 1; e < hi; e++) {
                int c = col[e];
                VT v = val[e];
                int64_t f = e - 1;
                while (f >= lo && col[f] > c) {
                    col[f + 1] = col[f];
                    val[f + 1] = val[f];
                    f--;
                }
                col[f + 1] = c;
                val[f + 1] = v;
            }
        }
    }
}

extern "C" int ps_hot_layout(const ps_csr_t *csr, int32_t *col_inout, void *val_inout, int32_t unit,
                             int32_t hot_max, double min_frac, int32_t *stride_inout, int32_t *counts_ws,
                             int32_t *perm, int32_t *H_out, int64_t *p_pad_out, void *stream)
{
    if (!csr || !col_inout || !val_inout || !counts_ws || !perm || !H_out || !stride_inout || !p_pad_out)
        return ps_fail(PS_EINVAL, "null argument");
    if (unit < 1) return ps_fail(PS_EINVAL, "unit must be >= 1");
    if (*stride_inout < 1 || (*stride_inout & (*stride_inout - 1)))
        return ps_fail(PS_EINVAL, "stride must be a power of two");
    if (hot_max < 0) return ps_fail(PS_EINVAL, "hot_max must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t p = csr->n_cols, n = csr->n_rows, nnz = csr->nnz;
    const int64_t nu = (p + unit - 1) / unit;
    const bool i64 = csr->row_ptr_type == PS_I64, f64 = csr->value_type == PS_F64;
    int grid = sm_count() * 8;
    int rows_grid = (int)((n + 255) / 256);
    CK(cudaMemsetAsync(counts_ws, 0, sizeof(int32_t) * nu, st), "ps_hot_layout memset");
    if (nnz > 0) {
        if (unit == 1) count_cols(col_inout, nnz, p, counts_ws, sm_count(), st);
        else if (i64) k_count_units<long long><<<rows_grid, 256, 0, st>>>(csr->row_ptr, col_inout, n, unit, counts_ws);
        else k_count_units<int><<<rows_grid, 256, 0, st>>>(csr->row_ptr, col_inout, n, unit, counts_ws);
    }
    // threshold: the smallest theta >= lo = max(1, ceil(min_frac * n)) with at
    // most hot_max units at or above it.  Candidates (count >= lo) are compacted
    // on the device; the host picks the (hot_max+1)-th largest from them.
    const int lo = std::max(1, (int)std::ceil(min_frac * (double)n));
    unsigned long long *cnt = nullptr;
    int32_t *cand = nullptr;
    const int64_t cap = std::min<int64_t>(nu, 1 << 24);
    CK(pool_alloc((void **)&cnt, sizeof(unsigned long long), st), "ps_hot_layout alloc");
    CK(pool_alloc((void **)&cand, sizeof(int32_t) * std::max<int64_t>(cap, 1), st), "ps_hot_layout alloc");
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st), "ps_hot_layout memset");
    k_collect_ge<<<grid, 256, 0, st>>>(counts_ws, nu, lo, cand, cnt, cap);
    unsigned long long m = 0;
    CK(cudaMemcpyAsync(&m, cnt, sizeof(m), cudaMemcpyDeviceToHost, st), "ps_hot_layout copy");
    CK(cudaStreamSynchronize(st), "ps_hot_layout sync");
    int theta = lo;
    int H = (int)std::min<unsigned long long>(m, (unsigned long long)cap);
    if ((int64_t)m > cap) return ps_fail(PS_EINVAL, "too many hot candidates; raise min_frac");
    if (m > (unsigned long long)hot_max) {
        std::vector<int32_t> hv(m);
        CK(cudaMemcpyAsync(hv.data(), cand, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st), "ps_hot_layout copy");
        CK(cudaStreamSynchronize(st), "ps_hot_layout sync");
        std::nth_element(hv.begin(), hv.begin() + hot_max, hv.end(), std::greater<int32_t>());
        theta = hv[hot_max] + 1;  // strictly above the (hot_max+1)-th largest count
        H = 0;
        for (int32_t v : hv) H += v >= theta;
    }
    CK(cudaFreeAsync(cand, st), "ps_hot_layout free");
    int S = *stride_inout;
    while (S > 1 && (int64_t)S * H > nu) S >>= 1;  // hot units at 0, S, 2S, ... (unit indices)
    const int64_t chunk = 1 << 10;  // one warp per chunk in k_perm: enough chunks to fill the GPU
    int nb = (int)((nu + chunk - 1) / chunk);
    int64_t *sums = nullptr;
    int32_t *perm_u = nullptr, *inv_u = nullptr;
    CK(pool_alloc((void **)&sums, sizeof(int64_t) * std::max(nb, 1), st), "ps_hot_layout alloc");
    CK(pool_alloc((void **)&perm_u, sizeof(int32_t) * std::max<int64_t>(nu, 1) * 2, st), "ps_hot_layout alloc");
    inv_u = perm_u + nu;
    k_flag_sums<<<nb, 256, 0, st>>>(counts_ws, nu, theta, chunk, sums);
    k_scan_small<<<1, 1024, 0, st>>>(sums, nb);
    k_perm<<<nb, 32, 0, st>>>(counts_ws, nu, theta, chunk, sums, H, S, perm_u, inv_u);
    k_coord_perm<<<grid, 256, 0, st>>>(perm_u, p, unit, perm);
    if (nnz > 0) {
        k_remap_cols<<<grid, 256, 0, st>>>(col_inout, nnz, perm);
        if (f64 && i64) k_sort_rows<double, long long><<<grid, 256, 0, st>>>(csr->row_ptr, col_inout, val_inout, n);
        else if (f64) k_sort_rows<double, int><<<grid, 256, 0, st>>>(csr->row_ptr, col_inout, val_inout, n);
        else if (i64) k_sort_rows<float, long long><<<grid, 256, 0, st>>>(csr->row_ptr, col_inout, val_inout, n);
        else k_sort_rows<float, int><<<grid, 256, 0, st>>>(csr->row_ptr, col_inout, val_inout, n);
    }
    CK(cudaGetLastError(), "ps_hot_layout launch");
    CK(cudaFreeAsync(perm_u, st), "ps_hot_layout free");
    CK(cudaFreeAsync(sums, st), "ps_hot_layout free");
    CK(cudaFreeAsync(cnt, st), "ps_hot_layout free");
    // no final synchronize: the permutation, remap and row sort are stream-ordered
    // before any later use of col / val / perm on this stream
    *H_out = H;
    *stride_inout = S;
    *p_pad_out = nu * unit;
    return PS_OK;
}

// out[j] = coord[4 * perm[j] + f]  (perm: original -> stored index)
__global__ void k_coord_get_perm(const double *coord, int64_t p, int f, const int32_t *perm, double *out)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = coord[4 * (int64_t)perm[j] + f];
}
__global__ void k_coord_set_perm(double *coord, int64_t p, int f, const int32_t *perm, const double *in)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x)
        coord[4 * (int64_t)perm[j] + f] = in[j];
}

extern "C" int ps_coord_get_perm(const double *coord, int64_t p, int32_t field, const int32_t *perm, double *out,
                                 void *stream)
{
    if (!coord || !out || !perm || field < 0 || field > 3) return ps_fail(PS_EINVAL, "bad argument");
    if (p <= 0) return PS_OK;
    k_coord_get_perm<<<(int)std::min<int64_t>((p + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(coord, p, field,
                                                                                                  perm, out);
    CK(cudaGetLastError(), "ps_coord_get_perm launch");
    return PS_OK;
}

extern "C" int ps_coord_set_perm(double *coord, int64_t p, int32_t field, const int32_t *perm, const double *in,
                                 void *stream)
{
    if (!coord || !in || !perm || field < 0 || field > 3) return ps_fail(PS_EINVAL, "bad argument");
    if (p <= 0) return PS_OK;
    k_coord_set_perm<<<(int)std::min<int64_t>((p + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(coord, p, field,
                                                                                                  perm, in);
    CK(cudaGetLastError(), "ps_coord_set_perm launch");
    return PS_OK;
}

// ---------------------------------------------------------------------------
// _atomics primitives
__global__ void k_check_idx(const int64_t *idx, int64_t m, int64_t len, int *bad)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        if (idx[q] < 0 || idx[q] >= len) atomicOr(bad, 1);
}
__global__ void k_gather(const double *arr, const int64_t *idx, int64_t m, double *out)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = ld_cg(arr + idx[q]);
}
__global__ void k_scatter_add(double *arr, const int64_t *idx, int64_t m, const double *d)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(arr + idx[q], d[q]);
}
__global__ void k_exchange(double *arr, const int64_t *idx, int64_t m, const double *val, double *old)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
        old[q] = atomic_exch(arr + idx[q], val[q]);
}
__global__ void k_fetch_add(long long *arr, int64_t i, long long delta, long long *old)
{
    *old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(arr + i), (unsigned long long)delta);
}
__global__ void k_add_repeat(double *cell, double delta, int64_t count)
{
    for (int64_t k = 0; k < count; k++) atomicAdd(cell, delta);
}

static int check_indices(const int64_t *idx, int64_t m, int64_t len, cudaStream_t st)
{
    if (m <= 0) return PS_OK;
    int *bad = nullptr, hbad = 0;
    CK(pool_alloc((void **)&bad, sizeof(int), st), "check alloc");
    CK(cudaMemsetAsync(bad, 0, sizeof(int), st), "check memset");
    k_check_idx<<<(int)std::min<int64_t>((m + 255) / 256, 4096), 256, 0, st>>>(idx, m, len, bad);
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "check readback");
    CK(cudaFreeAsync(bad, st), "check free");
    CK(cudaStreamSynchronize(st), "check sync");
    if (hbad) return ps_fail(PS_ERANGE, "cell index out of range");
    return PS_OK;
}

static inline int grid_for(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 4096)); }

extern "C" int ps_atomic_gather(const double *arr, int64_t len, const int64_t *idx, int64_t m, double *out,
                                void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    int r = check_indices(idx, m, len, st);
    if (r) return r;
    if (m > 0) k_gather<<<grid_for(m), 256, 0, st>>>(arr, idx, m, out);
    CK(cudaGetLastError(), "ps_atomic_gather");
    return PS_OK;
}

extern "C" int ps_atomic_scatter_add(double *arr, int64_t len, const int64_t *idx, int64_t m, const double *d,
                                     void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    int r = check_indices(idx, m, len, st);
    if (r) return r;
    if (m > 0) k_scatter_add<<<grid_for(m), 256, 0, st>>>(arr, idx, m, d);
    CK(cudaGetLastError(), "ps_atomic_scatter_add");
    return PS_OK;
}

extern "C" int ps_atomic_exchange(double *arr, int64_t len, const int64_t *idx, int64_t m, const double *val,
                                  double *old, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    int r = check_indices(idx, m, len, st);
    if (r) return r;
    if (m > 0) k_exchange<<<grid_for(m), 256, 0, st>>>(arr, idx, m, val, old);
    CK(cudaGetLastError(), "ps_atomic_exchange");
    return PS_OK;
}

extern "C" int ps_atomic_fetch_add_i64(long long *arr, int64_t len, int64_t i, long long delta, long long *old,
                                       void *stream)
{
    if (i < 0 || i >= len) return ps_fail(PS_ERANGE, "cell index out of range");
    k_fetch_add<<<1, 1, 0, (cudaStream_t)stream>>>(arr, i, delta, old);
    CK(cudaGetLastError(), "ps_atomic_fetch_add_i64");
    return PS_OK;
}

extern "C" int ps_atomic_add_repeat(double *cell, double delta, int64_t count, int32_t threads, void *stream)
{
    if (!cell || threads < 1 || count < 0) return ps_fail(PS_EINVAL, "bad argument");
    int tb = std::min(threads, 256);
    int grid = (threads + tb - 1) / tb;
    if (grid * tb != threads) return ps_fail(PS_EINVAL, "threads must be <= 256 or a multiple of 256");
    k_add_repeat<<<grid, tb, 0, (cudaStream_t)stream>>>(cell, delta, count);
    CK(cudaGetLastError(), "ps_atomic_add_repeat");
    return PS_OK;
}
