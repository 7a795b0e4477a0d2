// LibSVM text -> CSR on the device ("LibSVM ingestion
// to device CSR ... a GPU/parallel parser removes the host bottleneck").
//
// Semantics are those of the reference's parse_libsvm (data.py:309-363): one
// sample per line, "label idx:val ..." with 1-based strictly increasing
// indices, everything after '#' ignored, blank lines skipped, str.split()
// whitespace, float() / int() number syntax.  The device handles every line
// whose numbers it can convert exactly:
//   * indices: an optional sign and up to 18 decimal digits;
//   * label / values: [sign] digits [. digits] [e|E [sign] digits] with at
//     most 19 significant digits, converted to the correctly rounded double
//     (what float() returns): M * 10^E or M / 10^-E of two exact doubles when
//     M < 2^53 and |E| <= 22 (Clinger), else Eisel-Lemire with the 128-bit
//     powers of five of pow5_table.h (tools/gen_pow5.py).
// A line with any other number (more digits, inf/nan, underscores, subnormal
// or overflowing values) is flagged "host" and the caller parses that line
// with the reference semantics; definite errors (a token without ':', a
// non-increasing index) are reported with the byte offset / index so the
// caller raises the same ParseError the reference would, at the first
// offending line.
#include <cstdint>

#include "common.cuh"
#include "internal.h"
#include "pow5_table.h"

using namespace ps;

namespace {

enum : int32_t { LS_OK = 0, LS_BLANK = 1, LS_NO_COLON = 3, LS_NONINC = 4, LS_HOST = 5 };

__device__ __forceinline__ bool is_ws(uint8_t c)
{
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f);
}

__constant__ double k_pow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                   1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// Eisel-Lemire (Lemire, "Number Parsing at a Gigabyte per Second", 2021;
// the 128-bit power-of-five product suffices for <= 19 significant digits,
// Mushtak & Lemire 2023): the correctly rounded double of w * 10^q, or false
// for subnormal / overflowing results (left to the host).
__device__ bool eisel_lemire(int64_t q, uint64_t w, double &out)
{
    if (w == 0 || q < POW5_MIN_Q) {
        out = 0.0;
        return true;
    }
    if (q > POW5_MAX_Q) return false;
    const int lz = __clzll((long long)w);
    w <<= lz;
    const int idx = 2 * (int)(q - POW5_MIN_Q);
    const uint64_t t_hi = __ldg(k_pow5_128 + idx), t_lo = __ldg(k_pow5_128 + idx + 1);
    uint64_t hi = __umul64hi(w, t_hi), lo = w * t_hi;
    if ((hi & 0x1FF) == 0x1FF) {
        const uint64_t s_hi = __umul64hi(w, t_lo);
        lo += s_hi;
        if (s_hi > lo) hi++;
    }
    const int upper = (int)(hi >> 63);
    const int shift = upper + 9;
    uint64_t mant = hi >> shift;
    int64_t p2 = (((152170 + 65536) * q) >> 16) + 63 + upper - lz + 1023;
    if (p2 <= 0) return false;
    if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 && (mant << shift) == hi) mant &= ~1ull;
    mant += mant & 1;
    mant >>= 1;
    if (mant >= (2ull << 52)) {
        mant = 1ull << 52;
        p2++;
    }
    mant &= ~(1ull << 52);
    if (p2 >= 2047) return false;
    out = __longlong_as_double((long long)(((uint64_t)p2 << 52) | mant));
    return true;
}

// float() on [b, e): decimal syntax with at most 19 significant digits,
// converted exactly (Clinger's one-operation path when it applies, else
// Eisel-Lemire); false -> the host decides (other syntax, more digits,
// subnormal or overflowing values)
__device__ bool parse_float_fast(const uint8_t *b, const uint8_t *e, double &out)
{
    const uint8_t *p = b;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    uint64_t m = 0;
    int sig = 0, frac = 0, digits = 0;
    bool dot = false;
    for (; p < e; p++) {
        const uint8_t c = *p;
        if (c >= '0' && c <= '9') {
            digits++;
            if (m == 0 && c == '0') {
                if (dot) frac++;  // leading zeros after the point shift the exponent only
                continue;
            }
            if (++sig > 19) return false;
            m = m * 10 + (c - '0');
            if (dot) frac++;
        } else if (c == '.' && !dot) {
            dot = true;
        } else {
            break;
        }
    }
    if (digits == 0) return false;
    int ex = 0;
    if (p < e && (*p == 'e' || *p == 'E')) {
        p++;
        bool eneg = false;
        if (p < e && (*p == '+' || *p == '-')) eneg = *p++ == '-';
        int ed = 0;
        for (; p < e && *p >= '0' && *p <= '9'; p++) {
            if (++ed > 4) return false;
            ex = ex * 10 + (*p - '0');
        }
        if (ed == 0) return false;
        if (eneg) ex = -ex;
    }
    if (p != e) return false;
    const int E = ex - frac;
    double v;
    if (m == 0) {
        v = 0.0;
    } else if (m < (1ull << 53) && E >= -22 && E <= 22) {
        v = E >= 0 ? (double)m * k_pow10[E] : (double)m / k_pow10[-E];  // exact operands, one rounding
    } else if (!eisel_lemire(E, m, v)) {
        return false;
    }
    out = neg ? -v : v;
    return true;
}

// int() on [b, e): sign + up to 18 digits; false -> the host decides
__device__ bool parse_int_fast(const uint8_t *b, const uint8_t *e, int64_t &out)
{
    const uint8_t *p = b;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p == e || e - p > 18) return false;
    int64_t v = 0;
    for (; p < e; p++) {
        if (*p < '0' || *p > '9') return false;
        v = v * 10 + (*p - '0');
    }
    out = neg ? -v : v;
    return true;
}

// per line: label, feature count, status, detail (bad token offset or index)
__global__ void k_libsvm_scan(const uint8_t *buf, int64_t n, const int64_t *ls, int64_t m, double *labels,
                              int32_t *nfeat, int32_t *status, int64_t *detail, unsigned long long *max_idx)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t *p = buf + ls[j];
        const uint8_t *end = buf + (j + 1 < m ? ls[j + 1] : n);
        const uint8_t *hash = p;
        while (hash < end && *hash != '#' && *hash != '\n') hash++;
        end = hash;
        while (p < end && is_ws(*p)) p++;
        int32_t st = LS_OK, cnt = 0;
        int64_t det = 0, prev = 0, mx = 0;
        double lab = 0.0;
        if (p == end) {
            st = LS_BLANK;
        } else {
            const uint8_t *t = p;
            while (t < end && !is_ws(*t)) t++;
            if (!parse_float_fast(p, t, lab)) st = LS_HOST;
            p = t;
            while (st == LS_OK) {
                while (p < end && is_ws(*p)) p++;
                if (p == end) break;
                const uint8_t *te = p;
                while (te < end && !is_ws(*te)) te++;
                const uint8_t *colon = p;
                while (colon < te && *colon != ':') colon++;
                if (colon == te) {
                    st = LS_NO_COLON;
                    det = p - buf;
                    break;
                }
                int64_t idx;
                double v;
                if (!parse_int_fast(p, colon, idx) || !parse_float_fast(colon + 1, te, v)) {
                    st = LS_HOST;
                    break;
                }
                if (idx <= prev) {
                    st = LS_NONINC;
                    det = idx;
                    break;
                }
                prev = idx;
                mx = idx;
                cnt++;
                p = te;
            }
        }
        labels[j] = lab;
        nfeat[j] = cnt;
        status[j] = st;
        detail[j] = det;
        if (st == LS_OK && mx > 0) atomicMax(max_idx, (unsigned long long)mx);
    }
}

// per OK line: its (col = idx - 1, value) pairs at row_ptr[row_of_line[j]]
__global__ void k_libsvm_fill(const uint8_t *buf, int64_t n, const int64_t *ls, int64_t m, const int32_t *status,
                              const int64_t *row_of_line, const int64_t *row_ptr, int64_t *cols, double *vals)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        if (status[j] != LS_OK) continue;
        const uint8_t *p = buf + ls[j];
        const uint8_t *end = buf + (j + 1 < m ? ls[j + 1] : n);
        const uint8_t *hash = p;
        while (hash < end && *hash != '#' && *hash != '\n') hash++;
        end = hash;
        while (p < end && is_ws(*p)) p++;
        while (p < end && !is_ws(*p)) p++;  // label
        int64_t o = row_ptr[row_of_line[j]];
        while (true) {
            while (p < end && is_ws(*p)) p++;
            if (p == end) break;
            const uint8_t *te = p;
            while (te < end && !is_ws(*te)) te++;
            const uint8_t *colon = p;
            while (colon < te && *colon != ':') colon++;
            int64_t idx = 0;
            double v = 0.0;
            parse_int_fast(p, colon, idx);
            parse_float_fast(colon + 1, te, v);
            cols[o] = idx - 1;
            vals[o] = v;
            o++;
            p = te;
        }
    }
}

// line starts: chunk newline counts, exclusive scan, positions
constexpr int64_t LS_CHUNK = 1 << 14;
__global__ void k_nl_count(const uint8_t *buf, int64_t n, int64_t nchunk, int64_t *cnt)
{
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        int64_t a = c * LS_CHUNK, b = min(n, a + LS_CHUNK), k = 0;
        for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) k += buf[i] == '\n';
        k = __reduce_add_sync(FULL, (unsigned)k);
        __shared__ int64_t part[32];
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = k;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t s = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += part[w];
            cnt[c] = s;
        }
        __syncthreads();
    }
}

// one thread per chunk, sequential inside: ordered positions without a second scan
__global__ void k_nl_write(const uint8_t *buf, int64_t n, int64_t nchunk, const int64_t *off, int64_t *ls, int64_t m)
{
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunk; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = c * LS_CHUNK, b = min(n, a + LS_CHUNK), o = off[c] + 1;  // line 0 starts at 0
        for (int64_t i = a; i < b; i++)
            if (buf[i] == '\n' && o < m) ls[o++] = i + 1;
    }
}

}  // namespace

// scan helper from aux.cu (exclusive, in place, single CTA)
__global__ void k_scan_small(int64_t *sums, int nb);

extern "C" int ps_libsvm_index(const uint8_t *buf, int64_t n, int64_t *line_start, int64_t m, void *stream)
{
    if (!buf || !line_start || n < 1 || m < 1) return ps_fail(PS_EINVAL, "bad libsvm index arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nchunk = (n + LS_CHUNK - 1) / LS_CHUNK;
    if (nchunk > (1ll << 30)) return ps_fail(PS_EINVAL, "input too large");
    int64_t *cnt = nullptr;
    CK(cudaMallocAsync((void **)&cnt, sizeof(int64_t) * nchunk, st), "ps_libsvm_index alloc");
    k_nl_count<<<(int)std::min<int64_t>(nchunk, 1 << 16), 256, 0, st>>>(buf, n, nchunk, cnt);
    k_scan_small<<<1, 1024, 0, st>>>(cnt, (int)nchunk);
    CK(cudaMemsetAsync(line_start, 0, sizeof(int64_t), st), "ps_libsvm_index memset");
    k_nl_write<<<(int)((nchunk + 255) / 256), 256, 0, st>>>(buf, n, nchunk, cnt, line_start, m);
    CK(cudaGetLastError(), "ps_libsvm_index launch");
    CK(cudaFreeAsync(cnt, st), "ps_libsvm_index free");
    return PS_OK;
}

extern "C" int ps_libsvm_scan(const uint8_t *buf, int64_t n, const int64_t *line_start, int64_t m, double *labels,
                              int32_t *nfeat, int32_t *status, int64_t *detail, unsigned long long *max_idx,
                              void *stream)
{
    if (!buf || !line_start || !labels || !nfeat || !status || !detail || !max_idx || m < 1)
        return ps_fail(PS_EINVAL, "bad libsvm scan arguments");
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemsetAsync(max_idx, 0, sizeof(unsigned long long), st), "ps_libsvm_scan memset");
    k_libsvm_scan<<<(int)std::min<int64_t>((m + 127) / 128, 1 << 20), 128, 0, st>>>(buf, n, line_start, m, labels,
                                                                                    nfeat, status, detail, max_idx);
    CK(cudaGetLastError(), "ps_libsvm_scan launch");
    return PS_OK;
}

extern "C" int ps_libsvm_fill(const uint8_t *buf, int64_t n, const int64_t *line_start, int64_t m,
                              const int32_t *status, const int64_t *row_of_line, const int64_t *row_ptr, int64_t *cols,
                              double *vals, void *stream)
{
    if (!buf || !line_start || !status || !row_of_line || !row_ptr || !cols || !vals || m < 1)
        return ps_fail(PS_EINVAL, "bad libsvm fill arguments");
    cudaStream_t st = (cudaStream_t)stream;
    k_libsvm_fill<<<(int)std::min<int64_t>((m + 127) / 128, 1 << 20), 128, 0, st>>>(buf, n, line_start, m, status,
                                                                                    row_of_line, row_ptr, cols, vals);
    CK(cudaGetLastError(), "ps_libsvm_fill launch");
    return PS_OK;
}
