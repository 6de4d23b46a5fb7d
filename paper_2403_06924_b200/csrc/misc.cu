// Element-wise, layout and sparse kernels behind the rest of the reference's
// API surface (quantize.hpp / matrix.hpp / sparse.hpp).  None of these sit on
// the benchmarked hot path except the transposes used for parity dumps; they
// keep the drop-in complete without any CPU fallback.
#include <cfloat>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "misc.h"

namespace xg {
namespace {

constexpr int kT = 256;

inline int blocks_for(int64_t n, int per = kT) {
    int64_t b = (n + per - 1) / per;
    if (b < 1) b = 1;
    if (b > 65535LL * 16) b = 65535LL * 16;
    return (int)b;
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ double scale_of(int scheme, const double* s, int i, int j) {
    return scheme == kPerRow ? s[i] : scheme == kPerColumn ? s[j] : s[0];
}

// src: rows x cols int8 with pitch lds -> dst: cols x rows with pitch ldd
__global__ void k_transpose_i8(const int8_t* __restrict__ src, int rows, int cols, int64_t lds,
                               int8_t* __restrict__ dst, int64_t ldd) {
    XG_PDL_WAIT();
    __shared__ int8_t t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[k][threadIdx.x] = src[(int64_t)r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[(int64_t)c * ldd + r] = t[threadIdx.x][k];
    }
}

__global__ void k_quantize_with_scales(const float* __restrict__ a, int rows, int cols, int bits,
                                       int scheme, const double* __restrict__ s, int rounding,
                                       int8_t* __restrict__ q) {
    XG_PDL_WAIT();
    const int qmax = quant_max(bits);
    const int64_t n = (int64_t)rows * cols;
    GRID_STRIDE(x, n) {
        const int i = (int)(x / cols), j = (int)(x % cols);
        q[x] = (int8_t)quantize_scalar((double)a[x], scale_of(scheme, s, i, j), qmax, rounding);
    }
}

__global__ void k_dequantize(const int8_t* __restrict__ q, int rows, int cols, int scheme,
                             const double* __restrict__ s, const float* __restrict__ a,
                             float* __restrict__ out) {
    XG_PDL_WAIT();
    const int64_t n = (int64_t)rows * cols;
    GRID_STRIDE(x, n) {
        const int i = (int)(x / cols), j = (int)(x % cols);
        const float d = dequant_value(q[x], scale_of(scheme, s, i, j));
        out[x] = a ? __fsub_rn(a[x], d) : d;
    }
}

__global__ void k_dequant_product(const int32_t* __restrict__ p, int rows, int cols, int sa_scheme,
                                  const double* __restrict__ sa, int sb_scheme,
                                  const double* __restrict__ sb, float* __restrict__ out) {
    XG_PDL_WAIT();
    const int64_t n = (int64_t)rows * cols;
    GRID_STRIDE(x, n) {
        const int i = (int)(x / cols), j = (int)(x % cols);
        const double la = sa_scheme == kPerRow ? sa[i] : sa[0];
        const double lb = sb_scheme == kPerColumn ? sb[j] : sb[0];
        out[x] = dequant_product_value(p[x], la, lb);
    }
}

// matrix.cpp:75-95: fp64 accumulate over ascending k, then float.
__global__ void k_gemm_f32_exact(const float* __restrict__ a, const float* __restrict__ b, int m,
                                 int k, int n, float* __restrict__ c) {
    XG_PDL_WAIT();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= n || i >= m) return;
    double acc = 0.0;
    const float* ar = a + (int64_t)i * k;
    for (int p = 0; p < k; ++p) acc = __dadd_rn(acc, __dmul_rn((double)ar[p], (double)b[(int64_t)p * n + j]));
    c[(int64_t)i * n + j] = __double2float_rn(acc);
}

__global__ void k_axpby(float* __restrict__ d, float alpha, const float* __restrict__ c, float beta,
                        int64_t n) {
    XG_PDL_WAIT();
    GRID_STRIDE(x, n) { d[x] = __fadd_rn(__fmul_rn(alpha, d[x]), __fmul_rn(beta, c[x])); }
}
__global__ void k_subtract(const float* __restrict__ a, const float* __restrict__ b,
                           float* __restrict__ o, int64_t n) {
    XG_PDL_WAIT();
    GRID_STRIDE(x, n) { o[x] = __fsub_rn(a[x], b[x]); }
}
__global__ void k_add(float* __restrict__ d, const float* __restrict__ x, int64_t n) {
    XG_PDL_WAIT();
    GRID_STRIDE(i, n) { d[i] = __fadd_rn(d[i], x[i]); }
}

// ------------------------------------------------------------------ CSR ----
// Threshold of row (per_row) or column of element (i, j); sparse.cpp:49-55.
__device__ __forceinline__ double thr_at(const float* stat, int idx, double thr_m, int policy,
                                         double so, int inner) {
    if (policy == kAvg) return __dmul_rn(thr_m, (double)stat[idx]);
    return __ddiv_rn(__dmul_rn(__dmul_rn(thr_m, so), (double)stat[idx]), (double)inner);
}

// mode 0: reduce (|v| > t);  mode 1: csr_from_dense (v != 0)
__device__ __forceinline__ bool keep_at(int mode, const float* m, int cols, int i, int j,
                                        const float* stat, double thr_m, int policy, double so,
                                        int per_row, int rows) {
    const float v = m[(int64_t)i * cols + j];
    if (mode == 1) return v != 0.0f;
    const double t = per_row ? thr_at(stat, i, thr_m, policy, so, cols)
                             : thr_at(stat, j, thr_m, policy, so, rows);
    return fabs((double)v) > t;
}

// One warp per row: count, then (second kernel) ballot + popc ranks write
// ascending column order (sparse.hpp:11-13).
__global__ void k_csr_count(int mode, const float* __restrict__ m, int rows, int cols,
                            const float* stat, double thr_m, int policy, double so, int per_row,
                            int32_t* __restrict__ cnt) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    int c = 0;
    for (int j = lane; j < cols; j += 32)
        c += keep_at(mode, m, cols, w, j, stat, thr_m, policy, so, per_row, rows);
    c = warp_sum(c);
    if (lane == 0) cnt[w] = c;
}

__global__ void k_csr_fill(int mode, const float* __restrict__ m, int rows, int cols,
                           const float* stat, double thr_m, int policy, double so, int per_row,
                           const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
                           float* __restrict__ values) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    int pos = row_ptr[w];
    for (int j0 = 0; j0 < cols; j0 += 32) {
        const int j = j0 + lane;
        const bool k = j < cols && keep_at(mode, m, cols, w, j, stat, thr_m, policy, so, per_row, rows);
        const unsigned bal = __ballot_sync(0xffffffffu, k);
        if (k) {
            const int at = pos + __popc(bal & ((1u << lane) - 1u));
            col_idx[at] = j;
            values[at] = m[(int64_t)w * cols + j];
        }
        pos += __popc(bal);
    }
}

// exclusive scan of cnt[0..rows) into row_ptr[0..rows], row_ptr[rows] = total
__global__ void k_shift_total(int32_t* row_ptr, const int32_t* cnt, int rows) {
    XG_PDL_WAIT();
    row_ptr[rows] = rows > 0 ? row_ptr[rows - 1] + cnt[rows - 1] : 0;
}

// quantize_csr scales (sparse.cpp:198-225)
__global__ void k_csr_rowmax(int rows, const int32_t* __restrict__ rp, const float* __restrict__ v,
                             int bits, double* scales) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    float m = 0.0f;
    for (int p = rp[w] + lane; p < rp[w + 1]; p += 32) m = fmaxf(m, fabsf(v[p]));
    m = warp_maxf(m);
    if (lane == 0) scales[w] = compute_scale((double)m, bits);
}
__global__ void k_csr_colmax(int64_t nnz, const int32_t* __restrict__ ci, const float* __restrict__ v,
                             uint32_t* colmax, uint32_t* tmax) {
    XG_PDL_WAIT();
    GRID_STRIDE(p, nnz) {
        const uint32_t b = fbits(fabsf(v[p]));
        atomicMax(colmax + ci[p], b);
        atomicMax(tmax, b);
    }
}
__global__ void k_scales_from_bits(const uint32_t* bits_in, int n, int bits, double* scales) {
    XG_PDL_WAIT();
    GRID_STRIDE(i, (int64_t)n) { scales[i] = compute_scale((double)__uint_as_float(bits_in[i]), bits); }
}
__global__ void k_csr_quant(int rows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const float* __restrict__ v, int bits, int scheme,
                            const double* __restrict__ s, int rounding, int8_t* __restrict__ q) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int qmax = quant_max(bits);
    for (int p = rp[w] + lane; p < rp[w + 1]; p += 32) {
        const double lam = scheme == kPerRow ? s[w] : scheme == kPerColumn ? s[ci[p]] : s[0];
        q[p] = (int8_t)quantize_scalar((double)v[p], lam, qmax, rounding);
    }
}

// csr rows of each element (for transposes)
__global__ void k_csr_rows(int rows, const int32_t* __restrict__ rp, int32_t* __restrict__ r) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    for (int p = rp[w] + lane; p < rp[w + 1]; p += 32) r[p] = w;
}
__global__ void k_iota(int32_t* p, int64_t n) {
    XG_PDL_WAIT(); GRID_STRIDE(i, n) p[i] = (int32_t)i; }
__global__ void k_col_hist(int64_t nnz, const int32_t* __restrict__ ci, int32_t* cnt) {
    XG_PDL_WAIT();
    GRID_STRIDE(p, nnz) atomicAdd(cnt + ci[p], 1);
}
template <class T>
__global__ void k_gather_T(int64_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rows_of,
                           const T* __restrict__ v, int32_t* __restrict__ tci, T* __restrict__ tv) {
    XG_PDL_WAIT();
    GRID_STRIDE(p, nnz) {
        const int32_t src = perm[p];
        tci[p] = rows_of[src];
        tv[p] = v[src];
    }
}

// spmm_int (sparse.cpp:119-138): warp per (row, 256-column strip); exact s32.
__global__ void k_spmm_i8(int rows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const int8_t* __restrict__ v, const int8_t* __restrict__ d, int d_cols,
                          int32_t* __restrict__ out) {
    XG_PDL_WAIT();
    const int i = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows || j >= d_cols) return;
    int32_t acc = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) acc += (int32_t)v[p] * (int32_t)d[(int64_t)ci[p] * d_cols + j];
    out[(int64_t)i * d_cols + j] = acc;
}

// spmm (sparse.cpp:97-117): fp64 accumulation in CSR order per element.
__global__ void k_spmm_f32(int rows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const float* __restrict__ v, const float* __restrict__ d, int d_cols,
                           float* __restrict__ out) {
    XG_PDL_WAIT();
    const int i = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows || j >= d_cols) return;
    double acc = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
        acc = __dadd_rn(acc, __dmul_rn((double)v[p], (double)d[(int64_t)ci[p] * d_cols + j]));
    out[(int64_t)i * d_cols + j] = __double2float_rn(acc);
}

__global__ void k_densify(int rows, int cols, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const float* __restrict__ v,
                          float* __restrict__ out) {
    XG_PDL_WAIT();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= rows) return;
    for (int j = lane; j < cols; j += 32) out[(int64_t)w * cols + j] = 0.0f;
    __syncwarp();
    for (int p = rp[w] + lane; p < rp[w + 1]; p += 32) out[(int64_t)w * cols + ci[p]] = v[p];
}

__global__ void k_finite_max(const float* __restrict__ x, int64_t n, uint32_t* mx, int* bad) {
    XG_PDL_WAIT();
    float m = 0.0f;
    int b = 0;
    GRID_STRIDE(i, n) {
        const float v = x[i];
        m = fmaxf(m, fabsf(v));
        b |= isinf(v) ? 1 : (v != v ? 2 : 0);
    }
    m = warp_maxf(m);
    b = warp_max(b);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx, fbits(m));
        if (b) atomicOr(bad, b);
    }
}

__global__ void k_random_i8(int8_t* p, int64_t n, uint64_t seed) {
    XG_PDL_WAIT();
    GRID_STRIDE(i, n) {
        uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        p[i] = (int8_t)((int)((z ^ (z >> 31)) % 255) - 127);
    }
}

}  // namespace

void random_i8(int8_t* p, int64_t n, uint64_t seed, cudaStream_t s) {
    k_random_i8<<<blocks_for(n), kT, 0, s>>>(p, n, seed);
}

void transpose_i8(const int8_t* src, int rows, int cols, int64_t lds, int8_t* dst, int64_t ldd,
                  cudaStream_t s) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    k_transpose_i8<<<grid, block, 0, s>>>(src, rows, cols, lds, dst, ldd);
}

void quantize_with_scales(const float* a, int rows, int cols, int bits, int scheme,
                          const double* scales, int rounding, int8_t* q, cudaStream_t s) {
    k_quantize_with_scales<<<blocks_for((int64_t)rows * cols), kT, 0, s>>>(a, rows, cols, bits, scheme,
                                                                          scales, rounding, q);
}

void dequantize(const int8_t* q, int rows, int cols, int scheme, const double* scales,
                const float* minuend, float* out, cudaStream_t s) {
    k_dequantize<<<blocks_for((int64_t)rows * cols), kT, 0, s>>>(q, rows, cols, scheme, scales, minuend,
                                                                out);
}

void dequant_product(const int32_t* p, int rows, int cols, int sa_scheme, const double* sa,
                     int sb_scheme, const double* sb, float* out, cudaStream_t s) {
    k_dequant_product<<<blocks_for((int64_t)rows * cols), kT, 0, s>>>(p, rows, cols, sa_scheme, sa,
                                                                     sb_scheme, sb, out);
}

void gemm_f32_exact(const float* a, const float* b, int m, int k, int n, float* c, cudaStream_t s) {
    dim3 grid((n + 127) / 128, m);
    k_gemm_f32_exact<<<grid, 128, 0, s>>>(a, b, m, k, n, c);
}

void axpby(float* d, float alpha, const float* c, float beta, int64_t n, cudaStream_t s) {
    k_axpby<<<blocks_for(n), kT, 0, s>>>(d, alpha, c, beta, n);
}
void subtract(const float* a, const float* b, float* o, int64_t n, cudaStream_t s) {
    k_subtract<<<blocks_for(n), kT, 0, s>>>(a, b, o, n);
}
void add_inplace(float* d, const float* x, int64_t n, cudaStream_t s) {
    k_add<<<blocks_for(n), kT, 0, s>>>(d, x, n);
}
void finite_max(const float* x, int64_t n, uint32_t* mx, int* bad, cudaStream_t s) {
    int b = blocks_for(n);
    if (b > 148 * 8) b = 148 * 8;
    k_finite_max<<<b, kT, 0, s>>>(x, n, mx, bad);
}

// row_ptr must have rows+1 entries; cnt scratch of rows entries.
cudaError_t csr_count(int mode, const float* m, int rows, int cols, const float* stat, double thr_m,
                      int policy, double so, int per_row, int32_t* row_ptr, int32_t* cnt,
                      cudaStream_t s) {
    const int wb = (rows * 32 + kT - 1) / kT;
    k_csr_count<<<wb > 0 ? wb : 1, kT, 0, s>>>(mode, m, rows, cols, stat, thr_m, policy, so, per_row, cnt);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, row_ptr, rows, s);
    void* t = nullptr;
    cudaError_t e = cudaMallocAsync(&t, tmp ? tmp : 1, s);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::ExclusiveSum(t, tmp, cnt, row_ptr, rows, s);
    cudaFreeAsync(t, s);
    k_shift_total<<<1, 1, 0, s>>>(row_ptr, cnt, rows);
    return cudaGetLastError();
}

void csr_fill(int mode, const float* m, int rows, int cols, const float* stat, double thr_m,
              int policy, double so, int per_row, const int32_t* row_ptr, int32_t* col_idx,
              float* values, cudaStream_t s) {
    const int wb = (rows * 32 + kT - 1) / kT;
    k_csr_fill<<<wb > 0 ? wb : 1, kT, 0, s>>>(mode, m, rows, cols, stat, thr_m, policy, so, per_row,
                                             row_ptr, col_idx, values);
}

void csr_quantize(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v,
                  int64_t nnz, int bits, int scheme, int rounding, int8_t* q, double* scales,
                  uint32_t* scratch /* cols + 1 */, cudaStream_t s) {
    const int wb = (rows * 32 + kT - 1) / kT;
    if (scheme == kPerRow) {
        k_csr_rowmax<<<wb > 0 ? wb : 1, kT, 0, s>>>(rows, rp, v, bits, scales);
    } else {
        cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * ((size_t)cols + 1), s);
        if (nnz > 0) k_csr_colmax<<<blocks_for(nnz), kT, 0, s>>>(nnz, ci, v, scratch, scratch + cols);
        if (scheme == kPerColumn) k_scales_from_bits<<<blocks_for(cols), kT, 0, s>>>(scratch, cols, bits, scales);
        else k_scales_from_bits<<<1, 32, 0, s>>>(scratch + cols, 1, bits, scales);
    }
    k_csr_quant<<<wb > 0 ? wb : 1, kT, 0, s>>>(rows, rp, ci, v, bits, scheme, scales, rounding, q);
}

// Stable counting transpose: a stable radix sort of column keys keeps rows in
// ascending order inside every output row (sparse.cpp:168-188).
template <class T>
cudaError_t csr_transpose(int rows, int cols, const int32_t* rp, const int32_t* ci, const T* v,
                          int64_t nnz, int32_t* trp, int32_t* tci, T* tv, cudaStream_t s) {
    int32_t *cnt = nullptr, *rows_of = nullptr, *keys_out = nullptr, *idx = nullptr, *perm = nullptr;
    const size_t nz = nnz > 0 ? (size_t)nnz : 1;
    cudaError_t e = cudaMallocAsync(&cnt, sizeof(int32_t) * ((size_t)cols + 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&rows_of, sizeof(int32_t) * nz, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&keys_out, sizeof(int32_t) * nz, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&idx, sizeof(int32_t) * nz, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&perm, sizeof(int32_t) * nz, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)cols + 1), s);
    if (nnz > 0) {
        const int wb = (rows * 32 + kT - 1) / kT;
        k_csr_rows<<<wb > 0 ? wb : 1, kT, 0, s>>>(rows, rp, rows_of);
        k_iota<<<blocks_for(nnz), kT, 0, s>>>(idx, nnz);
        k_col_hist<<<blocks_for(nnz), kT, 0, s>>>(nnz, ci, cnt);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, ci, keys_out, idx, perm, (int)nnz, 0, 32, s);
        void* t = nullptr;
        e = cudaMallocAsync(&t, tmp ? tmp : 1, s);
        if (e != cudaSuccess) return e;
        cub::DeviceRadixSort::SortPairs(t, tmp, ci, keys_out, idx, perm, (int)nnz, 0, 32, s);
        cudaFreeAsync(t, s);
        k_gather_T<T><<<blocks_for(nnz), kT, 0, s>>>(nnz, perm, rows_of, v, tci, tv);
    }
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, trp, cols + 1, s);
    void* t = nullptr;
    e = cudaMallocAsync(&t, tmp ? tmp : 1, s);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::ExclusiveSum(t, tmp, cnt, trp, cols + 1, s);
    cudaFreeAsync(t, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(rows_of, s);
    cudaFreeAsync(keys_out, s);
    cudaFreeAsync(idx, s);
    cudaFreeAsync(perm, s);
    return cudaGetLastError();
}

template cudaError_t csr_transpose<int8_t>(int, int, const int32_t*, const int32_t*, const int8_t*,
                                           int64_t, int32_t*, int32_t*, int8_t*, cudaStream_t);
template cudaError_t csr_transpose<float>(int, int, const int32_t*, const int32_t*, const float*,
                                          int64_t, int32_t*, int32_t*, float*, cudaStream_t);

void spmm_i8(int rows, const int32_t* rp, const int32_t* ci, const int8_t* v, const int8_t* d,
             int d_cols, int32_t* out, cudaStream_t s) {
    dim3 grid((d_cols + 255) / 256, rows);
    k_spmm_i8<<<grid, 256, 0, s>>>(rows, rp, ci, v, d, d_cols, out);
}
void spmm_f32(int rows, const int32_t* rp, const int32_t* ci, const float* v, const float* d,
              int d_cols, float* out, cudaStream_t s) {
    dim3 grid((d_cols + 255) / 256, rows);
    k_spmm_f32<<<grid, 256, 0, s>>>(rows, rp, ci, v, d, d_cols, out);
}
void densify(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v, float* out,
             cudaStream_t s) {
    const int wb = (rows * 32 + kT - 1) / kT;
    k_densify<<<wb > 0 ? wb : 1, kT, 0, s>>>(rows, cols, rp, ci, v, out);
}

}  // namespace xg
