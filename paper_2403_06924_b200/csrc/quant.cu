// K1 (quantiser) and K3 (residual quantisation + threshold selection).
//
// HBM-bound integer/byte work: 128-bit coalesced loads, rows held in registers
// so each input byte leaves HBM once per pass, warp-shuffle + shared-memory
// block reductions, one atomic per CTA for the global maxima.
//
// Replaces (reference, proj/src/):
//   quantize / quantize_with_scales / slice_max_abs   quantize.cpp:28-36,107-150
//   DenseMatrix::all_finite / max_abs                 matrix.cpp:44-58
//   dequantize + subtract (max|R|)                    quantize.cpp:152-167, pipeline.cpp:79-84
//   residual quantize (always per-tensor)             pipeline.cpp:86-93
//   reduce_a / reduce_b (+density, quantize_csr values) sparse.cpp:36-95,193-240
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace xg {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
    v = warp_maxf(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float r = red[0];
#pragma unroll
    for (int i = 1; i < kThreads / 32; ++i) r = fmaxf(r, red[i]);
    return r;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    unsigned long long r = 0;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) r += red[i];
    return r;
}

// bit 0: +-inf (the reference's compute_scale throws), bit 1: NaN (only the
// pipeline's all_finite check rejects it; quantize() maps it to -qmax).
__device__ __forceinline__ int not_finite(float x) { return isinf(x) ? 1 : (x != x ? 2 : 0); }

// Row element e of this thread: column (v*256 + tid)*4 + (e%4).
template <int VPT>
__device__ __forceinline__ void load_row(const float* __restrict__ row, int cols, bool vec,
                                         float (&x)[VPT * 4]) {
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int c = (v * kThreads + (int)threadIdx.x) * 4;
        if (vec && c + 3 < cols) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(row + c));
            x[4 * v] = f.x;
            x[4 * v + 1] = f.y;
            x[4 * v + 2] = f.z;
            x[4 * v + 3] = f.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) x[4 * v + e] = (c + e < cols) ? __ldg(row + c + e) : 0.0f;
        }
    }
}

template <int VPT>
__device__ __forceinline__ void store_row_i8(int8_t* __restrict__ row, int cols, bool vec,
                                             const int (&q)[VPT * 4]) {
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int c = (v * kThreads + (int)threadIdx.x) * 4;
        if (vec && c + 3 < cols) {
            const uint32_t p = (uint32_t)(q[4 * v] & 0xff) | ((uint32_t)(q[4 * v + 1] & 0xff) << 8) |
                               ((uint32_t)(q[4 * v + 2] & 0xff) << 16) |
                               ((uint32_t)(q[4 * v + 3] & 0xff) << 24);
            *reinterpret_cast<uint32_t*>(row + c) = p;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (c + e < cols) row[c + e] = (int8_t)q[4 * v + e];
        }
    }
}

// ------------------------------------------------------------------ K1 rows --
// One CTA per row.  PerRow: row absmax -> lambda_i; quantize; residual via a
// 255-entry per-row table of float(q / lambda_i); max|residual|.
template <int VPT>
__global__ void __launch_bounds__(kThreads) k_quant_rows(const QuantRowsArgs a) {
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    const int qmax = quant_max(a.bits);
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (a.ldq % 4 == 0);
    float rmax_acc = 0.0f, gmax_acc = 0.0f;
    int bad = 0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        float x[VPT * 4];
        load_row<VPT>(a.x + (int64_t)r * a.ld, a.cols, vec, x);
        float m = 0.0f;
#pragma unroll
        for (int e = 0; e < VPT * 4; ++e) {
            m = fmaxf(m, fabsf(x[e]));
            bad |= not_finite(x[e]);
        }
        m = block_max(m, red);
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);  // slice_max_abs: fp64 max == float max
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        int q[VPT * 4];
        float rm = 0.0f;
#pragma unroll
        for (int e = 0; e < VPT * 4; ++e) {
            q[e] = quantize_scalar((double)x[e], lam, qmax, a.rounding);
            rm = fmaxf(rm, fabsf(__fsub_rn(x[e], lut[q[e] + qmax])));
        }
        store_row_i8<VPT>(a.q + (int64_t)r * a.ldq, a.cols, vec, q);
        rmax_acc = fmaxf(rmax_acc, rm);
        __syncthreads();  // lut reuse
    }
    rmax_acc = block_max(rmax_acc, red);
    if (threadIdx.x == 0) {
        if (a.rmax) atomicMax(a.rmax, fbits(rmax_acc));
        if (a.gmax) atomicMax(a.gmax, fbits(gmax_acc));
    }
    if (bad && a.nonfinite) atomicOr(a.nonfinite, bad);
}

// Generic (any column count) variant: two passes over the row, the second one
// served from L2.
__global__ void __launch_bounds__(kThreads) k_quant_rows_generic(const QuantRowsArgs a) {
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    const int qmax = quant_max(a.bits);
    float rmax_acc = 0.0f, gmax_acc = 0.0f;
    int bad = 0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        const float* row = a.x + (int64_t)r * a.ld;
        float m = 0.0f;
        for (int c = threadIdx.x; c < a.cols; c += kThreads) {
            const float v = row[c];
            m = fmaxf(m, fabsf(v));
            bad |= not_finite(v);
        }
        m = block_max(m, red);
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        float rm = 0.0f;
        for (int c = threadIdx.x; c < a.cols; c += kThreads) {
            const float v = row[c];
            const int q = quantize_scalar((double)v, lam, qmax, a.rounding);
            a.q[(int64_t)r * a.ldq + c] = (int8_t)q;
            rm = fmaxf(rm, fabsf(__fsub_rn(v, lut[q + qmax])));
        }
        rmax_acc = fmaxf(rmax_acc, rm);
        __syncthreads();
    }
    rmax_acc = block_max(rmax_acc, red);
    if (threadIdx.x == 0) {
        if (a.rmax) atomicMax(a.rmax, fbits(rmax_acc));
        if (a.gmax) atomicMax(a.gmax, fbits(gmax_acc));
    }
    if (bad && a.nonfinite) atomicOr(a.nonfinite, bad);
}

// --------------------------------------------------------------- absmaxes --
__global__ void __launch_bounds__(kThreads)
    k_absmax_global(const float* __restrict__ x, int64_t n, uint32_t* gmax, int* nonfinite) {
    __shared__ float red[kThreads / 32];
    float m = 0.0f;
    int bad = 0;
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n4; i += stride) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(x) + i);
        m = fmaxf(fmaxf(fmaxf(m, fabsf(f.x)), fmaxf(fabsf(f.y), fabsf(f.z))), fabsf(f.w));
        bad |= not_finite(f.x) | not_finite(f.y) | not_finite(f.z) | not_finite(f.w);
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        const float v = x[i];
        m = fmaxf(m, fabsf(v));
        bad |= not_finite(v);
    }
    m = block_max(m, red);
    if (threadIdx.x == 0) atomicMax(gmax, fbits(m));
    if (bad) atomicOr(nonfinite, bad);
}

// Column absmax of a row-major rows x cols matrix: each thread owns 4 adjacent
// columns over a 64-row slab; one atomicMax per column per slab.
constexpr int kColSlab = 64;
__global__ void __launch_bounds__(kThreads)
    k_absmax_cols(const float* __restrict__ x, int rows, int cols, int64_t ld, uint32_t* colmax,
                  uint32_t* gmax, int* nonfinite) {
    __shared__ float red[kThreads / 32];
    const int c = (blockIdx.x * kThreads + threadIdx.x) * 4;
    const int r0 = blockIdx.y * kColSlab;
    const int r1 = min(rows, r0 + kColSlab);
    const bool vec = (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && c + 3 < cols;
    float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
    int bad = 0;
    if (c < cols) {
        for (int r = r0; r < r1; ++r) {
            const float* p = x + (int64_t)r * ld + c;
            float4 f;
            if (vec) {
                f = __ldg(reinterpret_cast<const float4*>(p));
            } else {
                f.x = p[0];
                f.y = c + 1 < cols ? p[1] : 0.f;
                f.z = c + 2 < cols ? p[2] : 0.f;
                f.w = c + 3 < cols ? p[3] : 0.f;
            }
            m0 = fmaxf(m0, fabsf(f.x));
            m1 = fmaxf(m1, fabsf(f.y));
            m2 = fmaxf(m2, fabsf(f.z));
            m3 = fmaxf(m3, fabsf(f.w));
            bad |= not_finite(f.x) | not_finite(f.y) | not_finite(f.z) | not_finite(f.w);
        }
        atomicMax(colmax + c, fbits(m0));
        if (c + 1 < cols) atomicMax(colmax + c + 1, fbits(m1));
        if (c + 2 < cols) atomicMax(colmax + c + 2, fbits(m2));
        if (c + 3 < cols) atomicMax(colmax + c + 3, fbits(m3));
    }
    const float m = block_max(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), red);
    if (threadIdx.x == 0 && gmax) atomicMax(gmax, fbits(m));
    if (bad) atomicOr(nonfinite, bad);
}

// ------------------------------------------------------------- K1 columns --
// Tile of 128 rows (K) x 64 columns (N) of a row-major matrix: quantise with
// per-column (or per-tensor) scales and write the ints transposed (N x K,
// K-major) through shared memory — the layout the tensor-core B operand wants.
constexpr int kTK = 128, kTN = 64;

__device__ __forceinline__ void store_T_tile(const int8_t (*tq)[kTK + 16], int8_t* dst,
                                             int64_t ldq, int n0, int k0, int cols, int rows) {
    // 64 rows x 128 bytes; thread -> (row c = tid/4, 32-byte chunk (tid%4))
    const int c = threadIdx.x >> 2;
    const int kk = (threadIdx.x & 3) * 32;
    if (n0 + c >= cols) return;
    int8_t* d = dst + (int64_t)(n0 + c) * ldq + k0 + kk;
    const int kval = rows - (k0 + kk);  // valid bytes in this chunk
    if (kval >= 32 && (ldq % 16) == 0) {
        const int4* s = reinterpret_cast<const int4*>(&tq[c][kk]);
        reinterpret_cast<int4*>(d)[0] = s[0];
        reinterpret_cast<int4*>(d)[1] = s[1];
    } else {
        for (int j = 0; j < 32 && j < kval; ++j) d[j] = tq[c][kk + j];
    }
}

__global__ void __launch_bounds__(kThreads) k_quant_cols_T(const QuantColsArgs a) {
    __shared__ __align__(16) int8_t tq[kTN][kTK + 16];
    __shared__ double lam_s[kTN];
    __shared__ float red[kThreads / 32];
    const int n0 = blockIdx.x * kTN, k0 = blockIdx.y * kTK;
    const int qmax = quant_max(a.bits);
    if (threadIdx.x < kTN) {
        const int c = min(n0 + (int)threadIdx.x, a.cols - 1);
        double lam;
        if (a.per_col) {
            lam = compute_scale((double)__uint_as_float(a.colmax[c]), a.bits);
            if (blockIdx.y == 0 && a.lam_out && n0 + (int)threadIdx.x < a.cols) a.lam_out[c] = lam;
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        lam_s[threadIdx.x] = lam;
    }
    __syncthreads();
    const int cg = (threadIdx.x & 15) * 4;  // 4 columns
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (n0 + cg + 3 < a.cols);
    float rm = 0.0f;
#pragma unroll 4
    for (int i = 0; i < kTK / 16; ++i) {
        const int kr = (threadIdx.x >> 4) + 16 * i;
        const int k = k0 + kr;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (k < a.rows) {
            const float* p = a.x + (int64_t)k * a.ld + n0 + cg;
            if (vec) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(p));
                v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = (n0 + cg + e < a.cols) ? p[e] : 0.f;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double lam = lam_s[cg + e];
            const int q = quantize_scalar((double)v[e], lam, qmax, a.rounding);
            tq[cg + e][kr] = (int8_t)q;
            rm = fmaxf(rm, fabsf(__fsub_rn(v[e], dequant_value(q, lam))));
        }
    }
    __syncthreads();
    store_T_tile(tq, a.qT, a.ldq, n0, k0, a.cols, a.rows);
    rm = block_max(rm, red);
    if (threadIdx.x == 0 && a.rmax) atomicMax(a.rmax, fbits(rm));
}

// ------------------------------------------------------------- K3 rows --
// Per row i of A: RAq = quantize(a - deq(aq), lambda_RA) and the reduced
// operand A'q = (|a| > t_i) ? aq : 0 (quantize_csr values equal aq under
// PerRow scales; under PerTensor the retained-max scale is checked afterwards
// and a fix-up pass rewrites A'q if it differs).
__device__ __forceinline__ double threshold_of(int policy, double thr_m, float stat,
                                               double scale_other, int inner) {
    // sparse.cpp:49-55
    if (policy == kAvg) return __dmul_rn(thr_m, (double)stat);
    return __ddiv_rn(__dmul_rn(__dmul_rn(thr_m, scale_other), (double)stat), (double)inner);
}

template <int VPT>
__global__ void __launch_bounds__(kThreads) k_select_rows(const SelectArgs a) {
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    __shared__ unsigned long long redu[kThreads / 32];
    const int qmax = quant_max(a.bits);
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (a.ldq % 4 == 0);
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double scale_other =
        a.do_select && a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                                        : 1.0;
    double lam_fix = 0.0;
    if (a.fix_mode) {
        // PerTensor reduced operand: lambda' over the retained values (sparse.cpp:198-203)
        lam_fix = compute_scale((double)__uint_as_float(*a.retmax), a.bits);
        if (lam_fix == lam_t) return;  // usual case: A'q already correct
    }
    unsigned long long cnt = 0;
    float ret = 0.0f;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        float x[VPT * 4];
        load_row<VPT>(a.x + (int64_t)r * a.ld, a.cols, vec, x);
        const double lam = a.vec ? a.lam[r] : lam_t;
        const double t = a.do_select ? threshold_of(a.policy, a.thr_m, a.stat[r], scale_other, a.cols)
                                     : 0.0;
        if (!a.fix_mode) {
            if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
            __syncthreads();
        }
        int rq[VPT * 4], rd[VPT * 4];
#pragma unroll
        for (int e = 0; e < VPT * 4; ++e) {
            const int c = (e / 4 * kThreads + (int)threadIdx.x) * 4 + (e & 3);
            const bool in = c < a.cols;
            const bool keep = a.do_select && in && fabs((double)x[e]) > t;
            if (a.fix_mode) {
                rd[e] = keep ? quantize_scalar((double)x[e], lam_fix, qmax, a.rounding) : 0;
                rq[e] = 0;
            } else {
                const int q = quantize_scalar((double)x[e], lam, qmax, a.rounding);
                const float res = __fsub_rn(x[e], lut[q + qmax]);
                rq[e] = quantize_scalar((double)res, lam_r, qmax, a.rounding);
                rd[e] = keep ? q : 0;
                cnt += keep;
                if (keep) ret = fmaxf(ret, fabsf(x[e]));
            }
        }
        if (!a.fix_mode) store_row_i8<VPT>(a.rq + (int64_t)r * a.ldq, a.cols, vec, rq);
        if (a.do_select) store_row_i8<VPT>(a.red + (int64_t)r * a.ldq, a.cols, vec, rd);
        if (!a.fix_mode) __syncthreads();
    }
    if (!a.fix_mode && a.do_select) {
        cnt = block_sum_u64(cnt, redu);
        ret = block_max(ret, red);
        if (threadIdx.x == 0) {
            if (cnt) atomicAdd(a.nnz, cnt);
            atomicMax(a.retmax, fbits(ret));
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_select_rows_generic(const SelectArgs a) {
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    __shared__ unsigned long long redu[kThreads / 32];
    const int qmax = quant_max(a.bits);
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double scale_other =
        a.do_select && a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                                        : 1.0;
    double lam_fix = 0.0;
    if (a.fix_mode) {
        lam_fix = compute_scale((double)__uint_as_float(*a.retmax), a.bits);
        if (lam_fix == lam_t) return;
    }
    unsigned long long cnt = 0;
    float ret = 0.0f;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        const float* row = a.x + (int64_t)r * a.ld;
        const double lam = a.vec ? a.lam[r] : lam_t;
        const double t = a.do_select ? threshold_of(a.policy, a.thr_m, a.stat[r], scale_other, a.cols)
                                     : 0.0;
        if (!a.fix_mode) {
            if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
            __syncthreads();
        }
        for (int c = threadIdx.x; c < a.cols; c += kThreads) {
            const float v = row[c];
            const bool keep = a.do_select && fabs((double)v) > t;
            if (a.fix_mode) {
                a.red[(int64_t)r * a.ldq + c] =
                    (int8_t)(keep ? quantize_scalar((double)v, lam_fix, qmax, a.rounding) : 0);
            } else {
                const int q = quantize_scalar((double)v, lam, qmax, a.rounding);
                a.rq[(int64_t)r * a.ldq + c] = (int8_t)quantize_scalar(
                    (double)__fsub_rn(v, lut[q + qmax]), lam_r, qmax, a.rounding);
                if (a.do_select) a.red[(int64_t)r * a.ldq + c] = (int8_t)(keep ? q : 0);
                cnt += keep;
                if (keep) ret = fmaxf(ret, fabsf(v));
            }
        }
        if (!a.fix_mode) __syncthreads();
    }
    if (!a.fix_mode && a.do_select) {
        cnt = block_sum_u64(cnt, redu);
        ret = block_max(ret, red);
        if (threadIdx.x == 0) {
            if (cnt) atomicAdd(a.nnz, cnt);
            atomicMax(a.retmax, fbits(ret));
        }
    }
}

// ----------------------------------------------------------- K3 columns --
// B side: RBq^T and B'q^T (both N x K, K-major), column thresholds t_j.
__global__ void __launch_bounds__(kThreads) k_select_cols_T(const SelectArgs a) {
    __shared__ __align__(16) int8_t trq[kTN][kTK + 16];
    __shared__ __align__(16) int8_t tred[kTN][kTK + 16];
    __shared__ double lam_s[kTN];
    __shared__ double thr_s[kTN];
    __shared__ float red[kThreads / 32];
    __shared__ unsigned long long redu[kThreads / 32];
    const int n0 = blockIdx.x * kTN, k0 = blockIdx.y * kTK;
    const int qmax = quant_max(a.bits);
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    double lam_fix = 0.0;
    if (a.fix_mode) {
        lam_fix = compute_scale((double)__uint_as_float(*a.retmax), a.bits);
        if (lam_fix == lam_t) return;
    }
    if (threadIdx.x < kTN) {
        const int c = min(n0 + (int)threadIdx.x, a.cols - 1);
        lam_s[threadIdx.x] = a.vec ? a.lam[c] : lam_t;
        if (a.do_select) {
            const double so = a.policy == kMin
                                  ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                                  : 1.0;
            thr_s[threadIdx.x] = threshold_of(a.policy, a.thr_m, a.stat[c], so, a.rows);
        }
    }
    __syncthreads();
    const int cg = (threadIdx.x & 15) * 4;
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (n0 + cg + 3 < a.cols);
    unsigned long long cnt = 0;
    float ret = 0.0f;
#pragma unroll 2
    for (int i = 0; i < kTK / 16; ++i) {
        const int kr = (threadIdx.x >> 4) + 16 * i;
        const int k = k0 + kr;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (k < a.rows) {
            const float* p = a.x + (int64_t)k * a.ld + n0 + cg;
            if (vec) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(p));
                v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = (n0 + cg + e < a.cols) ? p[e] : 0.f;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool in = k < a.rows && n0 + cg + e < a.cols;
            const bool keep = a.do_select && in && fabs((double)v[e]) > thr_s[cg + e];
            if (a.fix_mode) {
                tred[cg + e][kr] = (int8_t)(keep ? quantize_scalar((double)v[e], lam_fix, qmax, a.rounding) : 0);
            } else {
                const double lam = lam_s[cg + e];
                const int q = quantize_scalar((double)v[e], lam, qmax, a.rounding);
                const float res = __fsub_rn(v[e], dequant_value(q, lam));
                trq[cg + e][kr] = (int8_t)quantize_scalar((double)res, lam_r, qmax, a.rounding);
                tred[cg + e][kr] = (int8_t)(keep ? q : 0);
                cnt += keep;
                if (keep) ret = fmaxf(ret, fabsf(v[e]));
            }
        }
    }
    __syncthreads();
    if (!a.fix_mode) store_T_tile(trq, a.rq, a.ldq, n0, k0, a.cols, a.rows);
    if (a.do_select) store_T_tile(tred, a.red, a.ldq, n0, k0, a.cols, a.rows);
    if (!a.fix_mode && a.do_select) {
        cnt = block_sum_u64(cnt, redu);
        ret = block_max(ret, red);
        if (threadIdx.x == 0) {
            if (cnt) atomicAdd(a.nnz, cnt);
            atomicMax(a.retmax, fbits(ret));
        }
    }
}

// ------------------------------------------------------------- scalars --
__global__ void k_lambdas(DevScalars* sc, int bits) {
    sc->lamA = compute_scale((double)__uint_as_float(sc->maxA), bits);
    sc->lamB = compute_scale((double)__uint_as_float(sc->maxB), bits);
}

// Density, dispatch (pipeline.cpp:106-111) and the per-tensor scales the
// compensation epilogue reads.
__global__ void k_dispatch(DevScalars* sc, int bits, int64_t MK, int64_t KN, double s, int reduce) {
    sc->lamRA = compute_scale((double)__uint_as_float(sc->maxRA), bits);
    sc->lamRB = compute_scale((double)__uint_as_float(sc->maxRB), bits);
    sc->lamAred = compute_scale((double)__uint_as_float(sc->retA), bits);
    sc->lamBred = compute_scale((double)__uint_as_float(sc->retB), bits);
    if (reduce) {
        const double da = __ddiv_rn((double)sc->nnzA, (double)MK);
        const double db = __ddiv_rn((double)sc->nnzB, (double)KN);
        sc->densA = da;
        sc->densB = db;
        const int sparse = fmax(da, db) < s;
        sc->sel = sparse;
        sc->path = sparse ? kSparse : kDense;
    } else {
        sc->densA = sc->densB = 0.0;
        sc->sel = 0;
        sc->path = kDense;
    }
}

__global__ void k_fill_u32(uint32_t* p, uint32_t v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_rows(int rows) { return rows < kNumSMs * 16 ? rows : kNumSMs * 16; }

}  // namespace

// ----------------------------------------------------------------- launches --
void launch_absmax_global(const float* x, int64_t n, uint32_t* gmax, int* nonfinite,
                          cudaStream_t s) {
    int64_t blocks = (n / 4 + kThreads - 1) / kThreads;
    blocks = blocks < 1 ? 1 : blocks > kNumSMs * 8 ? kNumSMs * 8 : blocks;
    k_absmax_global<<<(int)blocks, kThreads, 0, s>>>(x, n, gmax, nonfinite);
}

void launch_absmax_cols(const float* x, int rows, int cols, int64_t ld, uint32_t* colmax,
                        uint32_t* gmax, int* nonfinite, cudaStream_t s) {
    dim3 grid((cols + kThreads * 4 - 1) / (kThreads * 4), (rows + kColSlab - 1) / kColSlab);
    k_absmax_cols<<<grid, kThreads, 0, s>>>(x, rows, cols, ld, colmax, gmax, nonfinite);
}

void launch_quant_rows(const QuantRowsArgs& a, cudaStream_t s) {
    const int g = grid_rows(a.rows);
    const int vpt = (a.cols + kThreads * 4 - 1) / (kThreads * 4);
    if (vpt <= 1) k_quant_rows<1><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 2) k_quant_rows<2><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 4) k_quant_rows<4><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 8) k_quant_rows<8><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 16) k_quant_rows<16><<<g, kThreads, 0, s>>>(a);
    else k_quant_rows_generic<<<g, kThreads, 0, s>>>(a);
}

void launch_quant_cols_T(const QuantColsArgs& a, cudaStream_t s) {
    dim3 grid((a.cols + kTN - 1) / kTN, (a.rows + kTK - 1) / kTK);
    k_quant_cols_T<<<grid, kThreads, 0, s>>>(a);
}

void launch_select_rows(const SelectArgs& a, cudaStream_t s) {
    const int g = grid_rows(a.rows);
    const int vpt = (a.cols + kThreads * 4 - 1) / (kThreads * 4);
    if (vpt <= 1) k_select_rows<1><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 2) k_select_rows<2><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 4) k_select_rows<4><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 8) k_select_rows<8><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 16) k_select_rows<16><<<g, kThreads, 0, s>>>(a);
    else k_select_rows_generic<<<g, kThreads, 0, s>>>(a);
}

void launch_select_cols_T(const SelectArgs& a, cudaStream_t s) {
    dim3 grid((a.cols + kTN - 1) / kTN, (a.rows + kTK - 1) / kTK);
    k_select_cols_T<<<grid, kThreads, 0, s>>>(a);
}

void launch_lambdas(DevScalars* sc, int bits, cudaStream_t s) { k_lambdas<<<1, 1, 0, s>>>(sc, bits); }

void launch_dispatch(DevScalars* sc, int bits, int64_t MK, int64_t KN, double density_limit,
                     int reduce, cudaStream_t s) {
    k_dispatch<<<1, 1, 0, s>>>(sc, bits, MK, KN, density_limit, reduce);
}

void fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t s) {
    int64_t blocks = (n + 255) / 256;
    blocks = blocks < 1 ? 1 : blocks > 4096 ? 4096 : blocks;
    k_fill_u32<<<(int)blocks, 256, 0, s>>>(p, v, n);
}

}  // namespace xg
