// K1 (quantiser) and K3 (residual quantisation + threshold selection).
//
// HBM-bound byte work.  Design rules that the profile (profiles/) forced:
//  * the per-element quantisation runs in fp32 with a proven error margin and
//    an exact fp64 fallback (quantize.cpp:13-24 semantics) taken once per quad
//    of elements, rounding mode is a template parameter (no per-element
//    branches), and ints are packed from the float bit patterns;
//  * dequantisation float(q / lambda) is a 255-entry table per scale: one per
//    row for A (broadcast-ish LDS), column-interleaved lut[q][col] for B so the
//    32 lanes (32 different columns) hit 32 different banks;
//  * rows are held in registers (one HBM read per pass); B column tiles are
//    staged transposed through conflict-free [64][33]-word shared arrays so the
//    K-major int8 outputs leave as 16-byte stores.
//
// Replaces (reference, proj/src/):
//   quantize / quantize_with_scales / slice_max_abs   quantize.cpp:28-36,107-150
//   DenseMatrix::all_finite / max_abs                 matrix.cpp:44-58
//   dequantize + subtract (max|R|)                    quantize.cpp:152-167, pipeline.cpp:79-84
//   residual quantize (always per-tensor)             pipeline.cpp:86-93
//   reduce_a / reduce_b (+density, quantize_csr values) sparse.cpp:36-95,193-240
#include <cuda.h>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "internal.h"

namespace xg {

namespace {

constexpr int kThreads = 256;

// Early exit of the table-driven kernels once a non-finite input was seen
// (block-uniform: every thread reads the same flag).
#define XG_EXIT_IF_NONFINITE(flagp) \
    if ((flagp) && *(volatile const int*)(flagp)) return

template <int NT = kThreads>
__device__ __forceinline__ float block_max(float v, float* red) {
    v = warp_maxf(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float r = red[0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) r = fmaxf(r, red[i]);
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

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// ---- fp32 quantiser (see quantize32 in common.cuh for the error analysis) --
// Valid for |x*lambda| <= qmax (1 + 2^-52) (always so inside the pipeline);
// anything outside, NaN, or within the error margin of a rounding boundary
// raises `slow`, and the caller redoes the quad exactly.
template <int RND>
__device__ __forceinline__ int q32(float x, float lam32, float qlim, bool& slow) {
    const float t = __fmul_rn(x, lam32);
    if (RND == kNearest) {
        const float u = __fadd_rn(t, kMagic);  // rint, ties-even
        const float d = fabsf(__fsub_rn(t, __fsub_rn(u, kMagic)));
        slow |= !(d < 0.4999f) | !(fabsf(t) <= qlim);
        return __float_as_int(u) - 0x4B400000;
    } else {
        const float r = truncf(t);
        const float d = fabsf(__fsub_rn(t, r));
        slow |= (!(d >= 2e-4f && d <= 0.9998f) & (fabsf(t) > 0.5f)) | !(fabsf(t) <= qlim);
        return __float_as_int(__fadd_rn(r, kMagic)) - 0x4B400000;
    }
}

__device__ __forceinline__ int qexact(float x, double lam, float qmaxf, int rnd) {
    return quantize_slow(x, lam, qmaxf, rnd);
}

// Row element e of this thread: column (v*NT + tid)*4 + (e%4).
template <int VPT, int NT>
__device__ __forceinline__ void load_row(const float* __restrict__ row, int cols, bool vec,
                                         float (&x)[VPT * 4]) {
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int c = (v * NT + (int)threadIdx.x) * 4;
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

__device__ __forceinline__ void store_quad(int8_t* __restrict__ row, int c, int cols, bool vec,
                                           uint32_t packed) {
    if (vec && c + 3 < cols) {
        *reinterpret_cast<uint32_t*>(row + c) = packed;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (c + e < cols) row[c + e] = (int8_t)(packed >> (8 * e));
    }
}

// ------------------------------------------------------------------ K1 rows --
// One CTA per row, the row held in registers.  PerRow: row absmax -> lambda_i;
// quantise; residual through a 255-entry per-row table of float(q / lambda_i);
// max|residual|.  Non-finite codes: bit 0 = an infinite slice max (the
// reference's compute_scale throws), bit 1 = any NaN/inf (all_finite fails).
template <int VPT, int RND>
__global__ void __launch_bounds__(kThreads) k_quant_rows(const QuantRowsArgs a) {
    XG_PDL_WAIT();
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax;
    const float qlim = qmaxf + 0.25f;
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (a.ldq % 4 == 0);
    float rmax_acc = 0.0f, gmax_acc = 0.0f;
    int bad = 0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        float x[VPT * 4];
        load_row<VPT, kThreads>(a.x + (int64_t)r * a.ld, a.cols, vec, x);
        float m = 0.0f, s = 0.0f;
#pragma unroll
        for (int e = 0; e < VPT * 4; ++e) {
            m = fmaxf(m, fabsf(x[e]));
            s = __fadd_rn(s, x[e]);  // NaN / inf propagate (finite overflow is re-checked)
        }
        if (!(fabsf(s) <= FLT_MAX)) {
#pragma unroll
            for (int e = 0; e < VPT * 4; ++e) bad |= fabsf(x[e]) <= FLT_MAX ? 0 : 2;
        }
        m = block_max(m, red);
        bad |= m > FLT_MAX ? 1 : 0;
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);  // slice_max_abs: fp64 max == float max
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
            if (threadIdx.x == 0 && a.rcp_out) a.rcp_out[r] = ff_recip(lam);
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        const float lam32 = __double2float_rn(lam);
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        float rm = 0.0f;
        int8_t* qrow = a.q + (int64_t)r * a.ldq;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            bool slow = false;
            int q[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) q[e] = q32<RND>(x[4 * v + e], lam32, qlim, slow);
            if (slow) {
#pragma unroll
                for (int e = 0; e < 4; ++e) q[e] = qexact(x[4 * v + e], lam, qmaxf, RND);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) rm = fmaxf(rm, fabsf(__fsub_rn(x[4 * v + e], lut[q[e] + qmax])));
            store_quad(qrow, (v * kThreads + (int)threadIdx.x) * 4, a.cols, vec, pack4(q[0], q[1], q[2], q[3]));
        }
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
// served from L2.  Exact scalar path throughout.
__global__ void __launch_bounds__(kThreads) k_quant_rows_generic(const QuantRowsArgs a) {
    XG_PDL_WAIT();
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
            bad |= fabsf(v) <= FLT_MAX ? 0 : 2;
        }
        m = block_max(m, red);
        bad |= m > FLT_MAX ? 1 : 0;
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
            if (threadIdx.x == 0 && a.rcp_out) a.rcp_out[r] = ff_recip(lam);
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        float rm = 0.0f;
        for (int c = threadIdx.x; c < a.cols; c += kThreads) {
            const float v = row[c];
            const int q = quantize_fast((double)v, lam, (double)qmax, a.rounding);
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
    XG_PDL_WAIT();
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
    XG_PDL_WAIT();
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

// ---------------------------------------------------- column tiles (B side) --
// ---------------------------------------------------- column tiles (B side) --
// Tiles of 64 columns (N) x 128 rows (K) of a row-major K x N matrix whose ints
// are written transposed (N x K, K-major: the tensor-core B layout).  Warp w
// owns rows [16w, 16w+16) of the tile, lane l owns columns l and 32+l, so every
// global load is a coalesced 128-byte row segment and every thread packs 4
// consecutive K bytes into one 32-bit shared-memory word; the [64][33]-word
// staging array makes both the packed writes and the row-wise read-out
// bank-conflict free.  A CTA walks kColSub such tiles down the columns so the
// per-column dequant tables (built once per CTA) are amortised.
constexpr int kTK = 128, kTN = 64, kTW = kTK / 4 + 1;
constexpr int kColSub = 8;
constexpr int kColTileRows = kTK * kColSub;
constexpr int kLutBytes = 256 * kTN * 4;  // lut[q + qmax][column]

__device__ __forceinline__ void store_T_tile(const uint32_t (*t)[kTW], int8_t* dst, int64_t ldq,
                                             int n0, int k0, int cols, int rows) {
    const int r = threadIdx.x >> 2;     // 0..63 output row (column n of the input)
    const int seg = threadIdx.x & 3;    // 32-byte segment of the 128-byte row
    if (n0 + r >= cols) return;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = t[r][seg * 8 + i];
    int8_t* d = dst + (int64_t)(n0 + r) * ldq + k0 + seg * 32;
    const int kval = rows - (k0 + seg * 32);
    if (kval >= 32 && (ldq % 16) == 0) {
        reinterpret_cast<uint4*>(d)[0] = make_uint4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<uint4*>(d)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else if (kval > 0) {
        for (int j = 0; j < 32 && j < kval; ++j) d[j] = (int8_t)(w[j >> 2] >> (8 * (j & 3)));
    }
}

// v[c][i] = X[k0 + 16w + i][n0 + 32c + lane]
__device__ __forceinline__ void load_col_tile(const float* __restrict__ x, int rows, int cols,
                                              int64_t ld, int n0, int k0, float (&v)[2][16]) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int n = n0 + 32 * c + lane;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = k0 + 16 * w + i;
            v[c][i] = (n < cols && k < rows) ? __ldg(x + (int64_t)k * ld + n) : 0.0f;
        }
    }
}

__device__ __forceinline__ void build_col_luts(float (*lut)[kTN], const double* lam_s, int qmax) {
    for (int i = threadIdx.x; i < (2 * qmax + 1) * kTN; i += kThreads) {
        const int e = i / kTN, c = i % kTN;
        lut[e][c] = dequant_value(e - qmax, lam_s[c]);
    }
}

template <int RND>
__global__ void __launch_bounds__(kThreads) k_quant_cols_T(const QuantColsArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    extern __shared__ float4 dyn_smem[];
    float(*lut)[kTN] = reinterpret_cast<float(*)[kTN]>(dyn_smem);
    __shared__ uint32_t tq[kTN][kTW];
    __shared__ double lam_s[kTN];
    __shared__ float red[kThreads / 32];
    const int n0 = blockIdx.x * kTN;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax, qlim = qmaxf + 0.25f;
    if (threadIdx.x < kTN) {
        const int n = min(n0 + (int)threadIdx.x, a.cols - 1);
        const double lam = a.per_col ? compute_scale((double)__uint_as_float(a.colmax[n]), a.bits)
                                     : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        lam_s[threadIdx.x] = lam;
        if (a.per_col && blockIdx.y == 0 && a.lam_out && n0 + (int)threadIdx.x < a.cols) a.lam_out[n] = lam;
        if (a.per_col && blockIdx.y == 0 && a.rcp_out && n0 + (int)threadIdx.x < a.cols) a.rcp_out[n] = ff_recip(lam);
    }
    __syncthreads();
    build_col_luts(lut, lam_s, qmax);
    const double lamc[2] = {lam_s[lane], lam_s[32 + lane]};
    const float l32[2] = {__double2float_rn(lamc[0]), __double2float_rn(lamc[1])};
    __syncthreads();
    float rm = 0.0f;
    for (int sub = 0; sub < kColSub; ++sub) {
        const int k0 = blockIdx.y * kColTileRows + sub * kTK;
        if (k0 >= a.rows) break;  // uniform
        float v[2][16];
        load_col_tile(a.x, a.rows, a.cols, a.ld, n0, k0, v);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                bool slow = false;
                int q[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) q[e] = q32<RND>(v[c][4 * g + e], l32[c], qlim, slow);
                if (slow) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) q[e] = qexact(v[c][4 * g + e], lamc[c], qmaxf, RND);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    rm = fmaxf(rm, fabsf(__fsub_rn(v[c][4 * g + e], lut[q[e] + qmax][32 * c + lane])));
                tq[32 * c + lane][4 * w + g] = pack4(q[0], q[1], q[2], q[3]);
            }
        }
        __syncthreads();
        store_T_tile(tq, a.qT, a.ldq, n0, k0, a.cols, a.rows);
        __syncthreads();
    }
    rm = block_max(rm, red);
    if (threadIdx.x == 0 && a.rmax) atomicMax(a.rmax, fbits(rm));
}

// ------------------------------------------------------------- K3 rows --
// Per row i of A: RAq = quantize(a - deq(aq), lambda_RA) and the reduced
// operand A'q = (|a| > t_i) ? aq : 0 (quantize_csr values equal aq under
// PerRow scales; under PerTensor the retained-max scale is checked afterwards
// and a fix-up pass rewrites A'q if it differs).  No row reduction precedes the
// element work, so the row is streamed (low registers, full occupancy).
__device__ __forceinline__ double threshold_of(int policy, double thr_m, float stat,
                                               double scale_other, int inner) {
    // sparse.cpp:49-55
    if (policy == kAvg) return __dmul_rn(thr_m, (double)stat);
    return __ddiv_rn(__dmul_rn(__dmul_rn(thr_m, scale_other), (double)stat), (double)inner);
}

// Stage dump: OR the kept bits of the quad at columns c..c+3 (c % 4 == 0) of
// row r into the bitmask (sparse.cpp:61-71 keep test, |x| > t  <=>  |x| >= tf).
__device__ __forceinline__ void dump_keep4(const SelectArgs& a, int r, int c, const float (&x)[4], float tf) {
    uint32_t nib = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) nib |= (fabsf(x[e]) >= tf ? 1u : 0u) << e;
    if (nib) atomicOr(&a.keep[(int64_t)r * a.keep_ld + (c >> 5)], nib << (c & 31));
}

// One quad of the selection: q (main scale), rq (residual scale), red (kept q).
template <int RND>
__device__ __forceinline__ void select_quad(const float (&x)[4], const float* lutp, int lstride,
                                            double lam, float lam32, double lam_r, float lam_r32,
                                            float tf, float qmaxf, float qlim, int qmax,
                                            uint32_t& pq, uint32_t& pr, unsigned long long& cnt,
                                            float& ret) {
    bool slow = false;
    int q[4], rq[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) q[e] = q32<RND>(x[e], lam32, qlim, slow);
#pragma unroll
    for (int e = 0; e < 4; ++e)
        rq[e] = q32<RND>(__fsub_rn(x[e], lutp[(q[e] + qmax) * lstride]), lam_r32, qlim, slow);
    if (slow) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            q[e] = qexact(x[e], lam, qmaxf, RND);
            rq[e] = qexact(__fsub_rn(x[e], lutp[(q[e] + qmax) * lstride]), lam_r, qmaxf, RND);
        }
    }
    int d[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const bool keep = fabsf(x[e]) >= tf;
        d[e] = keep ? q[e] : 0;
        cnt += keep;
        ret = fmaxf(ret, keep ? fabsf(x[e]) : 0.0f);
    }
    pq = pack4(rq[0], rq[1], rq[2], rq[3]);
    pr = pack4(d[0], d[1], d[2], d[3]);
}

template <int RND>
__global__ void __launch_bounds__(kThreads) k_select_rows(const SelectArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    __shared__ float lut[256];
    __shared__ float red[kThreads / 32];
    __shared__ unsigned long long redu[kThreads / 32];
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax, qlim = qmaxf + 0.25f;
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (a.ldq % 4 == 0) && (a.cols % 4 == 0);
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const float lam_r32 = __double2float_rn(lam_r);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double scale_other =
        a.do_select && a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                                        : 1.0;
    unsigned long long cnt = 0;
    float ret = 0.0f;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        const float* row = a.x + (int64_t)r * a.ld;
        int8_t* rq_row = a.rq + (int64_t)r * a.ldq;
        int8_t* rd_row = a.do_select ? a.red + (int64_t)r * a.ldq : nullptr;
        const double lam = a.vec ? a.lam[r] : lam_t;
        const float lam32 = __double2float_rn(lam);
        const float tf = a.do_select
                             ? float_above(threshold_of(a.policy, a.thr_m, a.stat[r], scale_other, a.cols))
                             : __int_as_float(0x7f800000);
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        if (vec) {
#pragma unroll 2
            for (int c = threadIdx.x * 4; c < a.cols; c += kThreads * 4) {
                const float4 f = __ldg(reinterpret_cast<const float4*>(row + c));
                const float x[4] = {f.x, f.y, f.z, f.w};
                uint32_t pq, pr;
                select_quad<RND>(x, lut, 1, lam, lam32, lam_r, lam_r32, tf, qmaxf, qlim, qmax, pq, pr,
                                 cnt, ret);
                *reinterpret_cast<uint32_t*>(rq_row + c) = pq;
                if (rd_row) *reinterpret_cast<uint32_t*>(rd_row + c) = pr;
                if (a.keep) dump_keep4(a, r, c, x, tf);
            }
        } else {
            for (int c = threadIdx.x; c < a.cols; c += kThreads) {
                const float v = row[c];
                const int q = quantize_fast((double)v, lam, (double)qmax, RND);
                rq_row[c] = (int8_t)quantize_fast((double)__fsub_rn(v, lut[q + qmax]), lam_r, (double)qmax, RND);
                const bool keep = fabsf(v) >= tf;
                if (rd_row) rd_row[c] = (int8_t)(keep ? q : 0);
                if (a.keep && keep) atomicOr(&a.keep[(int64_t)r * a.keep_ld + (c >> 5)], 1u << (c & 31));
                cnt += keep && a.do_select;
                ret = fmaxf(ret, keep ? fabsf(v) : 0.0f);
            }
        }
        __syncthreads();
    }
    if (a.do_select) {
        cnt = block_sum_u64(cnt, redu);
        ret = block_max(ret, red);
        if (threadIdx.x == 0) {
            if (cnt) atomicAdd(a.nnz, cnt);
            atomicMax(a.retmax, fbits(ret));
        }
    }
}

// PerTensor reduced operand whose retained-max scale differs from the operand
// scale (sparse.cpp:198-203): rewrite the kept ints with lambda'.  Exits at
// once in the usual case lambda' == lambda.  Exact scalar path (rare).
__global__ void __launch_bounds__(kThreads) k_fix_rows(const SelectArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    const double lam_t = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double lam_fix = compute_scale((double)__uint_as_float(*a.retmax), a.bits);
    if (lam_fix == lam_t) return;
    const int qmax = quant_max(a.bits);
    const double so = a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits) : 1.0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        const float tf = float_above(threshold_of(a.policy, a.thr_m, a.stat[r], so, a.cols));
        for (int c = threadIdx.x; c < a.cols; c += kThreads) {
            const float v = a.x[(int64_t)r * a.ld + c];
            a.red[(int64_t)r * a.ldq + c] =
                (int8_t)(fabsf(v) >= tf ? quantize_fast((double)v, lam_fix, (double)qmax, a.rounding) : 0);
        }
    }
}

// B side: column j of the reduced operand is row j of B'q^T.
__global__ void __launch_bounds__(kThreads) k_fix_cols_T(const SelectArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    const double lam_t = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double lam_fix = compute_scale((double)__uint_as_float(*a.retmax), a.bits);
    if (lam_fix == lam_t) return;
    const int qmax = quant_max(a.bits);
    const double so = a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits) : 1.0;
    for (int n = blockIdx.x; n < a.cols; n += gridDim.x) {
        const float tf = float_above(threshold_of(a.policy, a.thr_m, a.stat[n], so, a.rows));
        for (int k = threadIdx.x; k < a.rows; k += kThreads) {
            const float v = a.x[(int64_t)k * a.ld + n];
            a.red[(int64_t)n * a.ldq + k] =
                (int8_t)(fabsf(v) >= tf ? quantize_fast((double)v, lam_fix, (double)qmax, a.rounding) : 0);
        }
    }
}

// ----------------------------------------------------------- K3 columns --
// B side: RBq^T and B'q^T (both N x K, K-major), column thresholds t_j.
template <int RND>
__global__ void __launch_bounds__(kThreads) k_select_cols_T(const SelectArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    extern __shared__ float4 dyn_smem[];
    float(*lut)[kTN] = reinterpret_cast<float(*)[kTN]>(dyn_smem);
    __shared__ uint32_t trq[kTN][kTW];
    __shared__ uint32_t tred[kTN][kTW];
    __shared__ double lam_s[kTN];
    __shared__ float red[kThreads / 32];
    __shared__ unsigned long long redu[kThreads / 32];
    const int n0 = blockIdx.x * kTN;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax, qlim = qmaxf + 0.25f;
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const float lam_r32 = __double2float_rn(lam_r);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double so = a.do_select && a.policy == kMin
                          ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                          : 1.0;
    if (threadIdx.x < kTN) {
        const int n = min(n0 + (int)threadIdx.x, a.cols - 1);
        lam_s[threadIdx.x] = a.vec ? a.lam[n] : lam_t;
    }
    __syncthreads();
    build_col_luts(lut, lam_s, qmax);
    double lamc[2];
    float l32[2], tf[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int nraw = n0 + 32 * c + lane;
        const int n = min(nraw, a.cols - 1);
        lamc[c] = lam_s[32 * c + lane];
        l32[c] = __double2float_rn(lamc[c]);
        tf[c] = (a.do_select && nraw < a.cols)
                    ? float_above(threshold_of(a.policy, a.thr_m, a.stat[n], so, a.rows))
                    : __int_as_float(0x7f800000);
    }
    __syncthreads();
    unsigned long long cnt = 0;
    float ret = 0.0f;
    for (int sub = 0; sub < kColSub; ++sub) {
        const int k0 = blockIdx.y * kColTileRows + sub * kTK;
        if (k0 >= a.rows) break;  // uniform
        float v[2][16];
        load_col_tile(a.x, a.rows, a.cols, a.ld, n0, k0, v);  // rows past K load as 0: never kept
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float x[4] = {v[c][4 * g], v[c][4 * g + 1], v[c][4 * g + 2], v[c][4 * g + 3]};
                uint32_t pq, pr;
                select_quad<RND>(x, &lut[0][32 * c + lane], kTN, lamc[c], l32[c], lam_r, lam_r32, tf[c],
                                 qmaxf, qlim, qmax, pq, pr, cnt, ret);
                if (a.keep && n0 + 32 * c + lane < a.cols && k0 + 16 * w + 4 * g < a.rows)
                    dump_keep4(a, n0 + 32 * c + lane, k0 + 16 * w + 4 * g, x, tf[c]);
                trq[32 * c + lane][4 * w + g] = pq;
                tred[32 * c + lane][4 * w + g] = pr;
            }
        }
        __syncthreads();
        store_T_tile(trq, a.rq, a.ldq, n0, k0, a.cols, a.rows);
        if (a.do_select) store_T_tile(tred, a.red, a.ldq, n0, k0, a.cols, a.rows);
        __syncthreads();
    }
    if (a.do_select) {
        cnt = block_sum_u64(cnt, redu);
        ret = block_max(ret, red);
        if (threadIdx.x == 0) {
            if (cnt) atomicAdd(a.nnz, cnt);
            atomicMax(a.retmax, fbits(ret));
        }
    }
}


// =================================================================== fast path
// Nearest rounding (the pipeline default), per-element cost ~15 instructions.
// Inside the pipeline |x * lambda| <= qmax (1 + 2^-52) because lambda is
// qmax / max|slice|, so no range test is needed: u = RN(t + 1.5*2^23) holds
// rint(t) in its low mantissa bits, |t - rint(t)| is accumulated with one
// FMNMX per element and a quad whose maximum reaches 0.4999 (a possible
// llround tie within the fp32 error bound) is redone exactly.  Rows / columns
// whose lambda32 is not a finite float, or that contain a NaN, take the exact
// path as a whole (uniform branch).  Table lookups address shared memory
// straight from the u bit pattern.
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
// table entry at adj + (u << SHIFT): one IMAD (adj already holds the -(magic << SHIFT) bias;
// opaque_u32 keeps the compiler from splitting the bias back out into a second add per lookup)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    uint32_t o;  // a shuffle with the own lane: opaque to ptxas's reassociation
    asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(o) : "r"(v), "r"((int)(threadIdx.x & 31)));
    return o;
}
template <int SHIFT>
__device__ __forceinline__ float lut_at(uint32_t u, uint32_t adj) {
    uint32_t a;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(u), "n"(1 << SHIFT), "r"(adj));
    return lds_f32(a);
}
// NaN-propagating max (PTX max.NaN): a NaN input makes dmax NaN, which sends
// the quad to the exact path (quantize.cpp:13-24 maps NaN to -qmax).
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// u = RN(x*lam32 + 1.5*2^23) rounds the exact product to an integer in one FMA
// (ties to even; a tie is excluded by the test below), and the distance of the
// exact product from that integer comes from a second FMA: 4 instructions.
// |x*lam32 - x*lam| <= 2^-24*|x*lam| <= 8e-6 for |x*lam| <= qmax, far inside the
// 1e-4 margin, so the reference's llround(double(x)*lam) is the same integer.
__device__ __forceinline__ uint32_t qn(float x, float lam32, float& dmax) {
    const float u = __fmaf_rn(x, lam32, kMagic);
    dmax = fmax_nan(dmax, fabsf(__fmaf_rn(x, lam32, -__fsub_rn(u, kMagic))));
    return __float_as_uint(u);
}
__device__ __forceinline__ uint32_t ubits(int q) { return (uint32_t)(q + 0x4B400000); }

// The same for 4 values with packed fp32x2 FMA/SUB (FFMA2 / FADD2: two IEEE
// round-to-nearest operations per instruction, results identical to qn's):
// u = RN(x*lam32 + magic), d = RN(x*lam32 + (magic - u)).
__device__ __forceinline__ void qn4(const float (&x)[4], float lam32, uint32_t (&u)[4], float& dmax) {
    const uint64_t L = pk2(lam32, lam32), MG = pk2(kMagic, kMagic);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const uint64_t X = pk2(x[2 * p], x[2 * p + 1]);
        const uint64_t U = fma2(X, L, MG);
        const uint64_t D = fma2(X, L, sub2(MG, U));
        float u0, u1, d0, d1;
        upk2(U, u0, u1);
        upk2(D, d0, d1);
        u[2 * p] = __float_as_uint(u0);
        u[2 * p + 1] = __float_as_uint(u1);
        dmax = fmax_nan(fmax_nan(dmax, fabsf(d0)), fabsf(d1));
    }
}
// Floor (quantize.cpp:16-20: 4-eps nudge away from zero, then truncation): u =
// the bits of magic + trunc(t), from floor(|t|) by a round-toward-zero add, and
// the distance of frac(|t|) from 0.5 in dmax - the fast result stands when
// frac lies in (2e-4, 1 - 2e-4), so neither the fp32 product's error (<= 1.5e-5
// at |t| <= 128) nor the nudge can move the truncation (the margin q32<kFloor> uses)
__device__ __forceinline__ uint32_t qf(float x, float lam32, float& dmax) {
    const float t = __fmul_rn(x, lam32);
    const float at = fabsf(t);
    const float f = __fadd_rz(at, kMagic);         // magic + floor(|t|)
    const float frac = __fsub_rn(at, __fsub_rn(f, kMagic));
    dmax = fmax_nan(dmax, fabsf(__fsub_rn(frac, 0.5f)));
    const uint32_t fb = __float_as_uint(f);
    return t < 0.0f ? 2u * 0x4B400000u - fb : fb;  // ubits(-floor(|t|)) for t < 0
}
// the quad quantiser of rounding mode RND and its acceptance bound on dmax
template <int RND>
__device__ __forceinline__ void qr4(const float (&x)[4], float lam32, uint32_t (&u)[4], float& dmax) {
    if constexpr (RND == kNearest) {
        qn4(x, lam32, u, dmax);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) u[e] = qf(x[e], lam32, dmax);
    }
}
template <int RND>
constexpr float qok() { return RND == kNearest ? 0.4999f : 0.4998f; }

__device__ __forceinline__ uint32_t pack4u(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

template <int VPT, int NT>
__global__ void __launch_bounds__(NT) k_quant_rows_fast(const QuantRowsArgs a) {
    XG_PDL_WAIT();
    __shared__ float lut[256];
    __shared__ float red[NT / 32];
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax;
    const bool vec = (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                     (a.ldq % 4 == 0);
    // lut[q + qmax] at smem address (u_bits << 2) + adj
    const uint32_t adj = smem_u32(lut) + 4u * (uint32_t)qmax - 4u * 0x4B400000u;
    float rmax_acc = 0.0f, gmax_acc = 0.0f;
    int bad = 0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x) {
        float x[VPT * 4];
        load_row<VPT, NT>(a.x + (int64_t)r * a.ld, a.cols, vec, x);
        float m = 0.0f, s = 0.0f;
#pragma unroll
        for (int e = 0; e < VPT * 4; ++e) {
            m = fmaxf(m, fabsf(x[e]));
            s = __fadd_rn(s, x[e]);  // NaN / inf propagate (finite overflow only costs the exact path)
        }
        const bool odd = !(fabsf(s) <= FLT_MAX);
        if (odd) {
#pragma unroll
            for (int e = 0; e < VPT * 4; ++e) bad |= fabsf(x[e]) <= FLT_MAX ? 0 : 2;
        }
        m = block_max<NT>(m, red);
        bad |= m > FLT_MAX ? 1 : 0;
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
            if (threadIdx.x == 0 && a.rcp_out) a.rcp_out[r] = ff_recip(lam);
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        const float lam32 = __double2float_rn(lam);
        const bool exact = odd || !(lam32 <= FLT_MAX);
        if (threadIdx.x <= 2 * qmax) lut[threadIdx.x] = dequant_value((int)threadIdx.x - qmax, lam);
        __syncthreads();
        float rm = 0.0f;
        int8_t* qrow = a.q + (int64_t)r * a.ldq;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            uint32_t u[4];
            float dmax = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) u[e] = qn(x[4 * v + e], lam32, dmax);
            if (exact || !(dmax < 0.4999f)) {
#pragma unroll
                for (int e = 0; e < 4; ++e) u[e] = ubits(qexact(x[4 * v + e], lam, qmaxf, kNearest));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) rm = fmaxf(rm, fabsf(__fsub_rn(x[4 * v + e], lut_at<2>(u[e], adj))));
            store_quad(qrow, (v * NT + (int)threadIdx.x) * 4, a.cols, vec, pack4u(u[0], u[1], u[2], u[3]));
        }
        rmax_acc = fmaxf(rmax_acc, rm);
        __syncthreads();  // lut reuse
    }
    rmax_acc = block_max<NT>(rmax_acc, red);
    if (threadIdx.x == 0) {
        if (a.rmax) atomicMax(a.rmax, fbits(rmax_acc));
        if (a.gmax) atomicMax(a.gmax, fbits(gmax_acc));
    }
    if (bad && a.nonfinite) atomicOr(a.nonfinite, bad);
}

// Selection quad, Nearest.  lut_adj: smem address of lut entry q = adj + (u << shift).
template <int SHIFT, int RND = kNearest>
__device__ __forceinline__ void select_quad_n(const float (&x)[4], uint32_t lut_adj, double lam,
                                              float lam32, double lam_r, float lam_r32, float tf,
                                              float qmaxf, bool exact, uint32_t& pq, uint32_t& pr,
                                              unsigned& cnt, float& lmax) {
    uint32_t u[4], ur[4];
    float dmax = 0.0f;
    qr4<RND>(x, lam32, u, dmax);
    float res[4];
#pragma unroll
    for (int p = 0; p < 2; ++p)  // residual x - deq(q), two per FADD2
        upk2(sub2(pk2(x[2 * p], x[2 * p + 1]),
                  pk2(lut_at<SHIFT>(u[2 * p], lut_adj), lut_at<SHIFT>(u[2 * p + 1], lut_adj))),
             res[2 * p], res[2 * p + 1]);
    qr4<RND>(res, lam_r32, ur, dmax);
    if (exact || !(dmax < qok<RND>())) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            u[e] = ubits(qexact(x[e], lam, qmaxf, RND));
            res[e] = __fsub_rn(x[e], lut_at<SHIFT>(u[e], lut_adj));
            ur[e] = ubits(qexact(res[e], lam_r, qmaxf, RND));
        }
    }
    uint32_t d[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float ax = fabsf(x[e]);
        const bool keep = ax >= tf;
        d[e] = keep ? u[e] : 0u;
        cnt += keep ? 1u : 0u;
        lmax = fmaxf(lmax, ax);
    }
    pq = pack4u(ur[0], ur[1], ur[2], ur[3]);
    pr = pack4u(d[0], d[1], d[2], d[3]);
}

__global__ void __launch_bounds__(kThreads) k_quant_cols_T_fast(const QuantColsArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    extern __shared__ float4 dyn_smem[];
    float(*lut)[kTN] = reinterpret_cast<float(*)[kTN]>(dyn_smem);
    __shared__ uint32_t tq[kTN][kTW];
    __shared__ double lam_s[kTN];
    __shared__ float red[kThreads / 32];
    const int n0 = blockIdx.x * kTN;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax;
    if (threadIdx.x < kTN) {
        const int n = min(n0 + (int)threadIdx.x, a.cols - 1);
        const double lam = a.per_col ? compute_scale((double)__uint_as_float(a.colmax[n]), a.bits)
                                     : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        lam_s[threadIdx.x] = lam;
        if (a.per_col && blockIdx.y == 0 && a.lam_out && n0 + (int)threadIdx.x < a.cols) a.lam_out[n] = lam;
        if (a.per_col && blockIdx.y == 0 && a.rcp_out && n0 + (int)threadIdx.x < a.cols) a.rcp_out[n] = ff_recip(lam);
    }
    __syncthreads();
    build_col_luts(lut, lam_s, qmax);
    double lamc[2];
    float l32[2];
    uint32_t adj[2];
    bool exact[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        lamc[c] = lam_s[32 * c + lane];
        l32[c] = __double2float_rn(lamc[c]);
        exact[c] = !(l32[c] <= FLT_MAX);
        // lut[q + qmax][32c + lane] = base + 256 (q + qmax) + 4 (32c + lane)
        adj[c] = smem_u32(lut) + 4u * (32 * c + lane) + 256u * (uint32_t)qmax - 256u * 0x4B400000u;
    }
    __syncthreads();
    float rm = 0.0f;
    for (int sub = 0; sub < kColSub; ++sub) {
        const int k0 = blockIdx.y * kColTileRows + sub * kTK;
        if (k0 >= a.rows) break;  // uniform
        float v[2][16];
        load_col_tile(a.x, a.rows, a.cols, a.ld, n0, k0, v);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t u[4];
                float dmax = 0.0f;
#pragma unroll
                for (int e = 0; e < 4; ++e) u[e] = qn(v[c][4 * g + e], l32[c], dmax);
                if (exact[c] || !(dmax < 0.4999f)) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) u[e] = ubits(qexact(v[c][4 * g + e], lamc[c], qmaxf, kNearest));
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    rm = fmaxf(rm, fabsf(__fsub_rn(v[c][4 * g + e], lds_f32((u[e] << 8) + adj[c]))));
                tq[32 * c + lane][4 * w + g] = pack4u(u[0], u[1], u[2], u[3]);
            }
        }
        __syncthreads();
        store_T_tile(tq, a.qT, a.ldq, n0, k0, a.cols, a.rows);
        __syncthreads();
    }
    rm = block_max(rm, red);
    if (threadIdx.x == 0 && a.rmax) atomicMax(a.rmax, fbits(rm));
}


// ============================================================ row kernels, r4
// One 128-thread CTA (4 warps) per row, 8 CTAs per SM.  Compared with a
// 256-thread kernel staging rows through a cp.async.bulk shared-memory ring: one CTA barrier per row instead of three (the
// dequant table is double-buffered, so building row i+1's table never waits
// for row i's readers), plain 16-byte streaming loads issued U at a time per
// lane for memory-level parallelism, and 7 rows per CTA so the static
// row-to-CTA assignment leaves no long tail.
constexpr int kRT = 128;
constexpr int kRCtasPerSM = 8;

__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// the 2*qmax+1 entries float(q / lam) (quantize.cpp:156), exact: fast product
// with a proven-safe rounding check, fp64 division otherwise
// float(-q / lam) == -float(q / lam) (round-to-nearest is symmetric): half the
// entries are computed, the negative ones mirrored (q = 0 keeps +0).
__device__ __forceinline__ void build_row_lut(float* lut, double lam, int qmax) {
    const double inv = __ddiv_rn(1.0, lam);
    for (int q = threadIdx.x; q <= qmax; q += kRT) {
        const float v = dequant_fast(q, inv, lam);
        lut[qmax + q] = v;
        if (q > 0) lut[qmax - q] = -v;
    }
}

template <int U, int MINB = kRCtasPerSM, bool KEEP = true, int RND = kNearest>
__global__ void __launch_bounds__(kRT, MINB) k_select_rows_r4(const SelectArgs a) {
    XG_PDL_WAIT();
    XG_EXIT_IF_NONFINITE(a.nonfinite);
    __shared__ float lut[2][256];
    __shared__ float redf[kRT / 32];
    __shared__ unsigned long long redu[kRT / 32];
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax;
    const double lam_r = compute_scale((double)__uint_as_float(*a.rmax), a.bits);
    const float lam_r32 = __double2float_rn(lam_r);
    const double lam_t = a.vec ? 0.0 : compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
    const double so = a.do_select && a.policy == kMin ? compute_scale((double)__uint_as_float(*a.other_max), a.bits)
                                                     : 1.0;
    unsigned cnt = 0;
    float ret = 0.0f;
    int it = 0;
    // the row's scale and statistic are fetched one row ahead, and the row's first
    // U loads are issued before its table is built: the per-row latency chain
    // (scalar loads -> fp64 threshold and table -> barrier -> row loads) overlaps
    int r = blockIdx.x;
    double lam_n = 0.0;
    float stat_n = 0.0f;
    if (r < a.rows) {
        lam_n = a.vec ? a.lam[r] : lam_t;
        if (a.do_select) stat_n = a.stat[r];
    }
    for (; r < a.rows; r += gridDim.x, ++it) {
        const float* row = a.x + (int64_t)r * a.ld;
        float4 f[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = threadIdx.x * 4 + u * kRT * 4;
            f[u] = c < a.cols ? ld_stream(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const double lam = lam_n;
        const float stat = stat_n;
        if (r + (int)gridDim.x < a.rows) {
            lam_n = a.vec ? a.lam[r + gridDim.x] : lam_t;
            if (a.do_select) stat_n = a.stat[r + gridDim.x];
        }
        const float tf = a.do_select ? float_above(threshold_of(a.policy, a.thr_m, stat, so, a.cols))
                                     : __int_as_float(0x7f800000);
        float* tb = lut[it & 1];
        build_row_lut(tb, lam, qmax);
        __syncthreads();  // table of this row complete (and the previous row's readers are past it)
        const float lam32 = __double2float_rn(lam);
        const bool exact = !(lam32 <= FLT_MAX) || !(lam_r32 <= FLT_MAX);
        const uint32_t adj = opaque_u32(smem_u32(tb) + 4u * (uint32_t)qmax - 4u * 0x4B400000u);
        int8_t* rq_row = a.rq + (int64_t)r * a.ldq;
        int8_t* rd_row = a.red + (int64_t)r * a.ldq;
        float lmax = 0.0f;
        for (int c0 = threadIdx.x * 4; c0 < a.cols; c0 += kRT * 4 * U) {
            if (c0 != (int)threadIdx.x * 4) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + u * kRT * 4;
                    f[u] = c < a.cols ? ld_stream(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + u * kRT * 4;
                if (c < a.cols) {
                    const float x[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
                    uint32_t pq, pr;
                    select_quad_n<2, RND>(x, adj, lam, lam32, lam_r, lam_r32, tf, qmaxf, exact, pq, pr, cnt, lmax);
                    *reinterpret_cast<uint32_t*>(rq_row + c) = pq;
                    if (a.do_select) *reinterpret_cast<uint32_t*>(rd_row + c) = pr;
                    if (KEEP && a.keep) dump_keep4(a, r, c, x, tf);
                }
            }
        }
        ret = fmaxf(ret, lmax >= tf ? lmax : 0.0f);
    }
    if (a.do_select) {
        unsigned long long c64 = warp_sum((unsigned long long)cnt);
        float rr = warp_maxf(ret);
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) { redu[w] = c64; redf[w] = rr; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < kRT / 32; ++i) { c64 += redu[i]; rr = fmaxf(rr, redf[i]); }
            if (c64) atomicAdd(a.nnz, c64);
            atomicMax(a.retmax, fbits(rr));
        }
    }
}

// K1, A side: the row lives in registers (VPT float4 per thread), absmax ->
// lambda -> table -> quantise -> residual max; two CTA barriers per row.
template <int VPT, int MINB = 4, int NT = kRT, int RND = kNearest>
__global__ void __launch_bounds__(NT, MINB) k_quant_rows_r4(const QuantRowsArgs a) {
    XG_PDL_WAIT();
    __shared__ float lut[2][256];
    __shared__ float red[2][NT / 32];
    const int qmax = quant_max(a.bits);
    const float qmaxf = (float)qmax;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    float rmax_acc = 0.0f, gmax_acc = 0.0f;
    int bad = 0;
    int it = 0;
    for (int r = blockIdx.x; r < a.rows; r += gridDim.x, ++it) {
        const float* row = a.x + (int64_t)r * a.ld;
        float4 f[VPT];
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const int c = (v * NT + (int)threadIdx.x) * 4;
            f[v] = c < a.cols ? ld_stream(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float m = 0.0f, sum = 0.0f;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            m = fmaxf(m, fmaxf(fmaxf(fabsf(f[v].x), fabsf(f[v].y)), fmaxf(fabsf(f[v].z), fabsf(f[v].w))));
            sum = __fadd_rn(sum, __fadd_rn(__fadd_rn(f[v].x, f[v].y), __fadd_rn(f[v].z, f[v].w)));
        }
        const bool odd = !(fabsf(sum) <= FLT_MAX);  // NaN / inf somewhere (or a finite overflow)
        if (odd) {
#pragma unroll
            for (int v = 0; v < VPT; ++v)
                bad |= (fabsf(f[v].x) <= FLT_MAX && fabsf(f[v].y) <= FLT_MAX && fabsf(f[v].z) <= FLT_MAX &&
                        fabsf(f[v].w) <= FLT_MAX) ? 0 : 2;
        }
        m = warp_maxf(m);
        float* rb = red[it & 1];
        if (l == 0) rb[w] = m;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) m = fmaxf(m, rb[i]);
        bad |= m > FLT_MAX ? 1 : 0;
        gmax_acc = fmaxf(gmax_acc, m);
        double lam;
        if (a.per_row) {
            lam = compute_scale((double)m, a.bits);
            if (threadIdx.x == 0 && a.lam_out) a.lam_out[r] = lam;
            if (threadIdx.x == 0 && a.rcp_out) a.rcp_out[r] = ff_recip(lam);
        } else {
            lam = compute_scale((double)__uint_as_float(*a.tensor_max), a.bits);
        }
        float* tb = lut[it & 1];
        build_row_lut(tb, lam, qmax);
        __syncthreads();
        const float lam32 = __double2float_rn(lam);
        const bool exact = odd || !(lam32 <= FLT_MAX);
        const uint32_t adj = opaque_u32(smem_u32(tb) + 4u * (uint32_t)qmax - 4u * 0x4B400000u);
        float rm = 0.0f;
        int8_t* qrow = a.q + (int64_t)r * a.ldq;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const int c = (v * NT + (int)threadIdx.x) * 4;
            const float x[4] = {f[v].x, f[v].y, f[v].z, f[v].w};
            uint32_t u[4];
            float dmax = 0.0f;
#pragma unroll
            qr4<RND>(x, lam32, u, dmax);
            if (exact || !(dmax < qok<RND>())) {
#pragma unroll
                for (int e = 0; e < 4; ++e) u[e] = ubits(qexact(x[e], lam, qmaxf, RND));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) rm = fmaxf(rm, fabsf(__fsub_rn(x[e], lut_at<2>(u[e], adj))));
            if (c < a.cols) *reinterpret_cast<uint32_t*>(qrow + c) = pack4u(u[0], u[1], u[2], u[3]);
        }
        rmax_acc = fmaxf(rmax_acc, rm);
    }
    rmax_acc = warp_maxf(rmax_acc);
    __syncthreads();
    if (l == 0) red[0][w] = rmax_acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < NT / 32; ++i) rmax_acc = fmaxf(rmax_acc, red[0][i]);
        if (a.rmax) atomicMax(a.rmax, fbits(rmax_acc));
        if (a.gmax) atomicMax(a.gmax, fbits(gmax_acc));
    }
    if (bad && a.nonfinite) atomicOr(a.nonfinite, bad);
}

// ============================================================ column kernels, w4
// B side (K x N row-major in, N x K K-major int8 out).  A WW-warp CTA (8, two
// CTAs per SM) works through a contiguous range of items in strip-major order,
// an item = 32-column strip x WW * 32 * kWSub rows; each warp streams its 32 x
// 32 fp32 sub-tiles through a private TMA ring of SLOTS slots (own mbarriers,
// no CTA barrier inside an item).  Lane l owns column l: it reads its column
// of the tile conflict-free, quantises 4 consecutive rows into one word, and
// writes its 32 output bytes of row n of B^T itself (two 16-byte stores), so
// no shared-memory transpose is needed.  The per-strip dequant tables
// lut[q][lane] are built when the strip changes (2 CTA barriers).
// strip width, sub-tile rows, sub-tiles per warp per item (1: items of 256 rows
// balance the persistent grid at K = 4096: select-B stage 83 -> 80 us at C2,
// 309 -> 304 us at C4, C3 unchanged; 2 and 4 measured no better)
constexpr int kWC = 32, kWR = 32, kWSub = 1;
template <int WW, int SLOTS>
constexpr int col_w_smem() { return WW * SLOTS * kWC * kWR * 4 + 256 * kWC * 4 + 1024; }

template <bool SELECT, int kWW, int kWSlots, int kWCtas, bool KEEP = true, int RND = kNearest>
__global__ void __launch_bounds__(kWW * 32, kWCtas)
    k_cols_w4(const __grid_constant__ CUtensorMap tmap, const QuantColsArgs qa, const SelectArgs sa) {
    XG_PDL_WAIT();
    constexpr int kWItemRows = kWW * kWR * kWSub;
    XG_EXIT_IF_NONFINITE(SELECT ? sa.nonfinite : qa.nonfinite);
    extern __shared__ float4 dyn_smem[];
    // 1024-byte alignment by arithmetic on the shared array itself (a uintptr_t
    // round trip makes the compiler emit generic LD for the tile reads, not LDS)
    const uint32_t pad = (1024u - (smem_u32(dyn_smem) & 1023u)) & 1023u;
    float* ring = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dyn_smem) + pad);
    float(*lut)[kWC] = reinterpret_cast<float(*)[kWC]>(ring + kWW * kWSlots * kWC * kWR);
    __shared__ uint64_t full[kWW][kWSlots];
    __shared__ float redf[kWW];
    __shared__ unsigned long long redu[kWW];
    const int rows = SELECT ? sa.rows : qa.rows, cols = SELECT ? sa.cols : qa.cols;
    const int bits = SELECT ? sa.bits : qa.bits;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qmax = quant_max(bits);
    const float qmaxf = (float)qmax;
    const int nstrips = (cols + kWC - 1) / kWC;
    const int nchunks = (rows + kWItemRows - 1) / kWItemRows;
    const int nitems = nstrips * nchunks;
    // a contiguous range of items in strip-major order: consecutive items share a
    // strip, so its scales, thresholds and dequant table are built once per strip
    const int it0 = (int)((int64_t)nitems * blockIdx.x / gridDim.x);
    const int my_items = (int)((int64_t)nitems * (blockIdx.x + 1) / gridDim.x) - it0;
    const int nsub = my_items * kWSub;  // sub-tiles this warp will consume
    double lam_r = 0.0, lam_t = 0.0, so = 1.0;
    if (SELECT) {
        lam_r = compute_scale((double)__uint_as_float(*sa.rmax), bits);
        lam_t = sa.vec ? 0.0 : compute_scale((double)__uint_as_float(*sa.tensor_max), bits);
        if (sa.do_select && sa.policy == kMin) so = compute_scale((double)__uint_as_float(*sa.other_max), bits);
    } else if (!qa.per_col) {
        lam_t = compute_scale((double)__uint_as_float(*qa.tensor_max), bits);
    }
    const float lam_r32 = __double2float_rn(lam_r);
    float* wring = ring + w * kWSlots * kWC * kWR;
    auto issue = [&](int g) {  // sub-tile g of this warp's sequence into slot g % kWSlots
        const int item = it0 + g / kWSub;
        const int strip = item / nchunks, chunk = item % nchunks;
        const int slot = g % kWSlots;
        mbar_expect_tx(&full[w][slot], kWC * kWR * 4);
        tma_load_2d(wring + slot * kWC * kWR, &tmap, &full[w][slot], strip * kWC,
                    chunk * kWItemRows + (w * kWSub + g % kWSub) * kWR);
    };
    if (threadIdx.x == 0) {
        tma_prefetch(&tmap);
        for (int i = 0; i < kWW; ++i)
            for (int j = 0; j < kWSlots; ++j) mbar_init(&full[i][j], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (lane == 0)
        for (int g = 0; g < kWSlots && g < nsub; ++g) issue(g);
    const uint32_t adj_base = opaque_u32(smem_u32(&lut[0][0]) + 4u * lane + 128u * (uint32_t)qmax - 128u * 0x4B400000u);
    float rm = 0.0f, ret = 0.0f;
    unsigned cnt = 0;
    int g = 0;
    int cur_strip = -1;
    double lam = 0.0;
    float lam32 = 0.0f, tf = 0.0f;
    bool exact = false;
    for (int i = 0; i < my_items; ++i) {
        const int item = it0 + i;
        const int strip = item / nchunks, chunk = item % nchunks;
        const int n = strip * kWC + lane;
        const int nc = min(n, cols - 1);
        if (strip != cur_strip) {
        if (SELECT) lam = sa.vec ? sa.lam[nc] : lam_t;
        else lam = qa.per_col ? compute_scale((double)__uint_as_float(qa.colmax[nc]), bits) : lam_t;
        if (!SELECT && qa.per_col && qa.lam_out && chunk == 0 && w == 0 && n < cols) qa.lam_out[n] = lam;
        if (!SELECT && qa.per_col && qa.rcp_out && chunk == 0 && w == 0 && n < cols) qa.rcp_out[n] = ff_recip(lam);
        lam32 = __double2float_rn(lam);
        exact = !(lam32 <= FLT_MAX) || (SELECT && !(lam_r32 <= FLT_MAX));
        tf = __int_as_float(0x7f800000);
        if (SELECT && sa.do_select && n < cols) tf = float_above(threshold_of(sa.policy, sa.thr_m, sa.stat[nc], so, rows));
        __syncthreads();  // previous strip's table readers are done
        {
            const double inv = __ddiv_rn(1.0, lam);
            constexpr int per = (128 + kWW - 1) / kWW;  // q in [0, qmax], mirrored (see build_row_lut)
            for (int q = w * per; q < (w + 1) * per; ++q)
                if (q <= qmax) {
                    const float v = dequant_fast(q, inv, lam);
                    lut[qmax + q][lane] = v;
                    if (q > 0) lut[qmax - q][lane] = -v;
                }
        }
        __syncthreads();
        cur_strip = strip;
        }
        float lmax = 0.0f;
        for (int j = 0; j < kWSub; ++j, ++g) {
            const int slot = g % kWSlots;
            const int k0 = chunk * kWItemRows + (w * kWSub + j) * kWR;
            mbar_wait(&full[w][slot], (g / kWSlots) & 1);
            const float* tile = wring + slot * kWC * kWR;
            float x[kWR];
#pragma unroll
            for (int r = 0; r < kWR; ++r) x[r] = tile[r * kWC + lane];
            __syncwarp();
            if (lane == 0 && g + kWSlots < nsub) {
                fence_proxy_async();
                issue(g + kWSlots);
            }
            uint32_t w0[kWR / 4], w1[kWR / 4];
#pragma unroll
            for (int q = 0; q < kWR / 4; ++q) {
                const float xq[4] = {x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]};
                if (SELECT) {
                    select_quad_n<7, RND>(xq, adj_base, lam, lam32, lam_r, lam_r32, tf, qmaxf, exact, w0[q], w1[q],
                                     cnt, lmax);
                    if (KEEP && sa.keep && n < cols && k0 + 4 * q < rows) dump_keep4(sa, n, k0 + 4 * q, xq, tf);
                } else {
                    uint32_t u[4];
                    float dmax = 0.0f;
                    qr4<RND>(xq, lam32, u, dmax);
                    if (exact || !(dmax < qok<RND>())) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) u[e] = ubits(qexact(xq[e], lam, qmaxf, RND));
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) rm = fmaxf(rm, fabsf(__fsub_rn(xq[e], lut_at<7>(u[e], adj_base))));
                    w0[q] = pack4u(u[0], u[1], u[2], u[3]);
                }
            }
            if (n < cols && k0 < rows) {
                int8_t* d0 = (SELECT ? sa.rq : qa.qT) + (int64_t)n * (SELECT ? sa.ldq : qa.ldq) + k0;
                int8_t* d1 = SELECT && sa.do_select ? sa.red + (int64_t)n * sa.ldq + k0 : nullptr;
                if (k0 + kWR <= rows) {
#pragma unroll
                    for (int v = 0; v < kWR / 16; ++v) {
                        reinterpret_cast<uint4*>(d0)[v] = make_uint4(w0[4 * v], w0[4 * v + 1], w0[4 * v + 2], w0[4 * v + 3]);
                        if (d1) reinterpret_cast<uint4*>(d1)[v] = make_uint4(w1[4 * v], w1[4 * v + 1], w1[4 * v + 2], w1[4 * v + 3]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < kWR / 4; ++q)
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (4 * q + e < rows - k0) {
                                d0[4 * q + e] = (int8_t)(w0[q] >> (8 * e));
                                if (d1) d1[4 * q + e] = (int8_t)(w1[q] >> (8 * e));
                            }
                }
            }
        }
        if (SELECT) ret = fmaxf(ret, lmax >= tf ? lmax : 0.0f);
    }
    // block reductions (all warps reach here)
    if (SELECT) {
        if (sa.do_select) {
            unsigned long long c64 = warp_sum((unsigned long long)cnt);
            float rr = warp_maxf(ret);
            if (lane == 0) { redu[w] = c64; redf[w] = rr; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int i = 1; i < kWW; ++i) { c64 += redu[i]; rr = fmaxf(rr, redf[i]); }
                if (c64) atomicAdd(sa.nnz, c64);
                atomicMax(sa.retmax, fbits(rr));
            }
        }
    } else {
        float r = warp_maxf(rm);
        if (lane == 0) redf[w] = r;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < kWW; ++i) r = fmaxf(r, redf[i]);
            if (qa.rmax) atomicMax(qa.rmax, fbits(r));
        }
    }
}

// ------------------------------------------- fused K1, B side (one DRAM pass)
// Column maxima and quantisation of B in one kernel.  A cluster of C CTAs
// owns a 32-column strip over all K rows (CTA rank r: rows [2048 r, 2048 r +
// 2048)).  Each warp streams its sub-tiles of every strip twice through its
// TMA ring: pass 0 takes the column maxima (|x| as integer bits: NaN > inf >
// finite), the cluster combines them in rank 0's shared memory (DSMEM
// red.max), and pass 1 re-reads the same sub-tiles - now L2-resident (C x
// 256 KB per strip in flight, ~40 MB in all) - and quantises them exactly as
// k_cols_w4 does.  The ring interleaves pass 1 of strip i with pass 0 of strip
// i+1, so DRAM keeps streaming while a strip is quantised and only the
// cluster exchange sits between strips.  B leaves DRAM once instead of twice
// (k_absmax_cols + k_cols_w4<0>).  A strip with a non-finite value raises
// `nonfinite` and is not quantised (the call fails, pipeline.cpp:50-52).
template <int kWW, int kWSlots, int kSub, int RND = kNearest>
__global__ void __launch_bounds__(kWW * 32, 1)
    k_cols_maxq(const __grid_constant__ CUtensorMap tmap, const QuantColsArgs qa, uint32_t* gmax, int* nonfinite) {
    XG_PDL_WAIT();
    constexpr int kRowsCta = kWW * kWR * kSub;
    extern __shared__ float4 dyn_smem[];
    float* ring = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(dyn_smem) +
                                           ((1024u - (smem_u32(dyn_smem) & 1023u)) & 1023u));
    float(*lut)[kWC] = reinterpret_cast<float(*)[kWC]>(ring + kWW * kWSlots * kWC * kWR);
    __shared__ uint64_t full[kWW][kWSlots];
    __shared__ __align__(16) uint32_t wmax[kWW][kWC];
    __shared__ uint32_t cmax[3][kWC];  // cluster maxima per strip (rank 0's copy), 3-deep for the resets
    __shared__ float redf[kWW];
    const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
    const int ncl = (int)(gridDim.x / csize), cid = (int)(blockIdx.x / csize);
    const int rows = qa.rows, cols = qa.cols, bits = qa.bits;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qmax = quant_max(bits);
    const float qmaxf = (float)qmax;
    const int nstrips = (cols + kWC - 1) / kWC;
    const int my_items = nstrips > cid ? (nstrips - cid + ncl - 1) / ncl : 0;
    // ring order: pass 0 of strip 0, then per strip i: pass 1 (i) tile j, pass 0 (i+1) tile j, ...
    const int ntiles = 2 * kSub * my_items;
    float* wring = ring + w * kWSlots * kWC * kWR;
    auto issue = [&](int g) {
        int item, j;
        if (g < kSub) {
            item = 0, j = g;
        } else {
            const int q = g - kSub;
            if (q < (my_items - 1) * 2 * kSub) {
                const int r = q % (2 * kSub);
                item = q / (2 * kSub) + (r & 1), j = r >> 1;
            } else {
                item = my_items - 1, j = q - (my_items - 1) * 2 * kSub;
            }
        }
        const int slot = g % kWSlots;
        mbar_expect_tx(&full[w][slot], kWC * kWR * 4);
        tma_load_2d(wring + slot * kWC * kWR, &tmap, &full[w][slot], (cid + item * ncl) * kWC,
                    (int)crank * kRowsCta + (w * kSub + j) * kWR);
    };
    if (threadIdx.x == 0) {
        tma_prefetch(&tmap);
        for (int i = 0; i < kWW; ++i)
            for (int j = 0; j < kWSlots; ++j) mbar_init(&full[i][j], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 3 * kWC) cmax[threadIdx.x / kWC][threadIdx.x % kWC] = 0u;
    __syncthreads();
    cluster_sync_all();  // every CTA's maxima zeroed before any remote max lands
    if (lane == 0)
        for (int g = 0; g < kWSlots && g < ntiles; ++g) issue(g);
    int g = 0;
    // next sub-tile of the ring into registers (lane = column), slot handed back to TMA
    auto consume = [&](float (&x)[kWR]) {
        const int slot = g % kWSlots;
        mbar_wait(&full[w][slot], (g / kWSlots) & 1);
        const float* tile = wring + slot * kWC * kWR;
#pragma unroll
        for (int r = 0; r < kWR; ++r) x[r] = tile[r * kWC + lane];
        __syncwarp();
        if (lane == 0 && g + kWSlots < ntiles) {
            fence_proxy_async();
            issue(g + kWSlots);
        }
        ++g;
    };
    // pass 0: the sub-tile read as float4 (lane l: columns 4 (l % 8) .. +3 of rows
    // l / 8 + 4 i, a quarter of the shared-memory loads of the column-per-lane read);
    // um4 holds |x| bit maxima of those 4 columns until the strip's exchange
    auto consume_max = [&](uint32_t (&m)[4]) {
        const int slot = g % kWSlots;
        mbar_wait(&full[w][slot], (g / kWSlots) & 1);
        const float4* tile = reinterpret_cast<const float4*>(wring + slot * kWC * kWR);
        float4 v[kWR / 4];
#pragma unroll
        for (int i = 0; i < kWR / 4; ++i) v[i] = tile[(lane >> 3) * (kWC / 4) + i * kWC + (lane & 7)];
        __syncwarp();
        if (lane == 0 && g + kWSlots < ntiles) {
            fence_proxy_async();
            issue(g + kWSlots);
        }
        ++g;
#pragma unroll
        for (int i = 0; i < kWR / 4; ++i) {
            m[0] = max(m[0], __float_as_uint(v[i].x) & 0x7fffffffu);
            m[1] = max(m[1], __float_as_uint(v[i].y) & 0x7fffffffu);
            m[2] = max(m[2], __float_as_uint(v[i].z) & 0x7fffffffu);
            m[3] = max(m[3], __float_as_uint(v[i].w) & 0x7fffffffu);
        }
    };
    const uint32_t cmax_r0 = mapa_shared(&cmax[0][0], 0);
    const uint32_t adj_base = opaque_u32(smem_u32(&lut[0][0]) + 4u * lane + 128u * (uint32_t)qmax - 128u * 0x4B400000u);
    float rm = 0.0f;
    uint32_t um4[4] = {0u, 0u, 0u, 0u};
    if (my_items > 0)
        for (int j = 0; j < kSub; ++j) consume_max(um4);  // pass 0 of the first strip
    for (int i = 0; i < my_items; ++i) {
        const int strip = cid + i * ncl;
        const int n = strip * kWC + lane;
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // lanes l, l ^ 8, l ^ 16, l ^ 24 hold the same 4 columns
            um4[e] = max(um4[e], __shfl_xor_sync(0xffffffffu, um4[e], 8));
            um4[e] = max(um4[e], __shfl_xor_sync(0xffffffffu, um4[e], 16));
        }
        if (lane < 8) *reinterpret_cast<uint4*>(&wmax[w][4 * lane]) = make_uint4(um4[0], um4[1], um4[2], um4[3]);
        __syncthreads();  // all warps' maxima; every warp is past the previous strip's table readers
        const int b = i % 3;
        if (w == 0) {
            uint32_t m = 0u;
#pragma unroll
            for (int k = 0; k < kWW; ++k) m = max(m, wmax[k][lane]);
            red_max_cluster_u32(cmax_r0 + 4u * (uint32_t)(b * kWC + lane), m);
            // rank 0 clears the buffer of strip i+1: its last readers (strip i-2) finished
            // before the previous cluster barrier, its writers start after the next one
            if (crank == 0) cmax[(i + 1) % 3][lane] = 0u;
        }
        cluster_sync_all();
        const uint32_t cm = ld_cluster_u32(cmax_r0 + 4u * (uint32_t)(b * kWC + lane));
        const bool bad = __any_sync(0xffffffffu, n < cols && cm > 0x7f7fffffu);  // uniform over the cluster
        const float cmf = __uint_as_float(cm);
        const double lam = compute_scale((double)cmf, bits);
        if (crank == 0 && w == 0) {
            if (n < cols) {
                if (qa.lam_out) qa.lam_out[n] = lam;
                if (qa.rcp_out) qa.rcp_out[n] = ff_recip(lam);
            }
            const float sm = warp_maxf(n < cols && !bad ? cmf : 0.0f);
            if (lane == 0) {
                if (bad) atomicOr(nonfinite, 1);
                else if (gmax) atomicMax(gmax, fbits(sm));
            }
        }
        if (!bad) {
            const double inv = __ddiv_rn(1.0, lam);
            constexpr int per = (128 + kWW - 1) / kWW;  // q in [0, qmax], mirrored (see build_row_lut)
            for (int q = w * per; q < (w + 1) * per; ++q)
                if (q <= qmax) {
                    const float v = dequant_fast(q, inv, lam);
                    lut[qmax + q][lane] = v;
                    if (q > 0) lut[qmax - q][lane] = -v;
                }
        }
        __syncthreads();
        const float lam32 = __double2float_rn(lam);
        const bool exact = !(lam32 <= FLT_MAX);
        const bool next = i + 1 < my_items;
#pragma unroll
        for (int e = 0; e < 4; ++e) um4[e] = 0u;
        for (int j = 0; j < kSub; ++j) {
            const int k0 = (int)crank * kRowsCta + (w * kSub + j) * kWR;
            float x[kWR];
            consume(x);  // pass 1 of this strip (L2)
            if (!bad) {
                uint32_t w0[kWR / 4];
#pragma unroll
                for (int q = 0; q < kWR / 4; ++q) {
                    const float xq[4] = {x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]};
                    uint32_t u[4];
                    float dmax = 0.0f;
                    qr4<RND>(xq, lam32, u, dmax);
                    if (exact || !(dmax < qok<RND>())) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) u[e] = ubits(qexact(xq[e], lam, qmaxf, RND));
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) rm = fmaxf(rm, fabsf(__fsub_rn(xq[e], lut_at<7>(u[e], adj_base))));
                    w0[q] = pack4u(u[0], u[1], u[2], u[3]);
                }
                if (n < cols && k0 < rows) {
                    int8_t* d0 = qa.qT + (int64_t)n * qa.ldq + k0;
                    if (k0 + kWR <= rows) {
#pragma unroll
                        for (int v = 0; v < kWR / 16; ++v)
                            reinterpret_cast<uint4*>(d0)[v] =
                                make_uint4(w0[4 * v], w0[4 * v + 1], w0[4 * v + 2], w0[4 * v + 3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < kWR / 4; ++q)
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (4 * q + e < rows - k0) d0[4 * q + e] = (int8_t)(w0[q] >> (8 * e));
                    }
                }
            }
            if (next) consume_max(um4);  // pass 0 of the next strip (DRAM)
        }
    }
    float r = warp_maxf(rm);
    if (lane == 0) redf[w] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kWW; ++k) r = fmaxf(r, redf[k]);
        if (qa.rmax) atomicMax(qa.rmax, fbits(r));
    }
    cluster_sync_all();  // no CTA leaves while another may still address its shared memory
}

// ------------------------------------------------------------- scalars --
__global__ void k_lambdas(DevScalars* sc, int bits) {
    XG_PDL_WAIT();
    sc->lamA = compute_scale((double)__uint_as_float(sc->maxA), bits);
    sc->lamB = compute_scale((double)__uint_as_float(sc->maxB), bits);
    sc->rA = ff_recip(sc->lamA);
    sc->rB = ff_recip(sc->lamB);
}

// Density, dispatch (pipeline.cpp:106-111) and the per-tensor scales the
// compensation epilogue reads.
__global__ void k_dispatch(DevScalars* sc, int bits, int64_t MK, int64_t KN, double s, int reduce, int M, int N,
                           int K, CompModel cm) {
    XG_PDL_WAIT();
    sc->lamRA = compute_scale((double)__uint_as_float(sc->maxRA), bits);
    sc->lamRB = compute_scale((double)__uint_as_float(sc->maxRB), bits);
    sc->lamAred = compute_scale((double)__uint_as_float(sc->retA), bits);
    sc->lamBred = compute_scale((double)__uint_as_float(sc->retB), bits);
    sc->rRA = ff_recip(sc->lamRA);
    sc->rRB = ff_recip(sc->lamRB);
    sc->rAred = ff_recip(sc->lamAred);
    sc->rBred = ff_recip(sc->lamBred);
    if (reduce) {
        const double da = __ddiv_rn((double)sc->nnzA, (double)MK);
        const double db = __ddiv_rn((double)sc->nnzB, (double)KN);
        sc->densA = da;
        sc->densB = db;
        const int sparse = fmax(da, db) < s;
        sc->sel = sparse;
        sc->path = sparse ? kSparse : kDense;
        // same result either way (exact integer sums): pick the faster compensation
        int csr = 0;
        if (sparse && cm.csr_ok) {
            if (cm.force == 2) {
                csr = 1;
            } else if (cm.force == 0) {
                const double mn = (double)M * (double)N;
                const double t_d = 4.0 * mn * (double)K / cm.p_tc;
                const double macs = (double)sc->nnzA * (double)N + (double)sc->nnzB * (double)M;
                // K > 8192 runs 8-line strips: twice the strips, half the columns per lane
                const double wf = K > 8192 ? 1.5 : 1.0;
                // the two CSR builds read A'q / B'q^T at ~1/3 of HBM bandwidth (measured)
                const double t_c = fmax(macs * wf / cm.p_sp, mn * cm.c_el * wf) + 3.0 * ((double)M + (double)N) * K / cm.bw;
                csr = t_c < 0.9 * t_d;
            }
        }
        sc->csr = csr;
    } else {
        sc->densA = sc->densB = 0.0;
        sc->sel = 0;
        sc->path = kDense;
    }
}

__global__ void k_fill_u32(uint32_t* p, uint32_t v, int64_t n) {
    XG_PDL_WAIT();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_rows(int rows) { return rows < kNumSMs * 16 ? rows : kNumSMs * 16; }

}  // namespace

template <class K>
void set_dyn_smem(K kern, int bytes) {
    // cheap; the kernels are distinct template instances of the same type
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

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

template <int RND>
void quant_rows_rnd(const QuantRowsArgs& a, cudaStream_t s) {
    const int g = grid_rows(a.rows);
    const int vpt = (a.cols + kThreads * 4 - 1) / (kThreads * 4);
    if (vpt <= 1) k_quant_rows<1, RND><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 2) k_quant_rows<2, RND><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 4) k_quant_rows<4, RND><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 8) k_quant_rows<8, RND><<<g, kThreads, 0, s>>>(a);
    else if (vpt <= 16) k_quant_rows<16, RND><<<g, kThreads, 0, s>>>(a);
    else k_quant_rows_generic<<<g, kThreads, 0, s>>>(a);
}

// the register-resident row kernels for K in [1024, 16384]; false otherwise
template <int RND>
bool launch_quant_rows_r4(const QuantRowsArgs& a, cudaStream_t s) {
    if (a.cols >= 1024 && a.cols <= 8192) {
        const int vpt = (a.cols + kRT * 4 - 1) / (kRT * 4);
        // CTAs per SM by row length (registers hold the row): 5 at VPT 16 (96
        // registers; C3 67.0 -> 64.0 us), 6 at VPT 8 (75; C2 24.4 -> 21.2 us),
        // 8 below; one more CTA spills in each case
        const int cap = kNumSMs * (vpt > 8 ? 5 : vpt > 4 ? 6 : 8);
        const int g = a.rows < cap ? a.rows : cap;
        if (vpt <= 2) k_quant_rows_r4<2, 8, kRT, RND><<<g, kRT, 0, s>>>(a);
        else if (vpt <= 4) k_quant_rows_r4<4, 8, kRT, RND><<<g, kRT, 0, s>>>(a);
        else if (vpt <= 8) k_quant_rows_r4<8, 6, kRT, RND><<<g, kRT, 0, s>>>(a);
        else k_quant_rows_r4<16, 5, kRT, RND><<<g, kRT, 0, s>>>(a);
        return true;
    }
    if (a.cols > 8192 && a.cols <= 16384) {
        // K in (8192, 16384] (C5): the same register-resident row over 256 threads
        const int cap = kNumSMs * 2;
        const int g = a.rows < cap ? a.rows : cap;
        k_quant_rows_r4<16, 2, 256, RND><<<g, 256, 0, s>>>(a);
        return true;
    }
    return false;
}

void launch_quant_rows(const QuantRowsArgs& a, cudaStream_t s) {
    const bool aligned = (a.ld % 4 == 0) && (a.ldq % 4 == 0) && (a.cols % 4 == 0) &&
                         ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
    if (aligned && (a.rounding == kNearest ? launch_quant_rows_r4<kNearest>(a, s) : launch_quant_rows_r4<kFloor>(a, s)))
        return;
    if (a.rounding == kNearest) {
        const int g = grid_rows(a.rows);
        const int vpt = (a.cols + kThreads * 4 - 1) / (kThreads * 4);
        if (vpt <= 1) k_quant_rows_fast<1, 256><<<g, 256, 0, s>>>(a);
        else if (vpt <= 2) k_quant_rows_fast<2, 256><<<g, 256, 0, s>>>(a);
        else if (vpt <= 4) k_quant_rows_fast<2, 512><<<g, 512, 0, s>>>(a);
        else if (vpt <= 8) k_quant_rows_fast<4, 512><<<g, 512, 0, s>>>(a);
        else if (vpt <= 16) k_quant_rows_fast<8, 512><<<g, 512, 0, s>>>(a);
        else k_quant_rows_generic<<<g, kThreads, 0, s>>>(a);
    } else {
        quant_rows_rnd<kFloor>(a, s);
    }
}



template <bool SELECT, int WW, int SLOTS, int CTAS, int RND>
void launch_cols_w(const CUtensorMap& tm, const QuantColsArgs& qa, const SelectArgs& sa, int rows, int cols,
                   cudaStream_t s) {
    constexpr int smem = col_w_smem<WW, SLOTS>();
    // no stage-dump bitmask: the variant without the per-quad check
    auto kern = (SELECT && !sa.keep) ? k_cols_w4<SELECT, WW, SLOTS, CTAS, false, RND>
                                     : k_cols_w4<SELECT, WW, SLOTS, CTAS, true, RND>;
    set_dyn_smem(kern, smem);
    const int items = ((cols + kWC - 1) / kWC) * ((rows + WW * kWR * kWSub - 1) / (WW * kWR * kWSub));
    const int cap = kNumSMs * CTAS;
    kern<<<items < cap ? items : cap, WW * 32, smem, s>>>(tm, qa, sa);
}

// Column-kernel shape: 8 warps x 1 ring slot per warp x 3 CTAs per SM (80
// registers; 24 warps per SM hide more latency than a deeper ring: select-B
// 102.4 -> 97.7 us at C3, reduce stage -5 / -8 us at C3 / C4, against 8x2x2;
// 16x2x1, 12x1x2, 24x1x1 and 4x4x2 measured slower, profiles/README.md)
template <bool SELECT>
void launch_cols_any(const CUtensorMap& tm, const QuantColsArgs& qa, const SelectArgs& sa, int rows, int cols,
                     int rounding, cudaStream_t s) {
    if (rounding == kNearest) launch_cols_w<SELECT, 8, 1, 3, kNearest>(tm, qa, sa, rows, cols, s);
    else launch_cols_w<SELECT, 8, 1, 3, kFloor>(tm, qa, sa, rows, cols, s);
}

// Fused column maxima + quantisation (k_cols_maxq); false when the shape or
// options need the two-kernel path.  Launched as 16 warps x 2 ring slots x 4
// sub-tiles per warp (8x4x8, 12x3x4 and 8x6x8 measured slower; 16x2x8 and
// 16x2x2 - clusters of 2 and 8 at K = 8192 - too: C3 K1 174 -> 190 / 186 us).
template <int WW, int SLOTS, int SUB, int RND>
bool launch_cols_maxq(const QuantColsArgs& a, uint32_t* gmax, int* nonfinite, cudaStream_t s) {
    constexpr int rows_cta = WW * kWR * SUB;
    const int csize = (a.rows + rows_cta - 1) / rows_cta;
    // K <= 8192 (clusters of <= 4): measured 1-5% faster end to end than the two
    // kernels at C2-C4; 8-CTA clusters (K = 16384) co-schedule worse with the
    // A side and measured ~1% slower, so larger K keeps the two-kernel path
    if (csize > 4) return false;
    alignas(64) CUtensorMap tm;
    if (!make_tmap_f32(&tm, a.x, a.rows, a.cols, a.ld, kWC, kWR)) return false;
    constexpr int smem = col_w_smem<WW, SLOTS>();
    auto kern = k_cols_maxq<WW, SLOTS, SUB, RND>;
    set_dyn_smem(kern, smem);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(WW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    static int max_clusters[9] = {0};  // co-resident clusters per cluster size (same part on every device)
    if (!max_clusters[csize]) {
        cfg.gridDim = dim3(csize * 256);
        int m = 0;
        if (cudaOccupancyMaxActiveClusters(&m, kern, &cfg) != cudaSuccess || m <= 0) {
            cudaGetLastError();
            m = kNumSMs / csize;
        }
        max_clusters[csize] = m;
    }
    const int nstrips = (a.cols + kWC - 1) / kWC;
    const int ncl = nstrips < max_clusters[csize] ? nstrips : max_clusters[csize];
    cfg.gridDim = dim3(csize * ncl);
    return cudaLaunchKernelEx(&cfg, kern, tm, a, gmax, nonfinite) == cudaSuccess;
}

template <int RND>
bool launch_quant_cols_fused_rnd(const QuantColsArgs& a, uint32_t* gmax, int* nonfinite, cudaStream_t s) {
    // short K: CTAs of fewer rows, so the cluster grid (strips x cluster size)
    // still spreads over the SMs (C1 1024^3: K1 19 -> 13 us; 2048^3: 25 -> 21 us)
    if (a.rows <= 1024) return launch_cols_maxq<8, 2, 1, RND>(a, gmax, nonfinite, s);
    if (a.rows <= 2048) return launch_cols_maxq<16, 2, 2, RND>(a, gmax, nonfinite, s);
    return launch_cols_maxq<16, 2, 4, RND>(a, gmax, nonfinite, s);
}

bool launch_quant_cols_fused(const QuantColsArgs& a, uint32_t* gmax, int* nonfinite, cudaStream_t s) {
    if (!a.per_col || a.rows < 256 || (a.ldq % 16) != 0) return false;
    return a.rounding == kNearest ? launch_quant_cols_fused_rnd<kNearest>(a, gmax, nonfinite, s)
                                  : launch_quant_cols_fused_rnd<kFloor>(a, gmax, nonfinite, s);
}

void launch_quant_cols_T(const QuantColsArgs& a, cudaStream_t s) {
    if (a.rows >= 256 && (a.ldq % 16) == 0) {
        alignas(64) CUtensorMap tm;
        if (make_tmap_f32(&tm, a.x, a.rows, a.cols, a.ld, kWC, kWR)) {
            launch_cols_any<false>(tm, a, SelectArgs{}, a.rows, a.cols, a.rounding, s);
            return;
        }
    }
    dim3 grid((a.cols + kTN - 1) / kTN, (a.rows + kColTileRows - 1) / kColTileRows);
    if (a.rounding == kNearest) {
        set_dyn_smem(k_quant_cols_T_fast, kLutBytes);
        k_quant_cols_T_fast<<<grid, kThreads, kLutBytes, s>>>(a);
    } else {
        set_dyn_smem(k_quant_cols_T<kFloor>, kLutBytes);
        k_quant_cols_T<kFloor><<<grid, kThreads, kLutBytes, s>>>(a);
    }
}

void launch_select_rows(const SelectArgs& a, cudaStream_t s) {
    const bool aligned = (a.ld % 4 == 0) && (a.ldq % 4 == 0) && (a.cols % 4 == 0) &&
                         ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
    if (!a.fix_mode && aligned && a.cols >= 512) {
        // 4 loads in flight per thread, kRCtasPerSM CTAs per SM (2x8, 8x6 and 4x12 measured slower)
        const int cap = kNumSMs * kRCtasPerSM;
        const int g = a.rows < cap ? a.rows : cap;
        if (a.rounding == kNearest) {
            if (a.keep) k_select_rows_r4<4><<<g, kRT, 0, s>>>(a);
            else k_select_rows_r4<4, kRCtasPerSM, false><<<g, kRT, 0, s>>>(a);  // no stage-dump bitmask
        } else {
            if (a.keep) k_select_rows_r4<4, kRCtasPerSM, true, kFloor><<<g, kRT, 0, s>>>(a);
            else k_select_rows_r4<4, kRCtasPerSM, false, kFloor><<<g, kRT, 0, s>>>(a);
        }
        return;
    }
    // the fix-up grid: two CTAs per SM; it exits at once in the common case (the
    // retained maximum is the tensor maximum), a full-size grid only paid its launch
    if (a.fix_mode) k_fix_rows<<<a.rows < 2 * kNumSMs ? a.rows : 2 * kNumSMs, kThreads, 0, s>>>(a);
    else if (a.rounding == kNearest) k_select_rows<kNearest><<<grid_rows(a.rows), kThreads, 0, s>>>(a);
    else k_select_rows<kFloor><<<grid_rows(a.rows), kThreads, 0, s>>>(a);
}

void launch_select_cols_T(const SelectArgs& a, cudaStream_t s) {
    if (a.fix_mode) {
        k_fix_cols_T<<<a.cols < 2 * kNumSMs ? a.cols : 2 * kNumSMs, kThreads, 0, s>>>(a);
        return;
    }
    if (a.rows >= 256 && (a.ldq % 16) == 0) {
        alignas(64) CUtensorMap tm;
        if (make_tmap_f32(&tm, a.x, a.rows, a.cols, a.ld, kWC, kWR)) {
            launch_cols_any<true>(tm, QuantColsArgs{}, a, a.rows, a.cols, a.rounding, s);
            return;
        }
    }
    dim3 grid((a.cols + kTN - 1) / kTN, (a.rows + kColTileRows - 1) / kColTileRows);
    if (a.rounding == kNearest) {
        set_dyn_smem(k_select_cols_T<kNearest>, kLutBytes);
        k_select_cols_T<kNearest><<<grid, kThreads, kLutBytes, s>>>(a);
    } else {
        set_dyn_smem(k_select_cols_T<kFloor>, kLutBytes);
        k_select_cols_T<kFloor><<<grid, kThreads, kLutBytes, s>>>(a);
    }
}

void launch_lambdas(DevScalars* sc, int bits, cudaStream_t s) { k_lambdas<<<1, 1, 0, s>>>(sc, bits); }

void launch_dispatch(DevScalars* sc, int bits, int64_t MK, int64_t KN, double density_limit,
                     int reduce, cudaStream_t s, int M, int N, int K, int csr_ok, const CompModel* model) {
    CompModel cm = model ? *model : comp_model();
    cm.csr_ok = csr_ok;
    k_dispatch<<<1, 1, 0, s>>>(sc, bits, MK, KN, density_limit, reduce, M, N, K, cm);
}

// B200 measurements (tools/csr_sweep.py, profiles/r2_csr_sweep_*.jsonl): the
// compensation launch 3.6e15 int8 op/s (4MNK masked-dense); 16-line strips
// (K <= 8192) ~9.6e12 MAC/s incremental and 7.7 ns of density-independent work
// per output element (8-line strips: x1.5); HBM 6.4e12 B/s
namespace {
CompModel g_model = [] {
    CompModel m{3.6e15, 9.6e12, 6.4e12, 7.7e-12, 0, 0};
    if (const char* e = getenv("XG_COMP")) m.force = atoi(e);  // 0 auto, 1 dense, 2 CSR
    if (const char* e = getenv("XG_P_SPMM")) m.p_sp = atof(e);
    return m;
}();
}  // namespace
const CompModel& comp_model() { return g_model; }
void set_comp_model(const CompModel& m) { g_model = m; }

void fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t s) {
    int64_t blocks = (n + 255) / 256;
    blocks = blocks < 1 ? 1 : blocks > 4096 ? 4096 : blocks;
    k_fill_u32<<<(int)blocks, 256, 0, s>>>(p, v, n);
}

}  // namespace xg
