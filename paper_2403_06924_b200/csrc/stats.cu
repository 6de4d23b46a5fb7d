// Row / column statistics of |D_F| that drive the threshold reduction
// (pipeline.cpp:215-247, selected at :98-101).
//
// MinRule is order-free (float min): exact with atomicMin on the bit pattern.
// AvgRule is an order-dependent fp64 sum in the reference (i outer, j inner).
// We sum in any order on the GPU and prove the float mean equal to the
// reference's with verified rounding: for n non-negative terms both orders lie
// within gamma_{n-1} * S of the exact sum, so if RN_f(RN_d(S_lo/n)) ==
// RN_f(RN_d(S_hi/n)) over the widened interval the reference's float is
// pinned.  The rare ambiguous statistics (~1e-5 each) are recomputed with the
// reference's exact sequential order.
#include <cfloat>

#include "common.cuh"
#include "internal.h"

namespace xg {
namespace {

constexpr int kThreads = 256;
constexpr int kSlabRows = 64;  // rows per CTA (measured at C3: 64 -> 56.9 us, 32 -> 61.1; half the column atomics)

// One pass over D_F: each thread owns 4 adjacent columns of a 32-row slab.
template <int POLICY, int kSlab = kSlabRows>
__global__ void __launch_bounds__(kThreads)
    k_stats_slab(const float* __restrict__ d, int rows, int cols, double* row_sum,
                 double* col_sum, uint32_t* row_min, uint32_t* col_min) {
    XG_PDL_WAIT();
    const int c = (blockIdx.x * kThreads + threadIdx.x) * 4;
    // slabs bottom-up: the D_F GEMM wrote the bottom row panels last, so the
    // first slabs read are still in L2
    const int r0 = (gridDim.y - 1 - blockIdx.y) * kSlab;
    const int lane = threadIdx.x & 31;
    const bool vec = (cols % 4 == 0) && c + 3 < cols;
    double cs0 = 0, cs1 = 0, cs2 = 0, cs3 = 0;
    float cm0 = FLT_MAX, cm1 = FLT_MAX, cm2 = FLT_MAX, cm3 = FLT_MAX;
    constexpr int kBatch = 8;  // rows loaded ahead of the (serialising) reductions
    for (int rb = 0; rb < kSlab; rb += kBatch) {
        if (r0 + rb >= rows) break;  // uniform across the CTA
        float4 fv[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int r = r0 + rb + u;
            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
            const float* p = d + (int64_t)r * cols + c;
            if (r < rows) {
                if (vec) {
                    f = __ldg(reinterpret_cast<const float4*>(p));
                } else if (c < cols) {
                    f.x = p[0];
                    if (c + 1 < cols) f.y = p[1];
                    if (c + 2 < cols) f.z = p[2];
                    if (c + 3 < cols) f.w = p[3];
                }
            }
            fv[u] = f;
        }
        double rsv[kBatch];
        float rmv[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int r = r0 + rb + u;
            const float4 f = fv[u];
            if (POLICY == kAvg) {
                const double a0 = fabs((double)f.x), a1 = fabs((double)f.y), a2 = fabs((double)f.z),
                             a3 = fabs((double)f.w);
                cs0 = __dadd_rn(cs0, a0);
                cs1 = __dadd_rn(cs1, a1);
                cs2 = __dadd_rn(cs2, a2);
                cs3 = __dadd_rn(cs3, a3);
                rsv[u] = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
            } else {
                const bool in0 = c < cols, in1 = c + 1 < cols, in2 = c + 2 < cols, in3 = c + 3 < cols;
                const bool rin = r < rows;
                const float a0 = in0 && rin ? fabsf(f.x) : FLT_MAX, a1 = in1 && rin ? fabsf(f.y) : FLT_MAX,
                            a2 = in2 && rin ? fabsf(f.z) : FLT_MAX, a3 = in3 && rin ? fabsf(f.w) : FLT_MAX;
                cm0 = fminf(cm0, a0);
                cm1 = fminf(cm1, a1);
                cm2 = fminf(cm2, a2);
                cm3 = fminf(cm3, a3);
                rmv[u] = fminf(fminf(a0, a1), fminf(a2, a3));
            }
        }
        if (POLICY != kAvg) {  // the same transposed reduction for the row minima (order-free)
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
            float k4[4], k2[2];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                k4[k] = fminf(b4 ? rmv[k + 4] : rmv[k], __shfl_xor_sync(0xffffffffu, b4 ? rmv[k] : rmv[k + 4], 16));
#pragma unroll
            for (int k = 0; k < 2; ++k)
                k2[k] = fminf(b3 ? k4[k + 2] : k4[k], __shfl_xor_sync(0xffffffffu, b3 ? k4[k] : k4[k + 2], 8));
            float v = fminf(b2 ? k2[1] : k2[0], __shfl_xor_sync(0xffffffffu, b2 ? k2[0] : k2[1], 4));
            v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 1));
            const int r = r0 + rb + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
            if ((lane & 3) == 0 && r < rows) atomicMin(row_min + r, fbits(v));
        }
        if (POLICY == kAvg) {
            // the 8 row partials of the warp reduced together: each exchange halves
            // the rows a lane keeps (9 double shuffles instead of 8 x 5); any order of
            // the fp64 additions is covered by the verified-mean bound
            static_assert(kBatch == 8, "transposed reduction of 8 rows");
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
            double k4[4], k2[2];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double send = b4 ? rsv[k] : rsv[k + 4];
                k4[k] = __dadd_rn(b4 ? rsv[k + 4] : rsv[k], __shfl_xor_sync(0xffffffffu, send, 16));
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double send = b3 ? k4[k] : k4[k + 2];
                k2[k] = __dadd_rn(b3 ? k4[k + 2] : k4[k], __shfl_xor_sync(0xffffffffu, send, 8));
            }
            double v = __dadd_rn(b2 ? k2[1] : k2[0], __shfl_xor_sync(0xffffffffu, b2 ? k2[0] : k2[1], 4));
            v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1));
            const int r = r0 + rb + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
            if ((lane & 3) == 0 && r < rows) atomicAdd(row_sum + r, v);
        }
    }
    if (c < cols) {
        if (POLICY == kAvg) {
            atomicAdd(col_sum + c, cs0);
            if (c + 1 < cols) atomicAdd(col_sum + c + 1, cs1);
            if (c + 2 < cols) atomicAdd(col_sum + c + 2, cs2);
            if (c + 3 < cols) atomicAdd(col_sum + c + 3, cs3);
        } else {
            atomicMin(col_min + c, fbits(cm0));
            if (c + 1 < cols) atomicMin(col_min + c + 1, fbits(cm1));
            if (c + 2 < cols) atomicMin(col_min + c + 2, fbits(cm2));
            if (c + 3 < cols) atomicMin(col_min + c + 3, fbits(cm3));
        }
    }
}

// float(S / n) with a proof that the reference's sequential sum rounds the
// same; returns false when the interval straddles a float rounding boundary.
__device__ __forceinline__ void mean_candidates(double S, int nterms, double n, float& lo, float& hi,
                                                int widen = 0) {
    const double u = 1.1102230246251565e-16;  // 2^-53
    const double k = (double)(nterms > 1 ? nterms - 1 : 0);
    const double gam = (k * u) / (1.0 - k * u);
    const double delta = ldexp(4.0 * gam * S, widen);
    lo = __double2float_rn(__ddiv_rn(__dsub_rn(S, delta), n));
    hi = __double2float_rn(__ddiv_rn(__dadd_rn(S, delta), n));
}
__device__ __forceinline__ bool verified_mean(double S, int nterms, double n, float& out, int widen) {
    float lo, hi;
    mean_candidates(S, nterms, n, lo, hi, widen);
    out = lo == hi ? lo : __double2float_rn(__ddiv_rn(S, n));
    return lo == hi;
}

__global__ void k_finalize_avg(const double* row_sum, const double* col_sum, int rows, int cols,
                               int col_n, float* row_stat, float* col_stat, int* flags, int* nflag,
                               int widen) {
    XG_PDL_WAIT();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows + cols) return;
    float v;
    bool ok;
    if (i < rows) {
        ok = verified_mean(row_sum[i], cols, (double)cols, v, widen);
        row_stat[i] = v;
    } else {
        ok = verified_mean(col_sum[i - rows], col_n, (double)col_n, v, widen);
        col_stat[i - rows] = v;
    }
    if (!ok) flags[atomicAdd(nflag, 1)] = i;
}

// Exact reference order for the flagged statistics: the CTA stages the slice
// through shared memory, one thread adds sequentially (pipeline.cpp:219-229).
//
// Deferred mode (`def.a != nullptr`, the pipeline without a stage dump): a
// statistic only matters through its threshold t = M * stat (sparse.cpp:49-65),
// and the reference's float mean is one of the two candidates lo/hi bracketing
// the verified interval.  The kept set of the operand slice (row i of A for a
// row statistic, column j of B for a column statistic) is the same under both
// candidates unless some |x| lies in [float_above(M*lo), float_above(M*hi)).
// One parallel scan of that slice decides; only then is the sequential sum
// paid (the mean stays `lo` otherwise: it is never observable).
constexpr int kChunk = 2048;
constexpr int kFallbackThreads = 1024;  // the membership scan is latency-bound: many loads in flight
__global__ void __launch_bounds__(kFallbackThreads)
    k_fallback_avg(const float* __restrict__ d, int rows, int cols, int col_n, const int* flags,
                   const int* nflag, float* row_stat, float* col_stat, const double* row_sum,
                   const double* col_sum, const StatsDefer def) {
    XG_PDL_WAIT();
    __shared__ float buf[kChunk];
    const int nf = *nflag;
    for (int f = blockIdx.x; f < nf; f += gridDim.x) {
        const int idx = flags[f];
        const bool is_row = idx < rows;
        const int len = is_row ? cols : col_n;
        if (def.a) {
            const double S = is_row ? row_sum[idx] : col_sum[idx - rows];
            float lo, hi;
            mean_candidates(S, len, (double)len, lo, hi, def.widen);
            const float tlo = float_above(__dmul_rn(def.thr_m, (double)lo));
            const float thi = float_above(__dmul_rn(def.thr_m, (double)hi));
            int amb = 0;
            // unrolled so a thread's loads (strided for a column) are all in flight at
            // once instead of one DRAM round trip per iteration (9.6 -> ~3 us at C3)
#pragma unroll 8
            for (int t = threadIdx.x; t < def.inner; t += kFallbackThreads) {
                const float x = is_row ? def.a[(int64_t)idx * def.lda + t]
                                       : def.b[(int64_t)t * def.ldb + (idx - rows)];
                amb |= (fabsf(x) >= tlo && fabsf(x) < thi) ? 1 : 0;
            }
            if (!__syncthreads_or(amb)) continue;  // uniform: membership identical under lo and hi
            if (!is_row && def.remote_cols) {      // row-sharded: the column spans other ranks
                if (threadIdx.x == 0) {
                    const int slot = atomicAdd(def.n_remote, 1);
                    if (slot < def.remote_cap) def.remote_cols[slot] = idx - rows;
                }
                continue;
            }
        }
        double s = 0.0;
        for (int base = 0; base < len; base += kChunk) {
            const int cnt = min(kChunk, len - base);
            for (int t = threadIdx.x; t < cnt; t += kFallbackThreads) {
                const int64_t off = is_row ? (int64_t)idx * cols + base + t
                                           : (int64_t)(base + t) * cols + (idx - rows);
                buf[t] = d[off];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
#pragma unroll 16
                for (int t = 0; t < cnt; ++t) s = __dadd_rn(s, fabs((double)buf[t]));
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const float v = __double2float_rn(__ddiv_rn(s, (double)len));
            if (is_row) row_stat[idx] = v;
            else col_stat[idx - rows] = v;
        }
    }
}

__global__ void k_zero(double* a, int na, double* b, int nb, int* n) {
    XG_PDL_WAIT();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) a[i] = 0.0;
    if (i < nb) b[i] = 0.0;
    if (i == 0) *n = 0;
}

}  // namespace

// One launch for all the per-call initialisation of the device pipeline:
// device scalars, column-max accumulators and the statistics accumulators
// (fp64 sums for AvgRule, FLT_MAX bit patterns for MinRule).
__global__ void k_pipe_init(uint32_t* sc, int sc_words, uint32_t* colmax, int N, double* rsum,
                            double* csum, uint32_t* rmin, uint32_t* cmin, int M, int policy, int reduce,
                            unsigned long long* ts0) {
    XG_PDL_WAIT();
    unsigned long long t0 = 0;
    if (ts0 && blockIdx.x == 0 && threadIdx.x == 0) t0 = globaltimer_ns();
    const int n = max(max(M, N), sc_words);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i < sc_words) sc[i] = 0u;
        if (i < N && colmax) colmax[i] = 0u;
        if (reduce) {
            if (policy == kAvg) {
                if (i < M) rsum[i] = 0.0;
                if (i < N) csum[i] = 0.0;
            } else {
                if (i < M) rmin[i] = 0x7f7fffffu;
                if (i < N) cmin[i] = 0x7f7fffffu;
            }
        }
    }
    if (ts0 && blockIdx.x == 0) {  // the scalars (block 0's range) are zero: stamp the start
        __syncthreads();
        if (threadIdx.x == 0) *ts0 = t0;
    }
}

void launch_pipe_init(void* sc, int sc_bytes, uint32_t* colmax, int N, double* rsum, double* csum,
                      float* rstat, float* cstat, int M, int policy, int reduce, cudaStream_t s,
                      unsigned long long* ts0) {
    const int n = M > N ? M : N;
    int blocks = (n + 255) / 256;
    blocks = blocks < 1 ? 1 : blocks > 1024 ? 1024 : blocks;
    k_pipe_init<<<blocks, 256, 0, s>>>(reinterpret_cast<uint32_t*>(sc), sc_bytes / 4, colmax, N, rsum, csum,
                                        reinterpret_cast<uint32_t*>(rstat), reinterpret_cast<uint32_t*>(cstat), M,
                                        policy, reduce, ts0);
}

void launch_stats_partial(const float* d, int rows, int cols, int policy, float* row_stat,
                          float* col_stat, double* row_sum, double* col_sum, int* nflag, cudaStream_t s,
                          int mode) {
    dim3 grid((cols + kThreads * 4 - 1) / (kThreads * 4), (rows + kSlabRows - 1) / kSlabRows);
    // 128-row slabs (half the column atomics again: 49 -> 47 us at C3) while the
    // grid still has >= 2 CTAs per SM; 64 otherwise (C2 would get 128 CTAs)
    const bool big = (int64_t)grid.x * ((rows + 127) / 128) >= 2 * 148;
    if (big) grid.y = (rows + 127) / 128;
    // grids below one CTA per SM (C1: 16 CTAs): 8-row slabs (C1 reduce 29 -> 26 us;
    // shrinking them on larger grids measured slower, C2 82 -> 93 us)
    int slab = big ? 128 : 64;
    if (!big && (int64_t)grid.x * grid.y < 148) {
        slab = 8;
        grid.y = (rows + 7) / 8;
    }
    if (policy == kAvg) {
        const int nz = rows > cols ? rows : cols;
        if (mode != 2) k_zero<<<(nz + 255) / 256, 256, 0, s>>>(row_sum, rows, col_sum, cols, nflag);
        if (mode != 1) {
            if (slab == 128) k_stats_slab<kAvg, 128><<<grid, kThreads, 0, s>>>(d, rows, cols, row_sum, col_sum, nullptr, nullptr);
            else if (slab == 64) k_stats_slab<kAvg><<<grid, kThreads, 0, s>>>(d, rows, cols, row_sum, col_sum, nullptr, nullptr);
            else k_stats_slab<kAvg, 8><<<grid, kThreads, 0, s>>>(d, rows, cols, row_sum, col_sum, nullptr, nullptr);
        }
    } else {
        // the float bit patterns of |x| order like uints; FLT_MAX initial value (pipeline.cpp:237-238)
        if (mode != 2) {
            fill_u32(reinterpret_cast<uint32_t*>(row_stat), 0x7f7fffffu, rows, s);
            fill_u32(reinterpret_cast<uint32_t*>(col_stat), 0x7f7fffffu, cols, s);
        }
        if (mode != 1) {
            uint32_t* rmn = reinterpret_cast<uint32_t*>(row_stat);
            uint32_t* cmn = reinterpret_cast<uint32_t*>(col_stat);
            if (slab == 128) k_stats_slab<kMin, 128><<<grid, kThreads, 0, s>>>(d, rows, cols, nullptr, nullptr, rmn, cmn);
            else if (slab == 64) k_stats_slab<kMin><<<grid, kThreads, 0, s>>>(d, rows, cols, nullptr, nullptr, rmn, cmn);
            else k_stats_slab<kMin, 8><<<grid, kThreads, 0, s>>>(d, rows, cols, nullptr, nullptr, rmn, cmn);
        }
    }
}

void launch_stats_final(const float* d, int rows, int cols, int col_n, int policy, float* row_stat,
                        float* col_stat, double* row_sum, double* col_sum, int* flags, int* nflag,
                        cudaStream_t s, const StatsDefer* def) {
    if (policy != kAvg) return;  // MinRule statistics are final after the partial pass (and min-reduce)
    k_finalize_avg<<<(rows + cols + 255) / 256, 256, 0, s>>>(row_sum, col_sum, rows, cols, col_n, row_stat,
                                                             col_stat, flags, nflag, def ? def->widen : 0);
    k_fallback_avg<<<64, kFallbackThreads, 0, s>>>(d, rows, cols, col_n, flags, nflag, row_stat, col_stat,
                                                   row_sum, col_sum, def ? *def : StatsDefer{});
}

void launch_stats(const float* d, int rows, int cols, int policy, float* row_stat, float* col_stat,
                  double* row_sum, double* col_sum, int* flags, int* nflag, cudaStream_t s,
                  const StatsDefer* def) {
    launch_stats_partial(d, rows, cols, policy, row_stat, col_stat, row_sum, col_sum, nflag, s);
    launch_stats_final(d, rows, cols, rows, policy, row_stat, col_stat, row_sum, col_sum, flags, nflag, s, def);
}

// Row-sharded rare path: exact sequential column sums (pipeline.cpp:219-229,
// i outer in global row order) of the listed columns from the gathered
// per-rank slices gath[rank][slot][row] (rank r holds rank_rows[r] rows).
__global__ void k_remote_col_means(const float* gath, int g, const int* rank_rows, int mpad, int cap,
                                   const int* cols_list, const int* n_list, int col_n, float* col_stat) {
    XG_PDL_WAIT();
    const int n = min(*n_list, cap);
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < g; ++r) {
            const float* src = gath + ((int64_t)r * cap + f) * mpad;
            for (int i = 0; i < rank_rows[r]; ++i) s = __dadd_rn(s, fabs((double)src[i]));
        }
        col_stat[cols_list[f]] = __double2float_rn(__ddiv_rn(s, (double)col_n));
    }
}

// Packs D_F[:, j] of the listed columns into buf[slot][row] (rows padded to mpad).
__global__ void k_pack_cols(const float* d, int rows, int cols, const int* cols_list, const int* n_list,
                            int cap, int mpad, float* buf) {
    XG_PDL_WAIT();
    const int n = min(*n_list, cap);
    for (int f = blockIdx.y; f < n; f += gridDim.y)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mpad; i += gridDim.x * blockDim.x)
            buf[(int64_t)f * mpad + i] = i < rows ? d[(int64_t)i * cols + cols_list[f]] : 0.0f;
}

// Every rank finds the same set of columns, but atomics fill the list in any
// order: sort it so the gathered slices line up across ranks.
__global__ void k_sort_list(int* list, const int* n_list, int cap) {
    XG_PDL_WAIT();
    const int n = min(*n_list, cap);
    for (int i = 1; i < n; ++i) {
        const int v = list[i];
        int j = i - 1;
        while (j >= 0 && list[j] > v) {
            list[j + 1] = list[j];
            --j;
        }
        list[j + 1] = v;
    }
}

void launch_pack_remote_cols(const float* d, int rows, int cols, const int* list, const int* n, int cap,
                             int mpad, float* buf, cudaStream_t s) {
    k_sort_list<<<1, 1, 0, s>>>(const_cast<int*>(list), n, cap);
    dim3 grid((mpad + 255) / 256 < 64 ? (mpad + 255) / 256 : 64, cap);
    k_pack_cols<<<grid, 256, 0, s>>>(d, rows, cols, list, n, cap, mpad, buf);
}

void launch_remote_col_means(const float* gath, int g, const int* rank_rows, int mpad, int cap,
                             const int* list, const int* n, int col_n, float* col_stat, cudaStream_t s) {
    k_remote_col_means<<<1, 32, 0, s>>>(gath, g, rank_rows, mpad, cap, list, n, col_n, col_stat);
}

}  // namespace xg
