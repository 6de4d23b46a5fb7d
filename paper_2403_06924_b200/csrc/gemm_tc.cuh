// K2 / K4+K5: persistent warp-specialised INT8 x INT8 -> INT32 GEMM on the
// 5th-generation tensor cores (tcgen05.mma kind::i8), TMA-fed shared-memory
// stages, accumulators in TMEM, and fused epilogues that apply the
// reference's exact dequantisation / compensation arithmetic.
//
// Replaces the reference hot loops
//   gemm_int          quantize.cpp:193-214   (i-k-j triple loop)
//   dequant_product   quantize.cpp:169-187   (fused into EPI_DF)
//   spmm_int x2       sparse.cpp:119-138 + pipeline.cpp:118-124 (masked-dense,
//                     bit-identical integer sums; EPI_COMP)
//   add_inplace x2    pipeline.cpp:141-145, axpby pipeline.cpp:195-202 (EPI_COMP)
//
// Operand layout: every operand is K-major int8 (A: rows x K, B^T: cols x K)
// with a row pitch that is a multiple of 16 bytes; TMA zero-fills the ragged
// edges so any M, N, K >= 1 runs through the same kernel.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace xg {

enum EpiMode : int {
    EPI_S32 = 0,   // store raw s32 accumulator
    EPI_DF = 1,    // store float(acc / (la_i * lb_j))
    EPI_COMP = 2,  // store ((D_F + float(acc0/(l1_i*l2_j))) + float(acc1/(l3_i*l4_j))), alpha/beta
    EPI_FULL3 = 3, // full residual: ((float(acc0/s0) + float(acc1/s1)) + float(acc2/s2))
    EPI_ACC = 4    // out = float(din + float(acc/(l_i*l_j))), then alpha/beta if `finalize`
};

struct ScaleRef {  // per-row (stride 1) or per-tensor (stride 0) fp64 scales
    const double* p;
    int stride;
    const float2* r;  // optional ff_recip(p[i]) written by the scale's producer (same stride)
    __device__ __forceinline__ double at(int i) const { return p[(int64_t)i * stride]; }
    __device__ __forceinline__ float2 rcp(int i) const { return r ? r[(int64_t)i * stride] : ff_recip(at(i)); }
};

constexpr int kMaxMaps = 6;

struct TmaMaps {
    CUtensorMap m[kMaxMaps];
};

// fp32 M x N output (and D_F input) maps: 32x32 boxes, 128-byte swizzle.
struct EpiMaps {
    CUtensorMap out;
    CUtensorMap din;
};

struct GemmArgs {
    int M, N, K;
    // operand map indices for accumulator a: [a][sel]
    int amap[3][2];
    int bmap[3][2];
    const int* sel_ptr;  // device flag choosing column 1 of the index tables (nullable)
    // the CUDA-core CSR path (spmm.cu) serves the call when *skip_ptr && !*skip_veto:
    // the launch then does no tile (and writes no stage stamps)
    const int* skip_ptr;
    const int* skip_veto;
    // epilogue
    int32_t* out_s32;
    float* out_f32;
    const float* df_in;  // EPI_COMP: D_F (may alias out_f32)
    const float* c_in;   // EPI_COMP: optional C for alpha*D + beta*C
    float alpha, beta;
    int has_c;
    // row scales / col scales per accumulator, [acc][sel]
    ScaleRef rs[3][2];
    ScaleRef cs[3][2];
    int debug;  // probes: bit 0 skip TMA loads (MMA on stale smem), bit 1 skip epilogue work
    int finalize;  // EPI_ACC: apply the alpha/beta tail (pipeline.cpp:195-202)
    int dual;      // pair EPI_ACC: both compensation terms per tile (term 0: amap/bmap/rs/cs[0],
                   // out = fl(din + deq); term 1: [1], finalize), TMEM buffers alternate by term
    int group_m;   // pair kernel: tile-raster group height in 256-row units (0: default)
    int pf_dist;   // pair kernel: L2 prefetch distance in k-blocks (0: off)
    unsigned long long* stamp;  // pair kernel: [0] %globaltimer at begin, [1] max at CTA exit (null: off)
    // pair kernel: the last CTA to finish copies rep_words words from rep_src to
    // rep_dst (the caller's pinned report, device-mapped) - no D2H copy node
    unsigned* done;
    const uint32_t* rep_src;
    uint32_t* rep_dst;
    int rep_words;
    int rep_flag;  // word of rep_dst written last (after a system fence); 0: none
};

template <int BN, int NACC>
struct GemmCfg {
    static constexpr int BM = 128;
    static constexpr int BK = 128;  // bytes == int8 elements; one 128B swizzle row
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = BN * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES;
    static constexpr int ACC_COLS = NACC * BN;
    static constexpr int ACC_BUFS = (512 / ACC_COLS) >= 2 ? 2 : 1;
    static constexpr int TMEM_COLS = ACC_BUFS * ACC_COLS <= 256 ? 256 : 512;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int GROUP_M = 16;
    static_assert(ACC_COLS * ACC_BUFS <= 512, "TMEM overflow");
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group_m, int& mb,
                                            int& nb) {
    const int per_group = group_m * num_n;
    const int g = t / per_group;
    const int first = g * group_m;
    const int gm = min(group_m, num_m - first);
    const int w = t - g * per_group;
    mb = first + w % gm;
    nb = w / gm;
    if (g & 1) nb = num_n - 1 - nb;  // serpentine: a group starts on the B panels the previous one ended on
}

// Column j's scale and its reciprocal live in lane j of the warp (computed once
// per 32-column chunk), fetched with a shuffle.
struct ColScale {
    double lam, inv;
    __device__ __forceinline__ void load(const ScaleRef& s, int col) {
        lam = s.at(col);
        inv = __ddiv_rn(1.0, lam);
    }
    __device__ __forceinline__ double lam_of(int j) const { return __shfl_sync(0xffffffffu, lam, j); }
    __device__ __forceinline__ double inv_of(int j) const { return __shfl_sync(0xffffffffu, inv, j); }
};

template <int NACC, int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& args, int sel,
                                               const uint32_t (&acc)[NACC][32], int row,
                                               int col0, double r0, double r1, double r2,
                                               double i0, double i1, double i2, bool active) {
    const int64_t obase = (int64_t)row * args.N + col0;
    const int ncol = min(32, args.N - col0);
    const bool full = ((args.N & 3) == 0) && ncol == 32;
    const int lane = threadIdx.x & 31;
    const int mycol = min(col0 + lane, args.N - 1);
    if constexpr (EPI == EPI_S32) {
        if (!active) return;
        int32_t* o = args.out_s32 + obase;
        if (full) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
                reinterpret_cast<int4*>(o)[v] = make_int4(acc[0][4 * v], acc[0][4 * v + 1],
                                                          acc[0][4 * v + 2], acc[0][4 * v + 3]);
        } else {
            for (int j = 0; j < ncol; ++j) o[j] = (int32_t)acc[0][j];
        }
    } else {
        float res[32];
        if constexpr (EPI == EPI_DF) {
            ColScale c0;
            c0.load(args.cs[0][sel], mycol);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                res[j] = dequant_product_fast((int32_t)acc[0][j], i0, c0.inv_of(j), r0, c0.lam_of(j));
            if (!active) return;
        } else if constexpr (EPI == EPI_COMP) {
            ColScale c0, c1;
            c0.load(args.cs[0][sel], mycol);
            c1.load(args.cs[1][sel], mycol);

            float din[32], cin[32];
            const float* dp = args.df_in + obase;
            const float* cp = args.c_in + obase;
            if (!active) {  // rows past M: compute on zeros, store nothing
#pragma unroll
                for (int j = 0; j < 32; ++j) din[j] = cin[j] = 0.0f;
            } else if (full) {
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const float4 x = reinterpret_cast<const float4*>(dp)[v];
                    din[4 * v] = x.x; din[4 * v + 1] = x.y; din[4 * v + 2] = x.z; din[4 * v + 3] = x.w;
                }
                if (args.has_c) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const float4 x = reinterpret_cast<const float4*>(cp)[v];
                        cin[4 * v] = x.x; cin[4 * v + 1] = x.y; cin[4 * v + 2] = x.z; cin[4 * v + 3] = x.w;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    din[j] = j < ncol ? dp[j] : 0.0f;
                    cin[j] = (args.has_c && j < ncol) ? cp[j] : 0.0f;
                }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                // pipeline.cpp:134-145: d_f += dr1; d_f += dr2 (fp32, this order)
                const float t1 = dequant_product_fast((int32_t)acc[0][j], i0, c0.inv_of(j), r0, c0.lam_of(j));
                const float t2 = dequant_product_fast((int32_t)acc[1 % NACC][j], i1, c1.inv_of(j), r1, c1.lam_of(j));
                float v = __fadd_rn(__fadd_rn(din[j], t1), t2);
                // pipeline.cpp:195-202 / matrix.cpp:102 (non-fused)
                if (args.has_c) v = __fadd_rn(__fmul_rn(args.alpha, v), __fmul_rn(args.beta, cin[j]));
                else if (args.alpha != 1.0f) v = __fmul_rn(v, args.alpha);
                res[j] = v;
            }
            if (!active) return;
        } else {  // EPI_FULL3
            ColScale c0, c1, c2;
            c0.load(args.cs[0][sel], mycol);
            c1.load(args.cs[1][sel], mycol);
            c2.load(args.cs[2][sel], mycol);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float t0 = dequant_product_fast((int32_t)acc[0][j], i0, c0.inv_of(j), r0, c0.lam_of(j));
                const float t1 = dequant_product_fast((int32_t)acc[1 % NACC][j], i1, c1.inv_of(j), r1, c1.lam_of(j));
                const float t2 = dequant_product_fast((int32_t)acc[2 % NACC][j], i2, c2.inv_of(j), r2, c2.lam_of(j));
                res[j] = __fadd_rn(__fadd_rn(t0, t1), t2);
            }
            if (!active) return;
        }
        float* o = args.out_f32 + obase;
        if (full) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
                reinterpret_cast<float4*>(o)[v] =
                    make_float4(res[4 * v], res[4 * v + 1], res[4 * v + 2], res[4 * v + 3]);
        } else {
            for (int j = 0; j < ncol; ++j) o[j] = res[j];
        }
    }
}

template <int BN, int NACC, int EPI>
__global__ void __launch_bounds__(256, 1)
    k_gemm_i8_tc(const __grid_constant__ TmaMaps maps, const GemmArgs args) {
    using Cfg = GemmCfg<BN, NACC>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the shared array (not through
    // uintptr_t) so the compiler keeps shared-space accesses (LDS/STS, not LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = (uint64_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_m = (args.M + Cfg::BM - 1) / Cfg::BM;
    const int num_n = (args.N + BN - 1) / BN;
    const int num_tiles_all = num_m * num_n;
    const int nkb = (args.K + Cfg::BK - 1) / Cfg::BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kMaxMaps; ++i) tma_prefetch(&maps.m[i]);
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    XG_PDL_WAIT_ONLY();
    const int sel = args.sel_ptr ? (*args.sel_ptr != 0) : 0;
    const bool skip = args.skip_ptr && *args.skip_ptr && !(args.skip_veto && *args.skip_veto);
    const int num_tiles = skip ? 0 : num_tiles_all;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int mb, nb;
                tile_coords(t, num_m, num_n, Cfg::GROUP_M, mb, nb);
                for (int kb = 0; kb < nkb; ++kb) {
                    for (int a = 0; a < NACC; ++a) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                        uint8_t* sB = sA + Cfg::A_BYTES;
                        mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                        tma_load_2d(sA, &maps.m[args.amap[a][sel]], &full[stage], kb * Cfg::BK,
                                    mb * Cfg::BM);
                        tma_load_2d(sB, &maps.m[args.bmap[a][sel]], &full[stage], kb * Cfg::BK,
                                    nb * BN);
                        if (++stage == Cfg::STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread) =====================
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_i8(Cfg::BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int buf = 0;
            uint32_t bphase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                mbar_wait(&tempty[buf], bphase ^ 1);
                tc_fence_after();
                const uint32_t dbase = tmem_base + buf * Cfg::ACC_COLS;
                for (int kb = 0; kb < nkb; ++kb) {
                    for (int a = 0; a < NACC; ++a) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                        const uint64_t da = smem_desc_k128(sA);
                        const uint64_t db = smem_desc_k128(sA + Cfg::A_BYTES);
#pragma unroll
                        for (int k = 0; k < Cfg::BK / 32; ++k) {
                            // +32 bytes along K inside the 128B swizzle row: +2 in the
                            // (addr >> 4) start-address field.
                            mma_i8(dbase + a * BN, da + 2 * k, db + 2 * k, idesc,
                                   (kb | k) != 0 ? 1u : 0u);
                        }
                        tc_commit(&empty[stage]);
                        if (++stage == Cfg::STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                tc_commit(&tfull[buf]);
                if (++buf == Cfg::ACC_BUFS) {
                    buf = 0;
                    bphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (4 warps, 128 TMEM lanes) =====================
        const int q = warp & 3;  // TMEM lane quadrant owned by this warp
        int buf = 0;
        uint32_t bphase = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int mb, nb;
            tile_coords(t, num_m, num_n, Cfg::GROUP_M, mb, nb);
            mbar_wait(&tfull[buf], bphase);
            tc_fence_after();
            const int row = mb * Cfg::BM + q * 32 + lane;
            const bool row_ok = row < args.M;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + buf * Cfg::ACC_COLS;
            double r0 = 1.0, r1 = 1.0, r2 = 1.0;
            if (EPI != EPI_S32 && row_ok) {  // row scales are fixed per thread
                r0 = args.rs[0][sel].at(row);
                if (NACC > 1) r1 = args.rs[1][sel].at(row);
                if (NACC > 2) r2 = args.rs[2][sel].at(row);
            }
            const double i0 = __ddiv_rn(1.0, r0), i1 = __ddiv_rn(1.0, r1), i2 = __ddiv_rn(1.0, r2);
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t acc[NACC][32];
#pragma unroll
                for (int a = 0; a < NACC; ++a) tmem_ld32(tbase + a * BN + c * 32, acc[a]);
                tmem_ld_wait();
                const int col0 = nb * BN + c * 32;
                if (col0 < args.N)  // warp-uniform; per-thread row validity passed down
                    epilogue_chunk<NACC, EPI>(args, sel, acc, row, col0, r0, r1, r2, i0, i1, i2, row_ok);
                __syncwarp();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if (++buf == Cfg::ACC_BUFS) {
                buf = 0;
                bphase ^= 1;
            }
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace xg

namespace xg {

// ---------------------------------------------------------------------------
// CTA-pair version (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile with one tcgen05.mma.cta_group::2 (M=256, N=256, K=32)
// issued by the leader.  Each CTA stages its own 128 rows of A and its own 128
// rows of B^T, so per-SM operand traffic is (128+128) B per K byte instead of
// (128+256) for the 1-CTA 128x256 tile: 64 B/clk/SM at full MMA rate.  The
// accumulator rows 0-127 land in the leader's TMEM, 128-255 in the peer's.
// 8 epilogue warps (two per TMEM lane quadrant, one per 128-column half).
template <int NACC, int EPI = EPI_DF, int ST = 0>
struct Gemm2Cfg {
    static constexpr int BM = 128;   // rows per CTA (pair M = 256)
    static constexpr int BN = 256;   // pair N
    static constexpr int BNH = 128;  // B^T rows staged per CTA
    static constexpr int BK = 128;
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = BNH * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr bool LOADS_DIN = EPI == EPI_COMP || EPI == EPI_ACC;
    // Stages of the operand ring: the D_F GEMM at 4 stages is 11% slower than at 5
    // (8192^3); the compensation GEMM, whose operands miss L2 more, went 0.711 ->
    // 0.639 -> 0.608 ms with a fifth and a sixth (C3; at K <= 4096 unchanged
    // within 1%).  The two-accumulator EPI_COMP has room for 4.  ST overrides.
    static constexpr int STAGES = ST > 0 ? ST : (LOADS_DIN ? (NACC > 1 ? 4 : 6) : 5);
    // epilogue chunk width (columns per TMEM load / staging tile): 16 (64B-swizzled
    // 32x16 tiles) for the compensation GEMM, whose smaller staging tiles leave
    // room for the sixth stage, and for the D_F GEMM (two tiles in the space of
    // one 32x32: stores overlap the next chunk); 32 (128B swizzle) for EPI_COMP
    static constexpr int CHW = ((EPI == EPI_ACC && STAGES >= 5) || EPI == EPI_DF) ? 16 : 32;
    static constexpr int ACC_COLS = NACC * BN;
    static constexpr int ACC_BUFS = (512 / ACC_COLS) >= 2 ? 2 : 1;
    static constexpr int TMEM_COLS = 512;
    static constexpr int THREADS = 384;
    static constexpr int EPI_WARPS = 8;
    // per epilogue warp: NSTG staging tiles of 32 x CHW fp32 (TMA store / load;
    // D_F loads run NSTG-1 chunks ahead) and NACC x 32 float-float column
    // reciprocals.  The five-stage compensation variant (K <= 4096, where the
    // epilogue bounds the tile) spends the sixth stage's 32 KB on four tiles
    static constexpr int NSTG = LOADS_DIN ? ((EPI == EPI_ACC && ST == 5) ? 4 : 2) : (CHW == 16 ? 2 : 1);
    static constexpr int STG_BYTES = 32 * CHW * 4;
    static constexpr int EPI_BYTES = EPI_WARPS * NSTG * STG_BYTES;
    static constexpr int SCL_BYTES = EPI_WARPS * NACC * 32 * 8;
    // alignment slack for the 1024-byte (128B-swizzle) tiles: the dynamic window
    // starts after the driver's 1 KiB on sm_100, so none is consumed in practice;
    // the kernel traps if more than the slack would be needed
    static constexpr int ALIGN_SLACK = LOADS_DIN ? 512 : 1024;
    static constexpr int NBUF = NSTG > 2 ? NSTG : 2;  // D_F load barriers per epilogue warp
    static constexpr int BAR_BYTES = (2 * STAGES + 4 + NBUF * EPI_WARPS) * 8 + 4 <= 256 ? 256 : 512;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + SCL_BYTES + ALIGN_SLACK + BAR_BYTES;
    static_assert(SMEM_BYTES <= 232448, "shared memory over the 227 KiB per-block limit");
    static_assert((2 * STAGES + 4 + NBUF * EPI_WARPS) * 8 + 4 <= BAR_BYTES, "barrier area");
    static constexpr int GROUP_M = 16;  // in 256-row units (measured: 16 > 8 > 32 at 8192^3)
    static_assert(ACC_COLS * ACC_BUFS <= 512, "TMEM overflow");
};

// PAIRS = 2: a 4-CTA cluster of two pairs stacked along M sharing B^T tiles
// through TMA multicast (not instantiated: measured slower on B200, fewer co-resident
// clusters).  Stages may only be overwritten once BOTH pairs' MMAs are done, so
// the MMA commits that free stages are multicast to all four CTAs.
//
// Epilogue: TMEM -> registers -> exact dequant -> 128B-swizzled smem tile ->
// TMA store; EPI_COMP prefetches its D_F tile by TMA into the same staging
// tile while the accumulator is still being produced.
template <int NACC, int EPI, int PAIRS, int ST = 0>
__global__ void __launch_bounds__(384, 1)
    k_gemm_i8_tc2(const __grid_constant__ TmaMaps maps, const GemmArgs args,
                  const __grid_constant__ EpiMaps emaps) {
    using Cfg = Gemm2Cfg<NACC, EPI, ST>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the shared array (not through
    // uintptr_t) so the compiler keeps shared-space accesses (LDS/STS, not LD/ST)
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    if (pad > (uint32_t)Cfg::ALIGN_SLACK) __trap();  // see Gemm2Cfg::ALIGN_SLACK
    uint8_t* smem = smem_raw + pad;
    float* epi_stage = (float*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);  // 1024-aligned
    double* epi_scale = (double*)((uint8_t*)epi_stage + Cfg::EPI_BYTES);
    uint64_t* full = (uint64_t*)((uint8_t*)epi_scale + Cfg::SCL_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    constexpr int NBUF = Cfg::NBUF;
    uint64_t* dbar = tempty + 2;  // [EPI_WARPS][NBUF] D_F tile loads
    uint32_t* tmem_slot = (uint32_t*)(dbar + NBUF * Cfg::EPI_WARPS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const uint32_t prank = rank & 1;                 // rank inside the pair
    const uint32_t pair = rank >> 1;                 // pair inside the cluster
    const bool leader = prank == 0;                  // pair leader issues the MMA
    const int cluster_id = blockIdx.x / (2 * PAIRS);
    const int nclusters = gridDim.x / (2 * PAIRS);
    const int num_m = (args.M + 2 * PAIRS * Cfg::BM - 1) / (2 * PAIRS * Cfg::BM);
    const int num_n = (args.N + Cfg::BN - 1) / Cfg::BN;
    const int num_tiles_all = num_m * num_n;
    const int nkb = (args.K + Cfg::BK - 1) / Cfg::BK;
    const int gm = args.group_m > 0 ? args.group_m : Cfg::GROUP_M;

    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], PAIRS);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * Cfg::EPI_WARPS);
        }
        for (int b = 0; b < NBUF * Cfg::EPI_WARPS; ++b) mbar_init(&dbar[b], 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kMaxMaps; ++i) tma_prefetch(&maps.m[i]);
        tma_prefetch(&emaps.out);
        tma_prefetch(&emaps.din);
    }
    if (warp == 2) tmem_alloc2(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // everything above overlaps the predecessor's tail under a programmatic edge
    XG_PDL_WAIT_ONLY();
    const bool skip = args.skip_ptr && *args.skip_ptr && !(args.skip_veto && *args.skip_veto);
    const int num_tiles = skip ? 0 : num_tiles_all;
    if (args.stamp && !skip && blockIdx.x == 0 && threadIdx.x == 0) args.stamp[0] = globaltimer_ns();
    const int sel = args.sel_ptr ? (*args.sel_ptr != 0) : 0;
    const int nterms = (EPI == EPI_ACC && args.dual) ? 2 : 1;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            const int pf = args.pf_dist;
            int it = 0;  // tiles already issued by this cluster
            for (int t = cluster_id; t < num_tiles; t += nclusters, ++it)
            for (int term = 0; term < nterms; ++term) {
                int mb, nb;
                tile_coords(t, num_m, num_n, gm, mb, nb);
                const int arow = (mb * PAIRS + (int)pair) * 2 * Cfg::BM + (int)prank * Cfg::BM;
                const int brow = nb * Cfg::BN + (int)prank * Cfg::BNH + (int)pair * (Cfg::BNH / PAIRS);
                for (int kb = 0; kb < nkb; ++kb) {
                    if (pf > 0 && nterms == 1 && !(args.debug & 1)) {  // L2 prefetch of the block `pf` ahead in this CTA's stream
                        const int f = it * nkb + kb + pf;
                        const int t2 = cluster_id + (f / nkb) * nclusters, kb2 = f % nkb;
                        if (t2 < num_tiles) {
                            int mb2, nb2;
                            tile_coords(t2, num_m, num_n, gm, mb2, nb2);
                            const int arow2 = (mb2 * PAIRS + (int)pair) * 2 * Cfg::BM + (int)prank * Cfg::BM;
                            const int brow2 = nb2 * Cfg::BN + (int)prank * Cfg::BNH + (int)pair * (Cfg::BNH / PAIRS);
                            for (int a = 0; a < NACC; ++a) {
                                tma_prefetch_l2(&maps.m[args.amap[a][sel]], kb2 * Cfg::BK, arow2);
                                tma_prefetch_l2(&maps.m[args.bmap[a][sel]], kb2 * Cfg::BK, brow2);
                            }
                        }
                    }
                    for (int a = 0; a < NACC; ++a) {
                        const int ai = a + term;  // operand-map index (term selects it in dual mode)
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                        uint8_t* sB = sA + Cfg::A_BYTES;
                        if (args.debug & 1) {  // probe: MMA on stale smem
                            if (leader) mbar_arrive(&full[stage]);
                        } else {
                            if (leader) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
                            tma_load_2d_pair(sA, &maps.m[args.amap[ai][sel]], &full[stage], kb * Cfg::BK, arow);
                            if (PAIRS == 1) {
                                tma_load_2d_pair(sB, &maps.m[args.bmap[ai][sel]], &full[stage], kb * Cfg::BK, brow);
                            } else {
                                tma_load_2d_pair_mc(sB + pair * (Cfg::B_BYTES / PAIRS), &maps.m[args.bmap[ai][sel]],
                                                    &full[stage], kb * Cfg::BK, brow,
                                                    (uint16_t)((1u << rank) | (1u << (rank ^ 2u))));
                            }
                        }
                        if (++stage == Cfg::STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA, one thread) =====================
        if (leader && elect_one()) {
            constexpr uint32_t idesc = idesc_i8(2 * Cfg::BM, Cfg::BN);
            int stage = 0;
            uint32_t phase = 0;
            int buf = 0;
            uint32_t bphase = 0;
            for (int t = cluster_id; t < num_tiles; t += nclusters)
            for (int term = 0; term < nterms; ++term) {
                mbar_wait(&tempty[buf], bphase ^ 1);
                tc_fence_after();
                const uint32_t dbase = tmem_base + buf * Cfg::ACC_COLS;
                for (int kb = 0; kb < nkb; ++kb) {
                    for (int a = 0; a < NACC; ++a) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                        const uint64_t da = smem_desc_k128(sA);
                        const uint64_t db = smem_desc_k128(sA + Cfg::A_BYTES);
#pragma unroll
                        if (!(args.debug & 32))  // probe: skip the MMAs
                            for (int k = 0; k < Cfg::BK / 32; ++k)
                                mma_i8_pair(dbase + a * Cfg::BN, da + 2 * k, db + 2 * k, idesc,
                                            (kb | k) != 0 ? 1u : 0u);
                        if (PAIRS == 1) tc_commit_pair(&empty[stage]);
                        else tc_commit_mc(&empty[stage], (uint16_t)0xF);
                        if (++stage == Cfg::STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                if (PAIRS == 1) tc_commit_pair(&tfull[buf]);
                else tc_commit_mc(&tfull[buf], (uint16_t)(3u << (2 * pair)));
                if (++buf == Cfg::ACC_BUFS) {
                    buf = 0;
                    bphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (8 warps per CTA) =====================
        const int q = warp & 3;            // TMEM lane quadrant
        const int half = (warp - 4) >> 2;  // 128-column half of the tile
        const int we = warp - 4;           // epilogue warp index 0..7
        const uint32_t tempty_leader0 = mapa_shared(&tempty[0], rank & ~1u);
        constexpr int CW = Cfg::CHW;  // chunk width (columns)
        constexpr int KV = CW / 4;     // 16-byte units per staged row
        constexpr int NS = Cfg::NSTG;   // staging tiles of this warp: chunk c uses tile c % NS
        constexpr int PD = NS - 1;      // D_F prefetch distance in chunks
        float* const stg0 = epi_stage + we * NS * (32 * CW);
        float2* scw = reinterpret_cast<float2*>(epi_scale) + we * NACC * 32;
        uint64_t* mybar = dbar + NBUF * we;
        uint32_t dph = 0;  // bit b: phase of tile b's load barrier
        // 128B swizzle (32 columns): unit k of row `lane` sits at k ^ (lane & 7);
        // 64B swizzle (16 columns): at k ^ ((lane >> 1) & 3)
        const int sw = CW == 32 ? (lane & 7) : ((lane >> 1) & 3);
        int buf = 0;
        uint32_t bphase = 0;
        for (int t = cluster_id; t < num_tiles; t += nclusters)
        for (int term = 0; term < nterms; ++term) {
            const int ts = term;  // scale / operand index of this accumulator (0 unless dual)
            const int fin = nterms == 2 ? term : args.finalize;
            int mb, nb;
            tile_coords(t, num_m, num_n, gm, mb, nb);
            const int rowbase = (mb * PAIRS + (int)pair) * 2 * Cfg::BM + (int)prank * Cfg::BM + q * 32;
            const int row = rowbase + lane;
            const bool row_ok = row < args.M;
            const int colbase = nb * Cfg::BN + half * (Cfg::BN / 2);
            const int nchunk = (args.debug & 2) ? 0 : min(Cfg::BN / 2 / CW, (args.N - colbase + CW - 1) / CW);
            // Dual term 1 reads back what term 0 just produced.  It walks the chunks
            // in reverse: the last NS term-0 chunks are still in their staging
            // tiles (chunk c in tile c % NS) and are updated in place; older ones
            // are reloaded once term 0's store of that chunk has landed.
            const bool rev = Cfg::LOADS_DIN && NS >= 2 && nterms == 2 && term == 1;
            const int nres = rev ? min(NS, nchunk) : 0;
            if (Cfg::LOADS_DIN && lane == 0 && !rev) {  // the first D_F chunks while the MMA still runs
                bulk_wait_read<0>();
                for (int cc = 0; cc < PD && cc < nchunk; ++cc) {
                    mbar_expect_tx(&mybar[cc % NS], Cfg::STG_BYTES);
                    tma_load_2d(stg0 + (cc % NS) * (32 * CW), &emaps.din, &mybar[cc % NS], colbase + cc * CW, rowbase);
                }
            }
            // row scales (fp64 for the rare exact redo) and their float-float
            // reciprocals, precomputed by the scale's producer (ScaleRef::r)
            double r0 = 1.0, r1 = 1.0;
            if (row_ok) {
                r0 = args.rs[ts][sel].at(row);
                if (NACC > 1) r1 = args.rs[1][sel].at(row);
            }
            float2 i0 = make_float2(1.0f, 0.0f), i1 = i0;
            if (row_ok) {
                i0 = args.rs[ts][sel].rcp(row);
                if (NACC > 1) i1 = args.rs[1][sel].rcp(row);
            }
            // column reciprocals: this term's scale refs hoisted, chunk i+1's values
            // loaded while chunk i is processed (a global load per chunk otherwise
            // sits on the epilogue's critical path)
            const ScaleRef csr0 = args.cs[ts][sel];
            const ScaleRef csr1 = args.cs[NACC > 1 ? 1 : ts][sel];
            auto col_rcp = [&](int chunk, float2& r0c, float2& r1c) {
                const int cl = min(colbase + chunk * CW + lane, args.N - 1);
                r0c = csr0.rcp(cl);
                if (NACC > 1) r1c = csr1.rcp(cl);
            };
            float2 nrc0 = make_float2(1.0f, 0.0f), nrc1 = nrc0;
            if (nchunk > 0) col_rcp(rev ? nchunk - 1 : 0, nrc0, nrc1);
            mbar_wait(&tfull[buf], bphase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + buf * Cfg::ACC_COLS +
                                   half * (Cfg::BN / 2);
            uint32_t acc2[2][CW];  // EPI_DF: the accumulator columns of a chunk pair
#pragma unroll 1
            for (int i = 0; i < nchunk; ++i) {
                const int c = rev ? nchunk - 1 - i : i;
                const int col0 = colbase + c * CW;
                const int sb = c % NS;
                float* tile = stg0 + sb * (32 * CW);
                const bool resident = i < nres;
                if (Cfg::LOADS_DIN && lane == 0 && i + PD < nchunk && !(rev && i + PD < nres)) {
                    // prefetch the chunk PD ahead into the tile the previous chunk's store read out
                    const int cn = rev ? c - PD : c + PD;
                    if (rev) {  // term 0's store of chunk cn (at most NS+1 newer groups) has landed
                        bulk_wait<NS + 1>();
                        fence_proxy_async();
                    }
                    bulk_wait_read<0>();
                    mbar_expect_tx(&mybar[cn % NS], Cfg::STG_BYTES);
                    tma_load_2d(stg0 + (cn % NS) * (32 * CW), &emaps.din, &mybar[cn % NS], colbase + cn * CW, rowbase);
                }
                // column reciprocals of this chunk, broadcast through shared memory
                scw[lane] = nrc0;
                if (NACC > 1) scw[32 + lane] = nrc1;
                if (i + 1 < nchunk) col_rcp(rev ? c - 1 : c + 1, nrc0, nrc1);
                uint32_t acc[NACC][CW];
                if constexpr (EPI == EPI_DF && NACC == 1) {
                    // two chunks per TMEM round trip (the D_F epilogue is latency-bound at K <= 4096):
                    // the odd chunk's accumulator columns arrived with the even one's
                    if ((i & 1) == 0) {
                        tmem_ld_cols<CW>(tbase + c * CW, acc2[0]);
                        if (i + 1 < nchunk) tmem_ld_cols<CW>(tbase + (c + 1) * CW, acc2[1]);
                        tmem_ld_wait();
                        if (i + 2 >= nchunk) {  // accumulator drained: hand TMEM back to the MMA early
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(tempty_leader0 + buf * 8);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < CW; ++j) acc[0][j] = (i & 1) ? acc2[1][j] : acc2[0][j];
                } else {
#pragma unroll
                for (int a = 0; a < NACC; ++a) tmem_ld_cols<CW>(tbase + a * Cfg::BN + c * CW, acc[a]);
                tmem_ld_wait();
                if (i == nchunk - 1) {  // accumulator drained: hand TMEM back to the MMA early
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader0 + buf * 8);
                }
                }
                if (args.debug & 4) continue;  // probe: TMEM drain only
                if (resident) {  // term-0 result in place: its own store must have read it out
                    if (lane == 0) {
                        if (i == 0) bulk_wait_read<0>();
                        else bulk_wait_read<1>();
                    }
                } else if (Cfg::LOADS_DIN) {
                    mbar_wait(&mybar[sb], (dph >> sb) & 1u);
                    dph ^= 1u << sb;
                } else if (lane == 0) {
                    bulk_wait_read<NS - 1>();  // this chunk's staging tile free again
                }
                __syncwarp();
                float4* rowp = reinterpret_cast<float4*>(tile + lane * CW);
                float res[CW];
                if constexpr (EPI == EPI_DF) {
                    bool slow = false;
                    if (args.debug & 64) {  // probe: no dequant math
#pragma unroll
                        for (int j = 0; j < CW; ++j) res[j] = __int_as_float(acc[0][j]);
                    } else if (args.debug & 128) {  // probe: fp32 math of similar count
#pragma unroll
                        for (int j = 0; j < CW; ++j) res[j] = __fmul_rn(__fmul_rn((float)(int32_t)acc[0][j], i0.x), scw[j].x);
                    } else {
                        uint32_t sm = 0;
#pragma unroll
                        for (int j = 0; j < CW; ++j) res[j] = dq_ff24((int32_t)acc[0][j], i0, scw[j], sm, 1u << j);
                        if (sm) {  // rare: exact redo of the flagged elements
                            const ScaleRef c0 = args.cs[0][sel];
#pragma unroll
                            for (int j = 0; j < CW; ++j)
                                if (sm & (1u << j))
                                    res[j] = dq_slow((int32_t)acc[0][j], i0, scw[j], r0, c0.at(min(col0 + j, args.N - 1)));
                        }
                    }
                    (void)slow;
                } else if constexpr (EPI == EPI_ACC) {
                    // pipeline.cpp:141-145 one term at a time: out = fl(din + deq(acc)).
                    // In place over res[] (register budget: 168/thread); the rare
                    // exact redo re-reads din from the staging tile.
#pragma unroll
                    for (int k = 0; k < KV; ++k) {
                        const float4 d = rowp[k ^ sw];
                        res[4 * k] = d.x; res[4 * k + 1] = d.y; res[4 * k + 2] = d.z; res[4 * k + 3] = d.w;
                    }
                    uint32_t sm = 0;
#pragma unroll
                    for (int j = 0; j < CW; ++j)
                        res[j] = __fadd_rn(res[j], dq_ff24((int32_t)acc[0][j], i0, scw[j], sm, 1u << j));
                    if (sm) {  // rare: exact redo of the flagged elements
                        const ScaleRef c0 = args.cs[ts][sel];
                        const float* rowf = tile + lane * CW;
#pragma unroll
                        for (int j = 0; j < CW; ++j)
                            if (sm & (1u << j))
                                res[j] = __fadd_rn(rowf[(((j >> 2) ^ sw) << 2) | (j & 3)],
                                                   dq_slow((int32_t)acc[0][j], i0, scw[j], r0,
                                                           c0.at(min(col0 + j, args.N - 1))));
                    }
                    if (fin) {  // pipeline.cpp:195-202 (non-fused)
                        const float* cin = args.c_in + (int64_t)row * args.N + col0;
#pragma unroll
                        for (int j = 0; j < CW; ++j) {
                            if (args.has_c) {
                                const float cv = (row_ok && col0 + j < args.N) ? cin[j] : 0.0f;
                                res[j] = __fadd_rn(__fmul_rn(args.alpha, res[j]), __fmul_rn(args.beta, cv));
                            } else if (args.alpha != 1.0f) {
                                res[j] = __fmul_rn(res[j], args.alpha);
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < KV; ++k) {
                        const float4 d = rowp[k ^ sw];
                        res[4 * k] = d.x; res[4 * k + 1] = d.y; res[4 * k + 2] = d.z; res[4 * k + 3] = d.w;
                    }
                    const ScaleRef c0 = args.cs[0][sel], c1 = args.cs[1][sel];
                    const float* cin = args.c_in + (int64_t)row * args.N + col0;
                    float t1[CW], t2[CW];
                    uint32_t sm1 = 0, sm2 = 0;
#pragma unroll
                    for (int j = 0; j < CW; ++j) {
                        t1[j] = dq_ff24((int32_t)acc[0][j], i0, scw[j], sm1, 1u << j);
                        t2[j] = dq_ff24((int32_t)acc[1 % NACC][j], i1, scw[32 + j], sm2, 1u << j);
                    }
                    if (sm1 | sm2) {  // rare: exact redo of the flagged elements
#pragma unroll
                        for (int j = 0; j < CW; ++j) {
                            const int cj = min(col0 + j, args.N - 1);
                            if (sm1 & (1u << j)) t1[j] = dq_slow((int32_t)acc[0][j], i0, scw[j], r0, c0.at(cj));
                            if (sm2 & (1u << j)) t2[j] = dq_slow((int32_t)acc[1 % NACC][j], i1, scw[32 + j], r1, c1.at(cj));
                        }
                    }
#pragma unroll
                    for (int j = 0; j < CW; ++j) {
                        float v = __fadd_rn(__fadd_rn(res[j], t1[j]), t2[j]);  // pipeline.cpp:141-145
                        if (args.has_c) {                                // pipeline.cpp:195-202
                            const float cv = (row_ok && col0 + j < args.N) ? cin[j] : 0.0f;
                            v = __fadd_rn(__fmul_rn(args.alpha, v), __fmul_rn(args.beta, cv));
                        } else if (args.alpha != 1.0f) {
                            v = __fmul_rn(v, args.alpha);
                        }
                        res[j] = v;
                    }
                }
#pragma unroll
                for (int k = 0; k < KV; ++k)
                    rowp[k ^ sw] = make_float4(res[4 * k], res[4 * k + 1], res[4 * k + 2], res[4 * k + 3]);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && !(args.debug & 8)) {  // bit 3 probe: no store
                    tma_store_2d(&emaps.out, tile, col0, rowbase);
                    bulk_commit();
                }
                __syncwarp();
            }
            if (nchunk <= 0) {  // nothing to store (N edge / probe): still release the accumulator
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader0 + buf * 8);
            }
            if (++buf == Cfg::ACC_BUFS) {
                buf = 0;
                bphase ^= 1;
            }
        }
        if (lane == 0) bulk_wait<0>();  // every store landed before exit
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
    }
    if (args.stamp && !skip && threadIdx.x == 128) atomicMax(&args.stamp[1], globaltimer_ns());  // stores landed above
    if (args.done) {
        __syncthreads();  // this CTA's stamp is in
        uint32_t* last = tmem_slot + 1;  // spare word of the barrier area
        if (threadIdx.x == 0) {
            __threadfence();
            *last = atomicAdd(args.done, 1u) == gridDim.x - 1 ? 1u : 0u;
        }
        __syncthreads();
        if (*last) {
            __threadfence();
            for (int i = threadIdx.x; i < args.rep_words; i += blockDim.x)
                if (i != args.rep_flag || args.rep_flag == 0)
                    args.rep_dst[i] = *reinterpret_cast<const volatile uint32_t*>(args.rep_src + i);
            __threadfence_system();
            __syncthreads();
            if (args.rep_dst && args.rep_flag > 0 && threadIdx.x == 0) {  // published last: the host polls it
                *reinterpret_cast<volatile uint32_t*>(args.rep_dst + args.rep_flag) = gridDim.x;
                __threadfence_system();
            }
        }
    }
}

}  // namespace xg
