// Host side of the tcgen05 GEMM: TMA tensor-map encoding and launch.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm.h"
#include "gemm_tc.cuh"

namespace xg {
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D map over a rows x K int8 K-major operand: box {128 bytes, box_rows},
// 128-byte swizzle (matches smem_desc_k128), zero fill out of bounds.
void encode(CUtensorMap* m, const KOperand& op, int K, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)op.rows};
    cuuint64_t strides[1] = {(cuuint64_t)op.ld};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)op.p, dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// fp32 M x N row-major matrix, 32-row boxes of box_cols (32: 128-byte swizzle,
// 16: 64-byte swizzle) - the epilogue staging tiles
void encode_f32_sw128(CUtensorMap* m, const float* p, int rows, int cols, int box_cols = 32) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, 32};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled (f32) failed: " + std::to_string((int)r));
}

constexpr int kDefaultPrefetch = 0;

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = kNumSMs;
    }
    return n;
}

template <int BN, int NACC, int EPI>
void run(const KOperand* ops, const int* is_b, int nops, const GemmArgs& args, cudaStream_t s) {
    using Cfg = GemmCfg<BN, NACC>;
    TmaMaps maps;
    std::memset(&maps, 0, sizeof maps);
    for (int i = 0; i < nops; ++i) encode(&maps.m[i], ops[i], args.K, is_b[i] ? BN : Cfg::BM);
    for (int i = nops; i < kMaxMaps; ++i) maps.m[i] = maps.m[0];
    auto kern = k_gemm_i8_tc<BN, NACC, EPI>;
    // function attributes are per device: set them for every device that runs the kernel
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    const int tiles = ((args.M + Cfg::BM - 1) / Cfg::BM) * ((args.N + BN - 1) / BN);
    const int grid = tiles < sm_count() ? tiles : sm_count();
    kern<<<grid, 256, Cfg::SMEM_BYTES, s>>>(maps, args);
}

template <int NACC, int EPI, int PAIRS, int ST = 0>
void run2(const KOperand* ops, const int* is_b, int nops, const GemmArgs& args, cudaStream_t s) {
    using Cfg = Gemm2Cfg<NACC, EPI, ST>;
    TmaMaps maps;
    std::memset(&maps, 0, sizeof maps);
    for (int i = 0; i < nops; ++i) encode(&maps.m[i], ops[i], args.K, is_b[i] ? 128 / PAIRS : 128);
    for (int i = nops; i < kMaxMaps; ++i) maps.m[i] = maps.m[0];
    auto kern = k_gemm_i8_tc2<NACC, EPI, PAIRS, ST>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    const int csize = 2 * PAIRS;
    const int tiles = ((args.M + 256 * PAIRS - 1) / (256 * PAIRS)) * ((args.N + 255) / 256);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(Cfg::THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent grid: only as many clusters as can be co-resident (4-CTA
    // clusters cannot use every SM), so no cluster waits for a second wave
    // co-resident clusters, queried once per process (all devices are the same part)
    static std::once_flag once;
    static int max_clusters = 0;
    std::call_once(once, [&] {
        cfg.gridDim = dim3(csize * 512);
        if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0) {
            cudaGetLastError();
            max_clusters = sm_count() / csize;
        }
    });
    cfg.gridDim = dim3(csize * (tiles < max_clusters ? tiles : max_clusters));
    static const int env_gm = [] { const char* e = getenv("XG_GEMM_GROUP"); return e ? atoi(e) : 0; }();
    static const int env_pf = [] { const char* e = getenv("XG_GEMM_PF"); return e ? atoi(e) : -1; }();
    static const int env_dbg = [] { const char* e = getenv("XG_GEMM_DEBUG"); return e ? atoi(e) : 0; }();
    GemmArgs a2 = args;
    a2.debug |= env_dbg;
    if (env_gm > 0) a2.group_m = env_gm;  // tuning aid overrides the caller's choice
    if (a2.pf_dist <= 0) a2.pf_dist = env_pf >= 0 ? env_pf : kDefaultPrefetch;
    EpiMaps em;
    std::memset(&em, 0, sizeof em);
    encode_f32_sw128(&em.out, args.out_f32, args.M, args.N, Cfg::CHW);
    encode_f32_sw128(&em.din, (EPI == EPI_COMP || EPI == EPI_ACC) ? args.df_in : args.out_f32, args.M, args.N,
                     Cfg::CHW);
    cudaLaunchKernelEx(&cfg, kern, maps, a2, em);
}

bool use_pair_kernel(const GemmArgs& args) {
    static const int env = [] {
        const char* e = getenv("XG_GEMM_1CTA");
        return e && *e == '1';
    }();
    return !env && args.M >= 256;
}


}  // namespace

bool pair_gemm_used(int M, int N) {
    GemmArgs a{};
    a.M = M;
    a.N = N;
    return use_pair_kernel(a) && (N % 4) == 0;
}

bool make_tmap_f32(void* tmap, const float* p, int rows, int cols, int64_t ld, int box_cols,
                   int box_rows) {
    if ((reinterpret_cast<uintptr_t>(p) & 15) || ((ld * 4) % 16)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return encode_fn()(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims,
                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       // 128-byte promotion: a box row is one 128-byte segment of a row of B;
                       // 256 B fetched the neighbouring strip's half too (select-B DRAM reads
                       // 328 -> 269 MB at C3, reduce stage -4 us)
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void gemm_i8(int epi, const KOperand* ops, const int* is_b, int nops, const GemmArgs& args,
             cudaStream_t s) {
    // the pair kernel's TMA-store epilogue needs 16-byte row pitch for the fp32 maps
    if (use_pair_kernel(args) && (epi == EPI_DF || epi == EPI_COMP || epi == EPI_ACC) && (args.N % 4) == 0) {
        // one pair per cluster: the 4-CTA variant (PAIRS = 2, B^T multicast to two
        // pairs) measured slower on B200 - 33 co-resident clusters, 132 SMs: D_F
        // 306 -> 365 us at C3 (profiles/README.md) - and is not instantiated
        switch (epi) {
            case EPI_DF: run2<1, EPI_DF, 1>(ops, is_b, nops, args, s); return;
            case EPI_COMP: run2<2, EPI_COMP, 1>(ops, is_b, nops, args, s); return;
            case EPI_ACC:  // K <= 4096: the epilogue bounds the tile - deeper D_F prefetch, 5 stages
                if (args.K <= 4096) run2<1, EPI_ACC, 1, 5>(ops, is_b, nops, args, s);
                else run2<1, EPI_ACC, 1>(ops, is_b, nops, args, s);
                return;
        }
    }
    switch (epi) {
        case EPI_S32: run<256, 1, EPI_S32>(ops, is_b, nops, args, s); break;
        case EPI_DF: run<256, 1, EPI_DF>(ops, is_b, nops, args, s); break;
        case EPI_COMP: run<128, 2, EPI_COMP>(ops, is_b, nops, args, s); break;
        case EPI_FULL3: run<128, 3, EPI_FULL3>(ops, is_b, nops, args, s); break;
        case EPI_ACC: throw std::invalid_argument("gemm_i8: EPI_ACC needs the pair kernel");
        default: throw std::invalid_argument("gemm_i8: bad epilogue");
    }
}

}  // namespace xg
