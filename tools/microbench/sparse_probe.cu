// Probe: tcgen05.mma.sp kind::i8 metadata layout and throughput on B200.
// Layout: A compressed (128 rows x 32 bytes = K 64 logical), byte j of every
// row = j+1; B (K=64 x N=64) = identity so D[m][n] = A_logical[m][n].  Each
// experiment writes a metadata pattern into TMEM, runs one sparse MMA and dumps
// D (128x64 int32) to out[exp].  Throughput: 4096 back-to-back dense
// (M128 N256 K32) vs sparse (M128 N256 K64) MMAs per CTA on 148 CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I ../../paper_2403_06924_b200/csrc sparse_probe.cu -o sparse_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace xg;

__device__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return ((uint64_t)(addr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t meta, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                 "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(meta), "r"(idesc), "r"(acc)
                 : "memory");
}

// pattern(exp, lane, col) -> metadata word
__device__ uint32_t pattern(int e, int lane, int col) {
    const uint32_t base = 0x44444444u;
    switch (e) {
        case 0: return base;
        case 1: return 0xEEEEEEEEu;
        case 2: return (lane == 0 && col == 0) ? 0xEEEEEEEEu : base;
        case 3: return (lane == 0 && col == 1) ? 0xEEEEEEEEu : base;
        case 4: return (lane == 1 && col == 0) ? 0xEEEEEEEEu : base;
        case 5: return (lane == 0 && col == 0) ? 0x4444444Eu : base;
        case 6: return (lane == 0 && col == 0) ? 0x444444E4u : base;
        case 7: return (lane == 0 && col == 0) ? 0xE4444444u : base;
        case 8: return (lane == 64 && col == 0) ? 0xEEEEEEEEu : base;
        case 9: return (lane == 32 && col == 0) ? 0xEEEEEEEEu : base;
        case 10: return (lane == 0 && col == 2) ? 0xEEEEEEEEu : base;
        case 11: return (lane == 0 && col == 3) ? 0xEEEEEEEEu : base;
        case 12: return (lane == 2 && col == 0) ? 0xEEEEEEEEu : base;
        case 13: return (lane == 16 && col == 0) ? 0xEEEEEEEEu : base;
        default: return 0x88888888u;  // (0,2)
    }
}
constexpr int NEXP = 15;

__global__ void k_layout(int8_t* gA, int8_t* gB, int32_t* out, int sel_bits) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t* sB = sA + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 128; i += blockDim.x) {  // A compressed, K-major SW128, 32 used bytes
        const int m = i / 128, kk = i % 128;
        sA[m * 128 + (((kk >> 4) ^ (m & 7)) << 4) + (kk & 15)] = kk < 32 ? (int8_t)(kk + 1) : 0;
    }
    for (int i = tid; i < 64 * 128; i += blockDim.x) {  // B^T (N=64 rows, K-major): identity on k < 64
        const int n = i / 128, kk = i % 128;
        sB[n * 128 + (((kk >> 4) ^ (n & 7)) << 4) + (kk & 15)] = (kk == n) ? 1 : 0;
    }
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (w == 0) tmem_alloc(&tslot, 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t meta = tmem + 128;  // metadata columns 128..
    uint32_t idesc = idesc_i8(128, 64) | (1u << 2) | (uint32_t)(sel_bits & 3);
    for (int e = 0; e < NEXP; ++e) {
        for (int c = 0; c < 8; ++c) tmem_st1(meta + ((uint32_t)(w * 32) << 16) + c, pattern(e, w * 32 + lane, c));
        tmem_st_wait();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (tid == 0) {
            mma_sp(tmem, desc_sw128(smem_u32(sA), 16, 1024), desc_sw128(smem_u32(sB), 16, 1024), meta, idesc, 0);
            tc_commit(&bar);
        }
        mbar_wait(&bar, e & 1);
        tc_fence_after();
        for (int c = 0; c < 2; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c * 32, r);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) out[((size_t)e * 128 + w * 32 + lane) * 64 + c * 32 + j] = (int32_t)r[j];
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    if (w == 0) tmem_dealloc(tmem, 256);
}

// throughput: ITER MMAs on garbage smem (values irrelevant), N=256
__global__ void k_tput(int sparse, int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s0 = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (w == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    for (int c = 0; c < 16; ++c) tmem_st1(tmem + 256 + ((uint32_t)(w * 32) << 16) + c, 0x44444444u);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t da = desc_sw128(smem_u32(s0), 16, 1024), db = desc_sw128(smem_u32(s0 + 65536), 16, 1024);
        const long long t0 = clock64();
        if (sparse) {
            const uint32_t idesc = idesc_i8(128, 256) | (1u << 2);
            for (int i = 0; i < iters; ++i) mma_sp(tmem, da + 2 * (i & 3), db + 4 * (i & 1), tmem + 256, idesc, 1);
        } else {
            const uint32_t idesc = idesc_i8(128, 256);
            for (int i = 0; i < iters; ++i) mma_i8(tmem, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc(tmem, 512);
}

int main() {
    int32_t* dout;
    cudaMalloc(&dout, sizeof(int32_t) * NEXP * 128 * 64);
    cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    std::vector<int32_t> h(NEXP * 128 * 64);
    for (int selb = 0; selb < 1; ++selb) {
        cudaMemset(dout, 0xff, sizeof(int32_t) * NEXP * 128 * 64);
        k_layout<<<1, 128, 40000>>>(nullptr, nullptr, dout, selb);
        cudaError_t e = cudaDeviceSynchronize();
        printf("layout sel=%d: %s\n", selb, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost);
        char fn[64];
        snprintf(fn, sizeof fn, "gpurun_out/sparse_layout_sel%d.bin", selb);
        FILE* f = fopen(fn, "wb");
        fwrite(h.data(), 4, h.size(), f);
        fclose(f);
        // print row 0, 1, 32, 64 of exp 0 and 1
        for (int ex = 0; ex < 2; ++ex)
            for (int m : {0, 1}) {
                printf("exp%d row%d:", ex, m);
                for (int n = 0; n < 64; ++n) printf(" %d", h[((size_t)ex * 128 + m) * 64 + n]);
                printf("\n");
            }
    }
    long long* dc;
    cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(k_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    for (int sp = 0; sp < 2; ++sp) {
        k_tput<<<148, 128, 140000>>>(sp, 4096, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> c(148);
        cudaMemcpy(c.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (auto x : c) avg += x;
        avg /= 148;
        const double macs = 128.0 * 256 * (sp ? 64 : 32) * 4096;
        printf("%s: %s, %.0f cycles for 4096 MMAs -> %.1f cycles/MMA, %.0f MAC/clk/SM\n", sp ? "sparse K64" : "dense K32",
               cudaGetErrorString(e), avg, avg / 4096, macs / avg);
    }
    return 0;
}
