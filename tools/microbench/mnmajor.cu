// Probe: does tcgen05.mma kind::i8 accept an MN-major (N-contiguous) B operand,
// and with which LBO/SBO?  One CTA, M=128, N=256, K=64 (two K=32 MMAs), A
// K-major SW128, B either K-major (control) or MN-major SW128 with candidate
// strides.  Prints mismatches per variant vs a CPU reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I ../../paper_2403_06924_b200/csrc mnmajor.cu -o mnmajor
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace xg;

constexpr int M = 128, N = 256, K = 64;

__device__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return ((uint64_t)(addr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}

// variant: 0 = B K-major control; 1.. = MN-major with (lbo, sbo) table
__global__ void k(const int8_t* A, const int8_t* B, int32_t* D, int variant, uint32_t lbo, uint32_t sbo) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t* sB = sA + 16384;  // A: 128 rows x 128 B (K padded to 128)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    // A K-major SW128: row m, byte k at m*128 + ((k/16) ^ (m%8))*16 + k%16
    for (int i = tid; i < M * 128; i += blockDim.x) {
        const int m = i / 128, kk = i % 128;
        sA[m * 128 + (((kk >> 4) ^ (m & 7)) << 4) + (kk & 15)] = kk < K ? A[m * K + kk] : 0;
    }
    if (variant == 0) {  // B^T K-major SW128: row n, byte k
        for (int i = tid; i < N * 128; i += blockDim.x) {
            const int n = i / 128, kk = i % 128;
            sB[n * 128 + (((kk >> 4) ^ (n & 7)) << 4) + (kk & 15)] = kk < K ? B[kk * N + n] : 0;
        }
    } else {  // MN-major: two N-atoms of 128 bytes; atom a holds rows k (K x 128 B), swizzled by k%8
        for (int i = tid; i < K * N; i += blockDim.x) {
            const int kk = i / N, n = i % N, a = n / 128, nn = n % 128;
            sB[a * (K * 128) + kk * 128 + (((nn >> 4) ^ (kk & 7)) << 4) + (nn & 15)] = B[kk * N + n];
        }
    }
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (tid < 32) tmem_alloc(&tslot, 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        uint32_t idesc = idesc_i8(M, N);
        if (variant != 0) idesc |= (1u << 16);  // B MN-major
        for (int s = 0; s < K / 32; ++s) {
            const uint64_t da = desc_sw128(smem_u32(sA) + 32 * s, 16, 1024);
            uint64_t db;
            if (variant == 0) db = desc_sw128(smem_u32(sB) + 32 * s, 16, 1024);
            else db = desc_sw128(smem_u32(sB) + 32 * 128 * s, lbo, sbo);
            mma_i8(tmem, da, db, idesc, s ? 1u : 0u);
        }
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int w = tid >> 5, lane = tid & 31;
    if (w < 4) {
        for (int c = 0; c < N / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c * 32, r);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) D[(w * 32 + lane) * N + c * 32 + j] = (int32_t)r[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tmem, 256);
}

int main() {
    std::vector<int8_t> a(M * K), b(K * N);
    srand(1);
    for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
    for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
    std::vector<int32_t> ref(M * N, 0), got(M * N);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int s = 0;
            for (int kk = 0; kk < K; ++kk) s += a[m * K + kk] * b[kk * N + n];
            ref[m * N + n] = s;
        }
    int8_t *da, *db;
    int32_t* dd;
    cudaMalloc(&da, M * K); cudaMalloc(&db, K * N); cudaMalloc(&dd, 4 * M * N);
    cudaMemcpy(da, a.data(), M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), K * N, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    struct V { int v; uint32_t lbo, sbo; } vs[] = {{0, 0, 0}, {1, 1024, 8192}, {1, 8192, 1024}, {1, 16, 1024},
                                                    {1, 1024, 16}, {1, 8192, 16}, {1, 16, 8192}};
    for (auto& v : vs) {
        cudaMemset(dd, 0, 4 * M * N);
        k<<<1, 128, 100000>>>(da, db, dd, v.v, v.lbo, v.sbo);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(got.data(), dd, 4 * M * N, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < M * N; ++i) bad += got[i] != ref[i];
        printf("variant %d lbo %u sbo %u: err=%s mismatches %d / %d\n", v.v, v.lbo, v.sbo, cudaGetErrorString(e), bad, M * N);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
