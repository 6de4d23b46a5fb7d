// Development probes (not part of the reference API; bound by bench.py only):
// the SIMT integer multiply-accumulate rate that the 3-term roofline of SURVEY
// section 8(d) charges the SpMM work against, measured on the box.
//   kind 0: IDP4A (4 int8 MACs per instruction)   kind 1: IMAD (1 MAC)
#include <cuda_runtime.h>

#include <cstdint>

namespace {

template <int KIND>
__global__ void __launch_bounds__(256) k_simt_rate(int iters, uint32_t seed, int* sink) {
    // 8 independent accumulators per thread: issue-bound, not latency-bound
    int acc[8];
    uint32_t x = seed ^ (threadIdx.x * 2654435761u), y = x * 747796405u + 1u;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = (int)(x + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0) acc[j] = __dp4a((int)x, (int)y, acc[j]);
            else acc[j] = acc[j] * (int)x + (int)y;
        }
        x += 0x01010101u;  // keep the operands live (the loop is not folded)
    }
    int s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s ^= acc[j];
    if (s == 0x7fffffff) *sink = s;
}

}  // namespace

extern "C" double xg_debug_simt_rate(int kind, int iters) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int* sink = nullptr;
    if (cudaMalloc(&sink, sizeof(int)) != cudaSuccess) return -1.0;
    const int blocks = sms * 8, threads = 256;
    auto launch = [&](int it) {
        if (kind == 0) k_simt_rate<0><<<blocks, threads>>>(it, 1234u, sink);
        else k_simt_rate<1><<<blocks, threads>>>(it, 1234u, sink);
    };
    launch(64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (cudaGetLastError() != cudaSuccess || ms <= 0) return -1.0;
    const double macs = (double)blocks * threads * iters * 8 * (kind == 0 ? 4 : 1);
    return macs / (ms * 1e-3);
}
