// Throughput microbenchmark of the instruction classes the exact epilogues use
// (DMUL, I2F.F64, F2F.F32.F64, FFMA, SHFL, LDS broadcast) on this B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipes.cu -o pipes
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dmul(double* out, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
        x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a);
        x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, a); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, a);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma(float* out, float a) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
        x0 = fmaf(x0, a, 1.f); x1 = fmaf(x1, a, 1.f); x2 = fmaf(x2, a, 1.f); x3 = fmaf(x3, a, 1.f);
        x4 = fmaf(x4, a, 1.f); x5 = fmaf(x5, a, 1.f); x6 = fmaf(x6, a, 1.f); x7 = fmaf(x7, a, 1.f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_i2f64(double* out, int a) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int v = threadIdx.x;
    for (int i = 0; i < ITERS; ++i) {
        s0 += (double)(v + i); s1 += (double)(v ^ i); s2 += (double)(v - i); s3 += (double)(v * a + i);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_f2f(float* out, double a) {
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    double v = threadIdx.x * a;
    for (int i = 0; i < ITERS; ++i) {
        s0 += __double2float_rn(v + i); s1 += __double2float_rn(v - i); s2 += __double2float_rn(v * 0.5 + i);
        s3 += __double2float_rn(v * 0.25 + i);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_i2f32(float* out, int a) {
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int v = threadIdx.x;
    for (int i = 0; i < ITERS; ++i) {
        s0 += (float)(v + i); s1 += (float)(v ^ i); s2 += (float)(v - i); s3 += (float)(v * a + i);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

template <class F>
float timeit(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    f();
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    double* dd; float* fd;
    cudaMalloc(&dd, sizeof(double) * blocks * threads);
    cudaMalloc(&fd, sizeof(float) * blocks * threads);
    const double n = (double)blocks * threads * ITERS;
    float ms;
    ms = timeit([&] { k_ffma<<<blocks, threads>>>(fd, 1.0001f); });
    printf("FFMA     %.2f Tops/s  (%.1f /clk/SM @1.965GHz)\n", 8 * n / ms / 1e9, 8 * n / ms / 1e-3 / sms / 1.965e9);
    ms = timeit([&] { k_dmul<<<blocks, threads>>>(dd, 1.0001); });
    printf("DMUL     %.2f Tops/s  (%.1f /clk/SM)\n", 8 * n / ms / 1e9, 8 * n / ms / 1e-3 / sms / 1.965e9);
    ms = timeit([&] { k_i2f64<<<blocks, threads>>>(dd, 3); });
    printf("I2F.F64+DADD %.2f Tops/s (%.1f pairs/clk/SM)\n", 4 * n / ms / 1e9, 4 * n / ms / 1e-3 / sms / 1.965e9);
    ms = timeit([&] { k_f2f<<<blocks, threads>>>(fd, 0.37); });
    printf("F2F.F32.F64+DADD+FADD %.2f Tops/s (%.1f /clk/SM)\n", 4 * n / ms / 1e9, 4 * n / ms / 1e-3 / sms / 1.965e9);
    ms = timeit([&] { k_i2f32<<<blocks, threads>>>(fd, 3); });
    printf("I2F.F32+FADD %.2f Tops/s (%.1f /clk/SM)\n", 4 * n / ms / 1e9, 4 * n / ms / 1e-3 / sms / 1.965e9);
    return 0;
}
