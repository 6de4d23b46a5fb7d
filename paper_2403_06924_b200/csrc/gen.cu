// Synthetic operand generator on the device (bench / test inputs only).
//
// The reference's generator is one sequential SplitMix64 stream
// (random_matrix.cpp:9-18, :105-116).  Every distribution used here consumes a
// fixed number of draws per element, so element i can jump straight to its
// stream position: state_i = seed + (draws*i + t) * golden.  Uniform values are
// bit-identical to the reference's (pure integer + fp32 arithmetic); normal and
// Student-t values go through the device log/cos and may differ from glibc in
// the last ulp, which is irrelevant for synthetic data.
#include <cstdint>

#include "common.cuh"

namespace xg {
namespace {

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double unit_at(uint64_t seed, uint64_t pos) {
    // pos-th draw (1-based) of the stream seeded with `seed`
    return (double)(mix(seed + pos * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t pos) {
    const double u1 = 1.0 - unit_at(seed, pos);
    const double u2 = unit_at(seed, pos + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

// kind 0: test_support uniform lo + float(u)*(hi-lo)   (1 draw)
// kind 1: normal(p1, p2)                                (2 draws)
// kind 2: Student-t(3) scaled by p2: z / sqrt((z1^2+z2^2+z3^2)/3)  (8 draws)
// kind 3: exponential(p1)                               (1 draw)
__global__ void k_generate(int kind, double p1, double p2, uint64_t seed, int64_t n, float* out) {
    XG_PDL_WAIT();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float v;
        if (kind == 0) {
            const float lo = (float)p1, hi = (float)p2;
            v = __fadd_rn(lo, __fmul_rn((float)unit_at(seed, (uint64_t)i + 1), __fsub_rn(hi, lo)));
        } else if (kind == 1) {
            v = (float)(p1 + p2 * normal_at(seed, 2 * (uint64_t)i + 1));
        } else if (kind == 2) {
            const uint64_t b = 8 * (uint64_t)i + 1;
            const double z = normal_at(seed, b);
            const double z1 = normal_at(seed, b + 2), z2 = normal_at(seed, b + 4),
                         z3 = normal_at(seed, b + 6);
            v = (float)(p2 * z / sqrt((z1 * z1 + z2 * z2 + z3 * z3) / 3.0));
        } else {
            v = (float)(-log(1.0 - unit_at(seed, (uint64_t)i + 1)) / p1);
        }
        out[i] = v;
    }
}

}  // namespace
}  // namespace xg

extern "C" int xg_generate(int kind, double p1, double p2, uint64_t seed, int64_t n, float* out,
                           void* stream) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    xg::k_generate<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(kind, p1, p2, seed, n, out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
