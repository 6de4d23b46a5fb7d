// Probe: packed fp32x2 ops (mul/fma/add/sub .rn.f32x2) against the scalar IEEE
// ops lane by lane on random operands incl. tiny/huge magnitudes and zeros.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 f32x2_check.cu -o f32x2_check
#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ void upk(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ float rnd(uint32_t& s) { s = s * 1664525u + 1013904223u; uint32_t e = (s >> 24) % 200 + 27; uint32_t m = (s * 2654435761u) & 0x7fffff; uint32_t sg = (s >> 7) & 1; return __uint_as_float((sg << 31) | (e << 23) | m); }
__global__ void k(int* bad, float* ex) {
    uint32_t s = blockIdx.x * 977u + threadIdx.x * 131u + 7u;
    for (int it = 0; it < 2000; ++it) {
        float a0 = rnd(s), a1 = rnd(s), b0 = rnd(s), b1 = rnd(s), c0 = rnd(s), c1 = rnd(s);
        if ((s & 15) == 0) c0 = 0.0f;
        uint64_t A = pk(a0, a1), B = pk(b0, b1), C = pk(c0, c1), R;
        float r0, r1;
        for (int op = 0; op < 4; ++op) {
            float e0, e1;
            if (op == 0) { asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B)); e0 = __fmul_rn(a0, b0); e1 = __fmul_rn(a1, b1); }
            else if (op == 1) { asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(R) : "l"(A), "l"(B), "l"(C)); e0 = __fmaf_rn(a0, b0, c0); e1 = __fmaf_rn(a1, b1, c1); }
            else if (op == 2) { asm("add.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B)); e0 = __fadd_rn(a0, b0); e1 = __fadd_rn(a1, b1); }
            else { asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B)); e0 = __fsub_rn(a0, b0); e1 = __fsub_rn(a1, b1); }
            upk(R, r0, r1);
            if (__float_as_uint(r0) != __float_as_uint(e0) || __float_as_uint(r1) != __float_as_uint(e1)) {
                int i = atomicAdd(&bad[op], 1);
                if (i < 4) { float* x = ex + (op * 4 + i) * 10; x[0]=a0;x[1]=a1;x[2]=b0;x[3]=b1;x[4]=c0;x[5]=c1;x[6]=r0;x[7]=r1;x[8]=e0;x[9]=e1; }
            }
        }
    }
}
int main() {
    int* bad; float* ex; cudaMalloc(&bad, 16); cudaMalloc(&ex, 4 * 4 * 10 * 4); cudaMemset(bad, 0, 16);
    k<<<148, 256>>>(bad, ex); cudaDeviceSynchronize();
    int hb[4]; float he[160]; cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost); cudaMemcpy(he, ex, sizeof he, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"mul", "fma", "add", "sub"};
    for (int op = 0; op < 4; ++op) {
        printf("%s: %d mismatches of %d\n", nm[op], hb[op], 148 * 256 * 2000);
        for (int i = 0; i < (hb[op] < 4 ? hb[op] : 4); ++i) { float* x = he + (op * 4 + i) * 10; printf("  a=(%g,%g) b=(%g,%g) c=(%g,%g) got=(%.9g,%.9g) want=(%.9g,%.9g)\n", x[0],x[1],x[2],x[3],x[4],x[5],x[6],x[7],x[8],x[9]); }
    }
    return 0;
}
