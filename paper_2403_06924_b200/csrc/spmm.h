// CUDA-core sparse compensation path (spmm.cu): quad-packed CSR build and the
// strip SpMM with the compensation epilogues.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace xg {

// Quad-packed rows of a sparse int8 operand: row r owns quads
// [seg[r].x, seg[r].x + seg[r].y).  A quad is one 16-byte record of 4 entries:
// bytes 0-7 the uint16 columns, bytes 8-11 the int8 values (padding entries
// have value 0), bytes 12-15 unused - one 16-byte load per quad.
struct QCsr {
    int2* seg;
    uint4* quad;
    unsigned long long* cursor;  // quads handed out (zeroed before the build)
    int64_t cap_q;               // capacity in quads
};

// per-tensor (stride 0) or per-row (stride 1) fp64 scales + optional float-float reciprocals
struct SpScale {
    const double* p;
    int stride;
    const float2* r;
};

enum SpmmMode : int {
    kSpmmS32 = 0,   // out_s32[r * ldo + l] = acc                          (spmm_int)
    kSpmmRows = 1,  // out[r * ldo + l] = fl(din[r * ldo + l] + deq(acc))  (dr1: r = row i, l = column j)
    kSpmmColsT = 2  // out[l * ldo + r] = fl(out[l * ldo + r] + deq(acc)), alpha/beta (dr2: r = column j, l = row i)
};

struct SpmmArgs {
    // sparse operand: nsp quad-packed rows over K
    const int2* seg;
    const uint4* quad;
    int nsp, K;
    // dense operand: nlines lines of K int8 (K-major, pitch ldd), or K x nlines row-major
    const int8_t* dense;
    int64_t ldd;
    int nlines;
    int src_rowmajor;
    int mode;
    int32_t* out_s32;
    float* out;
    const float* din;
    int64_t ldo;
    SpScale sp_scale, line_scale;  // dequantisation scales of the sparse row / dense line
    const float* c_in;
    int has_c;
    float alpha, beta;
    const int* run;    // device flag: run only when *run != 0 (null: always)
    const int* bad;    // device flag: the build overflowed -> do nothing (null: never)
    unsigned long long* stamp;      // %globaltimer at start (null: off)
    unsigned long long* stamp_end;  // atomicMax of %globaltimer at exit (null: off)
};

constexpr int kSpmmSmemMax = 128 * 1024;

// strip width for inner dimension K (16 or 8 lines), 0 if K is too large for the CUDA-core path
int spmm_strip_width(int K);
void launch_qcsr_build(const int8_t* x, int rows, int cols, int64_t ld, const QCsr& q, const int* run, int* bad,
                       int max_quads, cudaStream_t s);
void launch_qcsr_from_csr(const int32_t* rp, const int32_t* ci, const int8_t* v, int rows, const QCsr& q,
                          cudaStream_t s);
bool launch_spmm_strip(const SpmmArgs& a, cudaStream_t s);
void launch_random_masked_i8(int8_t* x, int rows, int cols, int64_t ld, double density, int qmax, uint64_t seed,
                             cudaStream_t s);

}  // namespace xg
