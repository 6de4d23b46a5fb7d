// Launch wrappers of misc.cu (API-surface kernels).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace xg {

void transpose_i8(const int8_t* src, int rows, int cols, int64_t lds, int8_t* dst, int64_t ldd,
                  cudaStream_t s);
void quantize_with_scales(const float* a, int rows, int cols, int bits, int scheme,
                          const double* scales, int rounding, int8_t* q, cudaStream_t s);
// out = minuend ? minuend - deq : deq
void dequantize(const int8_t* q, int rows, int cols, int scheme, const double* scales,
                const float* minuend, float* out, cudaStream_t s);
void dequant_product(const int32_t* p, int rows, int cols, int sa_scheme, const double* sa,
                     int sb_scheme, const double* sb, float* out, cudaStream_t s);
void gemm_f32_exact(const float* a, const float* b, int m, int k, int n, float* c, cudaStream_t s);
void axpby(float* d, float alpha, const float* c, float beta, int64_t n, cudaStream_t s);
void subtract(const float* a, const float* b, float* o, int64_t n, cudaStream_t s);
void add_inplace(float* d, const float* x, int64_t n, cudaStream_t s);
void finite_max(const float* x, int64_t n, uint32_t* mx, int* bad, cudaStream_t s);

// mode 0: threshold reduction (reduce_a / reduce_b); mode 1: csr_from_dense
cudaError_t csr_count(int mode, const float* m, int rows, int cols, const float* stat, double thr_m,
                      int policy, double so, int per_row, int32_t* row_ptr, int32_t* cnt,
                      cudaStream_t s);
void csr_fill(int mode, const float* m, int rows, int cols, const float* stat, double thr_m,
              int policy, double so, int per_row, const int32_t* row_ptr, int32_t* col_idx,
              float* values, cudaStream_t s);
void csr_quantize(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v,
                  int64_t nnz, int bits, int scheme, int rounding, int8_t* q, double* scales,
                  uint32_t* scratch, cudaStream_t s);
template <class T>
cudaError_t csr_transpose(int rows, int cols, const int32_t* rp, const int32_t* ci, const T* v,
                          int64_t nnz, int32_t* trp, int32_t* tci, T* tv, cudaStream_t s);
void spmm_i8(int rows, const int32_t* rp, const int32_t* ci, const int8_t* v, const int8_t* d,
             int d_cols, int32_t* out, cudaStream_t s);
void spmm_f32(int rows, const int32_t* rp, const int32_t* ci, const float* v, const float* d,
              int d_cols, float* out, cudaStream_t s);
void random_i8(int8_t* p, int64_t n, uint64_t seed, cudaStream_t s);  // uniform in [-127, 127]
void densify(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v, float* out,
             cudaStream_t s);

}  // namespace xg
