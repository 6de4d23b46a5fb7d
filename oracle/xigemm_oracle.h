/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the compensated INT8 GEMM path.
 *
 * A plain-C restatement of the reference algorithm (arXiv 2403.06924,
 * /root/reference/proj/src/{quantize,sparse,pipeline,matrix}.cpp).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker / CPU baseline.  The product
 * (paper_2403_06924_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against
 *   (a) the reference compiled from its own sources into oracle/_ref
 *       (oracle/Makefile, -Dxigemm=xigemm_ref), when that build exists, and
 *   (b) the committed golden vectors in tests/golden/ that were generated
 *       from oracle/_ref by tests/golden/make_golden.py, plus the reference
 *       test-suite known answers (test_quant.cpp, test_sparse.cpp, ...).
 *
 * Enum encodings mirror the reference enum declaration order:
 *   RoundingMode    Floor=0 Nearest=1          (quantize.hpp:18)
 *   ScaleScheme     PerTensor=0 PerRow=1 PerColumn=2 (quantize.hpp:20)
 *   QuantScheme     PerTensor=0 VectorWise=1   (pipeline.hpp:15)
 *   ReductionPolicy AvgRule=0 MinRule=1        (sparse.hpp:40)
 *   GemmPath        SparseResidual=0 DenseResidual=1 (pipeline.hpp:30)
 * Every function returns 0 on success and 1 where the reference throws
 * std::invalid_argument.
 */
#ifndef XIGEMM_ORACLE_H
#define XIGEMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int bits;             /* 4 or 8 */
    double threshold;     /* M */
    double density_limit; /* s */
    int scheme;           /* QuantScheme */
    int policy;           /* ReductionPolicy */
    int rounding;         /* RoundingMode */
} xo_config;

typedef struct {
    double density_a, density_b;
    int path;
    int64_t nnz_a, nnz_b;
} xo_report;

/* Optional intermediates of run_residual_pipeline (pipeline.cpp:44-149).
 * Any pointer may be NULL.  Layouts are the reference's row-major ones. */
typedef struct {
    int8_t *aq; double *aq_scales;      /* M*K, M|1 */
    int8_t *bq; double *bq_scales;      /* K*N, N|1 */
    int32_t *d_int; float *d_f;         /* M*N */
    int8_t *raq; double *raq_scale;     /* M*K, 1 */
    int8_t *rbq; double *rbq_scale;     /* K*N, 1 */
    float *row_stat; float *col_stat;   /* M, N */
    uint8_t *a_mask; uint8_t *b_mask;   /* M*K, K*N : retained entries */
    int8_t *a_red; double *a_red_scales;/* M*K dense form of the quantized CSR, M|1 */
    int8_t *b_red; double *b_red_scales;/* K*N, N|1 */
    int32_t *dr1; int32_t *dr2;         /* M*N */
} xo_dump;

int xo_version(void);

uint64_t xo_splitmix_next(uint64_t *state);
double xo_splitmix_unit(uint64_t *state);
/* random_matrix.cpp:105-116; kind: 0 uniform01 1 normal 2 exponential 3 poisson 4 chi-square */
int xo_generate(int kind, double p1, double p2, uint64_t seed, int rows, int cols, float *out);
/* test_support.hpp:16-24 */
void xo_random_dense(int rows, int cols, uint64_t seed, float lo, float hi, float *out);

int xo_quant_max(int bits);
int xo_gemm_int_max_inner(int bits);
int xo_compute_scale(double max_abs, int bits, double *out);
int32_t xo_quantize_scalar(double a, double lambda, int32_t qmax, int rounding);
float xo_max_abs(const float *a, int64_t n);
int xo_all_finite(const float *a, int64_t n);

int xo_quantize(const float *a, int rows, int cols, int bits, int scheme, int rounding,
                int8_t *q, double *scales);
int xo_quantize_with_scales(const float *a, int rows, int cols, int bits, int scheme,
                            const double *scales, int rounding, int8_t *q);
int xo_dequantize(const int8_t *q, int rows, int cols, int scheme, const double *scales,
                  float *out);
int xo_residual(const float *a, const int8_t *q, int rows, int cols, int scheme,
                const double *scales, float *out);
int xo_dequant_product(const int32_t *p, int rows, int cols, int scheme_a, const double *sa,
                       int scheme_b, const double *sb, float *out);
int xo_gemm_int(const int8_t *a, const int8_t *b, int m, int k, int n, int bits_a, int bits_b,
                int32_t *c);
int xo_gemm_f32(const float *a, const float *b, int m, int k, int n, float *c);
int xo_axpby(float *d, float alpha, const float *c, float beta, int64_t n);

int xo_avg_vectors(const float *d, int rows, int cols, float *row, float *col);
int xo_abs_min_vectors(const float *d, int rows, int cols, float *row, float *col);

/* reduce_a (per_row=1) / reduce_b (per_row=0), sparse.cpp:36-85.  row_ptr has
 * rows+1 entries; col_idx/values need capacity rows*cols. */
int xo_reduce(const float *m, int rows, int cols, const float *stat, double thr_m, int policy,
              double scale_other, int per_row, int32_t *row_ptr, int32_t *col_idx,
              float *values, int64_t *nnz);
int xo_quantize_csr(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                    const float *values, int bits, int scheme, int rounding, int8_t *qvals,
                    double *scales);
int xo_csr_transpose_i8(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                        const int8_t *values, int32_t *t_row_ptr, int32_t *t_col_idx,
                        int8_t *t_values);
int xo_spmm_int(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                const int8_t *values, const int8_t *d, int d_cols, int d_bits, int32_t *out);
int xo_spmm_f32(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                const float *values, const float *d, int d_cols, float *out);

/* pipeline.cpp:44-213.  reduce=1: xigemm; reduce=0: quantized_gemm_full_residual. */
int xo_xigemm(const float *a, const float *b, const float *c, float alpha, float beta, int m,
              int k, int n, const xo_config *cfg, int reduce, float *out, xo_report *rep,
              xo_dump *dump);
int xo_gemm_direct(const float *a, const float *b, int m, int k, int n, const xo_config *cfg,
                   float *out);

#ifdef __cplusplus
}
#endif
#endif
