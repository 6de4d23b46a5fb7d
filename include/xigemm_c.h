/*
 * xigemm_c.h — C-ABI of the B200-native compensated INT8 GEMM
 * (arXiv 2403.06924, "xigemm").  Plain pointers, sizes and POD enums only.
 *
 * Two kinds of entry points:
 *   xg_*      device-pointer, stream-ordered functions (inputs and outputs in
 *             HBM).  They replace the reference's functions one for one; each
 *             declaration cites the reference interface it replaces.
 *   xg_*_host the same operation on HOST buffers (H2D, compute, D2H inside the
 *             call) — what the C++ drop-in (include/xigemm/*.hpp) binds.
 *
 * Matrices are row-major with the reference's shapes (matrix.hpp:11-46).
 * Enums follow the reference's declaration order:
 *   bits: 4 | 8 (QuantBits, quantize.hpp:12)
 *   rounding: XG_FLOOR=0, XG_NEAREST=1            (RoundingMode, quantize.hpp:18)
 *   scale scheme: XG_PER_TENSOR=0, XG_PER_ROW=1, XG_PER_COLUMN=2 (quantize.hpp:20)
 *   quant scheme: XG_Q_PER_TENSOR=0, XG_Q_VECTORWISE=1 (pipeline.hpp:15)
 *   policy: XG_AVG_RULE=0, XG_MIN_RULE=1           (sparse.hpp:40)
 *   path: XG_SPARSE_RESIDUAL=0, XG_DENSE_RESIDUAL=1 (pipeline.hpp:30)
 * Every function returns an xg_status; XG_EINVAL is exactly where the
 * reference throws std::invalid_argument, and xg_last_error() (thread-local)
 * carries the message.
 */
#ifndef XIGEMM_C_H
#define XIGEMM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *xg_stream; /* cudaStream_t */

typedef enum {
    XG_OK = 0,
    XG_EINVAL = 1,   /* std::invalid_argument in the reference */
    XG_ECUDA = 2,    /* CUDA runtime / launch failure (no reference equivalent) */
    XG_ENOMEM = 3,
    XG_EINTERNAL = 4,
    XG_EAGAIN = 5    /* row-sharded only: rerun with a larger exchange buffer (xg_shard_finish) */
} xg_status;

enum { XG_FLOOR = 0, XG_NEAREST = 1 };
enum { XG_PER_TENSOR = 0, XG_PER_ROW = 1, XG_PER_COLUMN = 2 };
enum { XG_Q_PER_TENSOR = 0, XG_Q_VECTORWISE = 1 };
enum { XG_AVG_RULE = 0, XG_MIN_RULE = 1 };
enum { XG_SPARSE_RESIDUAL = 0, XG_DENSE_RESIDUAL = 1 };

/* XigemmConfig, pipeline.hpp:19-28 (same defaults via xg_config_default). */
typedef struct {
    int bits;
    double threshold;
    double density_limit;
    int scheme;
    int policy;
    int rounding;
} xg_config;

/* GemmReport minus the result matrix, pipeline.hpp:32-39.  Stage times are
 * device (CUDA event) times in ns under the reference's four keys. */
typedef struct {
    double density_a, density_b;
    int path;
    int64_t nnz_a, nnz_b;
    double ns_quant, ns_xxmm, ns_reduce, ns_package;
    int stats_fallbacks; /* AvgRule statistics recomputed in exact order */
    double ns_gemm_df;   /* device time of the D_F GEMM launch (K2) */
    double ns_gemm_comp; /* device time of the compensation GEMM launch (K4+K5) */
    int comp_kernel;     /* the sparse terms ran on: 0 tcgen05 masked-dense launch,
                            1 CUDA-core quad-packed CSR SpMM (same result, bit for bit) */
} xg_report;

/* Device pointers (reference row-major layouts) receiving pipeline
 * intermediates; any may be NULL.  Used by the stage-wise parity tests. */
typedef struct {
    int8_t *aq; double *aq_scales;   /* M*K ; M|1 */
    int8_t *bq; double *bq_scales;   /* K*N ; N|1 */
    float *d_f;                      /* M*N */
    int8_t *raq; double *raq_scale;  /* M*K ; 1 */
    int8_t *rbq; double *rbq_scale;  /* K*N ; 1 */
    float *row_stat; float *col_stat;/* M ; N */
    int8_t *a_red; int8_t *b_red;    /* M*K ; K*N (quantized reduced operands, dense form) */
    double *a_red_scale; double *b_red_scale; /* per-tensor scale of the reduced operands */
    /* kept-element index sets of reduce_a / reduce_b (sparse.cpp:36-85) as written
     * by the selection kernels: bit (k % 32) of word [i * ceil(K/32) + k / 32] of
     * a_keep is set iff a[i][k] is retained; b_keep likewise for b[k][j] at word
     * [j * ceil(K/32) + k / 32] (one row per column of B).  Zeroed by the call. */
    uint32_t *a_keep; uint32_t *b_keep;  /* M*ceil(K/32) ; N*ceil(K/32) */
} xg_dump;

const char *xg_last_error(void);
int xg_version(void);
xg_config xg_config_default(void);
/* 1 if a usable sm_100 device is present and the kernels load. */
int xg_device_ok(void);
/* Frees the cached per-device workspace. */
xg_status xg_workspace_release(void);
/* Number of this library's kernels launched on the calling thread since the
 * last reset (a claim the bench reports as gpu_launches). */
int64_t xg_launch_count(int reset);

/* ---- quantize.hpp -------------------------------------------------------- */
/* quantize() quantize.hpp:80 / quantize.cpp:107-133.  scales: 1|rows|cols. */
xg_status xg_quantize(const float *a, int rows, int cols, int bits, int scheme, int rounding,
                      int8_t *q, double *scales, xg_stream s);
/* quantize_with_scales() quantize.hpp:84 / quantize.cpp:135-150 */
xg_status xg_quantize_with_scales(const float *a, int rows, int cols, int bits, int scheme,
                                  const double *scales, int rounding, int8_t *q, xg_stream s);
/* dequantize() quantize.hpp:87 / quantize.cpp:152-160 */
xg_status xg_dequantize(const int8_t *q, int rows, int cols, int scheme, const double *scales,
                        float *out, xg_stream s);
/* residual() quantize.hpp:91 / quantize.cpp:162-167 */
xg_status xg_residual(const float *a, const int8_t *q, int rows, int cols, int scheme,
                      const double *scales, float *out, xg_stream s);
/* dequant_product() quantize.hpp:95 / quantize.cpp:169-187 */
xg_status xg_dequant_product(const int32_t *p, int rows, int cols, int scheme_a,
                             const double *sa, int scheme_b, const double *sb, float *out,
                             xg_stream s);
/* gemm_int() quantize.hpp:100 / quantize.cpp:193-214 (tcgen05 kind::i8) */
xg_status xg_gemm_i8(const int8_t *a, const int8_t *b, int m, int k, int n, int bits_a,
                     int bits_b, int32_t *c, xg_stream s);
/* gemm_int_max_inner() quantize.hpp:103 */
int xg_gemm_max_inner(int bits);

/* ---- matrix.hpp ---------------------------------------------------------- */
/* gemm_f32() matrix.hpp:50 / matrix.cpp:75-95 (fp64 accumulation, ascending k) */
xg_status xg_gemm_f32(const float *a, const float *b, int m, int k, int n, float *c, xg_stream s);
/* axpby_inplace() matrix.hpp:53 / matrix.cpp:97-105 */
xg_status xg_axpby(float *d, float alpha, const float *c, float beta, int64_t n, xg_stream s);
/* subtract() / add_inplace() matrix.hpp:55-56 */
xg_status xg_subtract(const float *a, const float *b, float *out, int64_t n, xg_stream s);
xg_status xg_add_inplace(float *d, const float *x, int64_t n, xg_stream s);
/* DenseMatrix::max_abs / all_finite (matrix.cpp:44-58): *max_abs, *finite */
xg_status xg_max_abs(const float *a, int64_t n, float *max_abs, int *finite, xg_stream s);

/* ---- sparse.hpp ---------------------------------------------------------- */
/* reduce_a (per_row=1) / reduce_b (per_row=0), sparse.hpp:46-54 /
 * sparse.cpp:36-85.  Two phases: xg_reduce_count fills row_ptr (rows+1) and
 * *nnz; xg_reduce_fill writes col_idx / values (capacity *nnz). */
xg_status xg_reduce_count(const float *m, int rows, int cols, const float *stat, double thr_m,
                          int policy, double scale_other, int per_row, int32_t *row_ptr,
                          int64_t *nnz, xg_stream s);
xg_status xg_reduce_fill(const float *m, int rows, int cols, const float *stat, double thr_m,
                         int policy, double scale_other, int per_row, const int32_t *row_ptr,
                         int32_t *col_idx, float *values, xg_stream s);
/* quantize_csr() sparse.hpp:74 / sparse.cpp:193-240 */
xg_status xg_quantize_csr(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                          const float *values, int64_t nnz, int bits, int scheme, int rounding,
                          int8_t *qvals, double *scales, xg_stream s);
/* csr_transpose<int8_t>() sparse.hpp:70 / sparse.cpp:168-188 */
xg_status xg_csr_transpose_i8(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                              const int8_t *values, int64_t nnz, int32_t *t_row_ptr,
                              int32_t *t_col_idx, int8_t *t_values, xg_stream s);
xg_status xg_csr_transpose_f32(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                               const float *values, int64_t nnz, int32_t *t_row_ptr,
                               int32_t *t_col_idx, float *t_values, xg_stream s);
/* spmm_int() sparse.hpp:64 / sparse.cpp:119-138 */
xg_status xg_spmm_i8(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                     const int8_t *values, const int8_t *d, int d_cols, int d_bits, int32_t *out,
                     xg_stream s);
/* Compensation kernel choice of the SparseResidual branch (no reference
 * equivalent: the reference always runs spmm_int there, pipeline.cpp:118-124).
 * The device picks the tcgen05 masked-dense launch or the CUDA-core CSR SpMM
 * from t_dense = 4MNK/p_tc against t_csr = max((nnzA N + nnzB M)/p_sp,
 * 16MN/bw) + (M+N)K/bw; force 0 auto, 1 dense, 2 CSR.  Values <= 0 (force < 0)
 * keep the current setting.  Process-wide. */
xg_status xg_comp_model_set(double p_tc, double p_sp, double bw, int force);
void xg_comp_model_get(double *p_tc, double *p_sp, double *bw, int *force);
/* calibrate_eta() calibrate.hpp:28 / calibrate.cpp:68-100 on the device: the
 * tcgen05 gemm_int against the CSR spmm_int on size x size int8 operands (random
 * CSR at bisected densities, CUDA-event timed, best of reps), eta = the density
 * where they cost the same.  Also returns the measured rates (int8 op/s of the
 * GEMM, MAC/s of the SpMM at eta); install != 0 makes them the compensation
 * cost model above. */
xg_status xg_calibrate_eta(int size, int bits, uint64_t seed, int install, double *eta, int *reps,
                           double *p_tc, double *p_sp);
/* spmm() sparse.hpp:61 / sparse.cpp:97-117 */
xg_status xg_spmm_f32(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                      const float *values, const float *d, int d_cols, float *out, xg_stream s);
/* csr_from_dense() / densify() sparse.hpp:66-67 */
xg_status xg_csr_from_dense_count(const float *a, int rows, int cols, int32_t *row_ptr,
                                  int64_t *nnz, xg_stream s);
xg_status xg_csr_from_dense_fill(const float *a, int rows, int cols, const int32_t *row_ptr,
                                 int32_t *col_idx, float *values, xg_stream s);
xg_status xg_densify(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                     const float *values, float *out, xg_stream s);

/* ---- pipeline.hpp -------------------------------------------------------- */
/* get_avg_vectors / get_abs_min_vectors, pipeline.hpp:64-67 */
xg_status xg_avg_vectors(const float *d, int rows, int cols, float *row, float *col, xg_stream s);
xg_status xg_abs_min_vectors(const float *d, int rows, int cols, float *row, float *col,
                             xg_stream s);
/* xigemm() pipeline.hpp:57-62 / pipeline.cpp:182-213: out = alpha*AB~ + beta*C.
 * c may be NULL (then beta is ignored).  reduce=0 gives
 * quantized_gemm_full_residual (pipeline.cpp:177-180). */
xg_status xg_xigemm(const float *a, const float *b, const float *c, float alpha, float beta,
                    int m, int k, int n, const xg_config *cfg, int reduce, float *out,
                    xg_report *rep, xg_dump *dump, xg_stream s);
/* quantized_gemm_direct(a, b, cfg), pipeline.hpp:44-45 / pipeline.cpp:166-175 */
xg_status xg_gemm_direct(const float *a, const float *b, int m, int k, int n,
                         const xg_config *cfg, float *out, xg_stream s);
/* quantized_gemm_direct(aq, bq), pipeline.hpp:48 / pipeline.cpp:162-164 */
xg_status xg_gemm_direct_q(const int8_t *aq, int scheme_a, const double *sa, const int8_t *bq,
                           int scheme_b, const double *sb, int m, int k, int n, int bits_a,
                           int bits_b, float *out, xg_stream s);

/* ---- row-sharded xigemm (multi-GPU) ----------------
 * The reference has no distributed path; this splits its xigemm()
 * (pipeline.cpp:182-213) by rows of A and C across ranks with B replicated.
 * Each rank creates a handle over its rows, then for p = 0..5 runs
 * xg_shard_step(h, p) followed by the collectives xg_shard_exchange(h, p, i)
 * describes (i = 0, 1, ... until *count == 0), executed by the caller on the
 * same stream order (NCCL over NVLink, or any exact reduction):
 *   dtype 0 uint32, 1 uint64, 2 float64, 3 float32;
 *   op 0 MAX, 1 SUM, 2 MIN (in place on send), 3 ALLGATHER (send -> recv,
 *   nranks * count elements in rank order).
 * After step 5, xg_shard_finish synchronises and fills the (global) report;
 * out_rows holds this rank's rows of the result, bit-identical to the
 * single-GPU xg_xigemm on the full problem. */
typedef struct xg_shard xg_shard;
xg_status xg_shard_create(const float *a_rows, const float *b, const float *c_rows, float alpha,
                          float beta, int rank, int nranks, const int *rank_rows, int k, int n,
                          const xg_config *cfg, int reduce, float *out_rows, xg_shard **h);
xg_status xg_shard_step(xg_shard *h, int step, xg_stream s);
xg_status xg_shard_exchange(xg_shard *h, int point, int idx, void **send, void **recv,
                            int64_t *count, int *dtype, int *op);
xg_status xg_shard_finish(xg_shard *h, xg_report *rep, xg_stream s);
void xg_shard_destroy(xg_shard *h);
/* Point 3 all-gathers the D_F columns of the (rare) AvgRule column means that
 * need the exact sequential sum; the buffer holds xg_shard_remote_cap(h)
 * columns (8 by default).  When a run flags more, xg_shard_finish returns
 * XG_EAGAIN (every rank sees the same count) and the results are not valid:
 * call xg_shard_set_remote_cap(h, xg_shard_remote_needed(h)) on every rank,
 * re-query the point-3 exchange (its buffers changed) and rerun steps 0-5. */
int xg_shard_remote_cap(const xg_shard *h);
int xg_shard_remote_needed(const xg_shard *h);
xg_status xg_shard_set_remote_cap(xg_shard *h, int cap);

/* ---- host-buffer entry points (what the C++ drop-in binds) --------------- */
xg_status xg_xigemm_host(const float *a, const float *b, const float *c, float alpha, float beta,
                         int m, int k, int n, const xg_config *cfg, int reduce, float *out,
                         xg_report *rep);
xg_status xg_gemm_direct_host(const float *a, const float *b, int m, int k, int n,
                              const xg_config *cfg, float *out);

/* ---- synthetic inputs (random_matrix.hpp analogue; bench/test data) ------ */
/* kind 0 uniform lo=p1 hi=p2 (test_support.hpp:16-24, bit-identical),
 * 1 normal(p1,p2), 2 Student-t(3)*p2, 3 exponential(p1).  n floats. */
int xg_generate(int kind, double p1, double p2, uint64_t seed, int64_t n, float *out,
                xg_stream s);

#ifdef __cplusplus
}
#endif
#endif
