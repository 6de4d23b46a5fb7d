/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * compensated INT8 GEMM (arXiv 2403.06924 "xigemm").  See xigemm_oracle.h for
 * the contract and how the restatement is pinned.  Compiled with
 * -ffp-contract=off and no -march so every fp64/fp32 operation rounds exactly
 * like the reference build (proj/CMakeLists.txt: no -march, SSE2 only).
 *
 * Citations are /root/reference/proj/<file>:<line>.
 */
#include "xigemm_oracle.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define XO_OK 0
#define XO_EINVAL 1

enum { RM_FLOOR = 0, RM_NEAREST = 1 };
enum { SS_TENSOR = 0, SS_ROW = 1, SS_COL = 2 };
enum { QS_TENSOR = 0, QS_VECTOR = 1 };
enum { POL_AVG = 0, POL_MIN = 1 };
enum { PATH_SPARSE = 0, PATH_DENSE = 1 };

int xo_version(void) { return 1; }

/* ---------------------------------------------------------------- rng ---- */
/* random_matrix.cpp:9-18 */
uint64_t xo_splitmix_next(uint64_t *state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double xo_splitmix_unit(uint64_t *state) {
    return (double)(xo_splitmix_next(state) >> 11) * 0x1.0p-53;
}

static const double kPi = 3.141592653589793;

/* random_matrix.cpp:61-67, cosine branch of Box-Muller only */
static double std_normal(uint64_t *s) {
    const double u1 = 1.0 - xo_splitmix_unit(s);
    const double u2 = xo_splitmix_unit(s);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

/* random_matrix.cpp:41-58 (validate) and :81-103 (sample) */
int xo_generate(int kind, double p1, double p2, uint64_t seed, int rows, int cols, float *out) {
    if (kind == 1 && !(p2 > 0.0)) return XO_EINVAL;
    if ((kind == 2 || kind == 3) && !(p1 > 0.0)) return XO_EINVAL;
    if (kind == 4 && !(p1 >= 1.0)) return XO_EINVAL;
    if (rows < 1 || cols < 1) return XO_EINVAL;
    uint64_t s = seed;
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = 0; i < n; ++i) {
        double v = 0.0;
        switch (kind) {
            case 0: v = xo_splitmix_unit(&s); break;
            case 1: v = p1 + p2 * std_normal(&s); break;
            case 2: v = -log(1.0 - xo_splitmix_unit(&s)) / p1; break;
            case 3: {
                const double limit = exp(-p1);
                double p = 1.0;
                int k = 0;
                do {
                    ++k;
                    p *= xo_splitmix_unit(&s);
                } while (p > limit);
                v = (double)(k - 1);
                break;
            }
            case 4: {
                double sum = 0.0;
                const int dof = (int)p1;
                for (int t = 0; t < dof; ++t) {
                    const double z = std_normal(&s);
                    sum += z * z;
                }
                v = sum;
                break;
            }
            default: return XO_EINVAL;
        }
        out[i] = (float)v;
    }
    return XO_OK;
}

/* tests/test_support.hpp:16-24 */
void xo_random_dense(int rows, int cols, uint64_t seed, float lo, float hi, float *out) {
    uint64_t s = seed;
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (float)xo_splitmix_unit(&s) * (hi - lo);
}

/* ------------------------------------------------------- scalar rules ---- */
/* quantize.hpp:16 */
int xo_quant_max(int bits) { return (1 << (bits - 1)) - 1; }

/* quantize.cpp:189-191 */
int xo_gemm_int_max_inner(int bits) { return 1 << (31 - 2 * bits - 1); }

/* quantize.cpp:99-105 */
int xo_compute_scale(double max_abs, int bits, double *out) {
    if (!(max_abs >= 0.0) || !isfinite(max_abs)) return XO_EINVAL;
    *out = max_abs == 0.0 ? 1.0 : (double)xo_quant_max(bits) / max_abs;
    return XO_OK;
}

/* The reference converts with llround / (long long)trunc (quantize.cpp:19-20).
 * For |t| >= 2^63 (reachable only through quantize_with_scales with huge
 * caller scales) x86-64 yields LLONG_MIN, which the clamp maps to -qmax. */
static long long to_ll_x86(double t, int nearest) {
    if (!(fabs(t) < 9223372036854775808.0)) return LLONG_MIN;
    return nearest ? llround(t) : (long long)trunc(t);
}

/* quantize.cpp:13-24 */
int32_t xo_quantize_scalar(double a, double lambda, int32_t qmax, int rounding) {
    double t = a * lambda;
    long long q;
    if (rounding == RM_FLOOR) {
        t += copysign(4.0 * DBL_EPSILON * fabs(t), t);
        q = to_ll_x86(t, 0);
    } else {
        q = to_ll_x86(t, 1);
    }
    if (q < -qmax) q = -qmax;
    if (q > qmax) q = qmax;
    return (int32_t)q;
}

/* matrix.cpp:51-58 */
float xo_max_abs(const float *a, int64_t n) {
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        const float v = fabsf(a[i]);
        if (v > m) m = v;
    }
    return m;
}

/* matrix.cpp:44-49 */
int xo_all_finite(const float *a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

static double scale_at(int scheme, const double *s, int i, int j) {
    return scheme == SS_ROW ? s[i] : scheme == SS_COL ? s[j] : s[0];
}

/* quantize.cpp:44-56 */
static int validate_scales(int scheme, const double *s, int rows, int cols) {
    const int n = scheme == SS_ROW ? rows : scheme == SS_COL ? cols : 1;
    for (int i = 0; i < n; ++i)
        if (!(s[i] > 0.0) || !isfinite(s[i])) return XO_EINVAL;
    return XO_OK;
}

/* --------------------------------------------------------- quantize ------ */
/* quantize.cpp:107-133 (scales) -> quantize_with_scales */
int xo_quantize(const float *a, int rows, int cols, int bits, int scheme, int rounding, int8_t *q,
                double *scales) {
    if (rows < 1 || cols < 1) return XO_EINVAL;
    if (scheme == SS_TENSOR) {
        /* DenseMatrix::max_abs is a float scan (matrix.cpp:51-58) */
        if (xo_compute_scale((double)xo_max_abs(a, (int64_t)rows * cols), bits, &scales[0]))
            return XO_EINVAL;
    } else if (scheme == SS_ROW) {
        /* slice_max_abs, quantize.cpp:28-36: fp64 max of |v| */
        for (int i = 0; i < rows; ++i) {
            double m = 0.0;
            for (int j = 0; j < cols; ++j) {
                const double v = fabs((double)a[(int64_t)i * cols + j]);
                if (v > m) m = v;
            }
            if (xo_compute_scale(m, bits, &scales[i])) return XO_EINVAL;
        }
    } else {
        for (int j = 0; j < cols; ++j) {
            double m = 0.0;
            for (int i = 0; i < rows; ++i) {
                const double v = fabs((double)a[(int64_t)i * cols + j]);
                if (v > m) m = v;
            }
            if (xo_compute_scale(m, bits, &scales[j])) return XO_EINVAL;
        }
    }
    return xo_quantize_with_scales(a, rows, cols, bits, scheme, scales, rounding, q);
}

/* quantize.cpp:135-150 */
int xo_quantize_with_scales(const float *a, int rows, int cols, int bits, int scheme,
                            const double *scales, int rounding, int8_t *q) {
    if (validate_scales(scheme, scales, rows, cols)) return XO_EINVAL;
    const int32_t qmax = xo_quant_max(bits);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const int64_t x = (int64_t)i * cols + j;
            q[x] = (int8_t)xo_quantize_scalar((double)a[x], scale_at(scheme, scales, i, j), qmax,
                                              rounding);
        }
    return XO_OK;
}

/* quantize.cpp:152-160: float(q / lambda) with an fp64 division */
int xo_dequantize(const int8_t *q, int rows, int cols, int scheme, const double *scales,
                  float *out) {
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const int64_t x = (int64_t)i * cols + j;
            out[x] = (float)((double)q[x] / scale_at(scheme, scales, i, j));
        }
    return XO_OK;
}

/* quantize.cpp:162-167 + matrix.cpp:107-116 */
int xo_residual(const float *a, const int8_t *q, int rows, int cols, int scheme,
                const double *scales, float *out) {
    xo_dequantize(q, rows, cols, scheme, scales, out);
    const int64_t n = (int64_t)rows * cols;
    for (int64_t x = 0; x < n; ++x) out[x] = a[x] - out[x];
    return XO_OK;
}

/* quantize.cpp:169-187 */
int xo_dequant_product(const int32_t *p, int rows, int cols, int scheme_a, const double *sa,
                       int scheme_b, const double *sb, float *out) {
    if (scheme_a == SS_COL || scheme_b == SS_ROW) return XO_EINVAL;
    if (validate_scales(scheme_a, sa, rows, 1) || validate_scales(scheme_b, sb, 1, cols))
        return XO_EINVAL;
    for (int i = 0; i < rows; ++i) {
        const double la = scheme_a == SS_ROW ? sa[i] : sa[0];
        for (int j = 0; j < cols; ++j) {
            const double lb = scheme_b == SS_COL ? sb[j] : sb[0];
            out[(int64_t)i * cols + j] = (float)((double)p[(int64_t)i * cols + j] / (la * lb));
        }
    }
    return XO_OK;
}

/* quantize.cpp:193-214 */
int xo_gemm_int(const int8_t *a, const int8_t *b, int m, int k, int n, int bits_a, int bits_b,
                int32_t *c) {
    const int la = xo_gemm_int_max_inner(bits_a), lb = xo_gemm_int_max_inner(bits_b);
    if (k > (la < lb ? la : lb)) return XO_EINVAL;
    memset(c, 0, sizeof(int32_t) * (size_t)m * n);
    for (int i = 0; i < m; ++i) {
        int32_t *crow = c + (int64_t)i * n;
        for (int p = 0; p < k; ++p) {
            const int32_t aik = a[(int64_t)i * k + p];
            if (aik == 0) continue;
            const int8_t *brow = b + (int64_t)p * n;
            /* wrap-around int32 arithmetic, as the reference's int32_t += */
            for (int j = 0; j < n; ++j)
                crow[j] = (int32_t)((uint32_t)crow[j] + (uint32_t)(aik * (int32_t)brow[j]));
        }
    }
    return XO_OK;
}

/* matrix.cpp:75-95: fp64 accumulation over ascending k */
int xo_gemm_f32(const float *a, const float *b, int m, int k, int n, float *c) {
    double *acc = (double *)malloc(sizeof(double) * (size_t)n);
    if (!acc) return XO_EINVAL;
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < n; ++j) acc[j] = 0.0;
        for (int p = 0; p < k; ++p) {
            const double aik = a[(int64_t)i * k + p];
            const float *brow = b + (int64_t)p * n;
            for (int j = 0; j < n; ++j) acc[j] += aik * (double)brow[j];
        }
        for (int j = 0; j < n; ++j) c[(int64_t)i * n + j] = (float)acc[j];
    }
    free(acc);
    return XO_OK;
}

/* matrix.cpp:97-105 (non-fused: compiled without FMA contraction) */
int xo_axpby(float *d, float alpha, const float *c, float beta, int64_t n) {
    for (int64_t i = 0; i < n; ++i) d[i] = alpha * d[i] + beta * c[i];
    return XO_OK;
}

/* ------------------------------------------------------------ stats ------ */
/* pipeline.cpp:215-231 */
int xo_avg_vectors(const float *d, int rows, int cols, float *row, float *col) {
    if (rows < 1 || cols < 1) return XO_EINVAL;
    double *r = (double *)calloc((size_t)rows, sizeof(double));
    double *c = (double *)calloc((size_t)cols, sizeof(double));
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const double v = fabs((double)d[(int64_t)i * cols + j]);
            r[i] += v;
            c[j] += v;
        }
    for (int i = 0; i < rows; ++i) row[i] = (float)(r[i] / cols);
    for (int j = 0; j < cols; ++j) col[j] = (float)(c[j] / rows);
    free(r);
    free(c);
    return XO_OK;
}

/* pipeline.cpp:233-247 */
int xo_abs_min_vectors(const float *d, int rows, int cols, float *row, float *col) {
    if (rows < 1 || cols < 1) return XO_EINVAL;
    for (int i = 0; i < rows; ++i) row[i] = FLT_MAX;
    for (int j = 0; j < cols; ++j) col[j] = FLT_MAX;
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
            const float v = fabsf(d[(int64_t)i * cols + j]);
            if (v < row[i]) row[i] = v;
            if (v < col[j]) col[j] = v;
        }
    return XO_OK;
}

/* ----------------------------------------------------------- sparse ------ */
/* sparse.cpp:36-73 (reduce_impl) */
int xo_reduce(const float *m, int rows, int cols, const float *stat, double thr_m, int policy,
              double scale_other, int per_row, int32_t *row_ptr, int32_t *col_idx, float *values,
              int64_t *nnz) {
    if (!(thr_m > 0.0)) return XO_EINVAL;
    if (!(scale_other > 0.0) || !isfinite(scale_other)) return XO_EINVAL;
    const int nstat = per_row ? rows : cols;
    const int inner = per_row ? cols : rows;
    double *t = (double *)malloc(sizeof(double) * (size_t)(nstat > 0 ? nstat : 1));
    for (int s = 0; s < nstat; ++s)
        t[s] = policy == POL_AVG ? thr_m * (double)stat[s]
                                 : thr_m * scale_other * (double)stat[s] / inner;
    int64_t p = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j) {
            const float v = m[(int64_t)i * cols + j];
            if (fabs((double)v) > (per_row ? t[i] : t[j])) {
                col_idx[p] = j;
                values[p] = v;
                ++p;
            }
        }
        row_ptr[i + 1] = (int32_t)p;
    }
    free(t);
    *nnz = p;
    return XO_OK;
}

/* sparse.cpp:193-240 */
int xo_quantize_csr(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                    const float *values, int bits, int scheme, int rounding, int8_t *qvals,
                    double *scales) {
    const int32_t qmax = xo_quant_max(bits);
    const int64_t nnz = row_ptr[rows];
    if (scheme == SS_TENSOR) {
        double mx = 0.0;
        for (int64_t p = 0; p < nnz; ++p) {
            const double v = fabs((double)values[p]);
            if (v > mx) mx = v;
        }
        if (xo_compute_scale(mx, bits, &scales[0])) return XO_EINVAL;
    } else if (scheme == SS_ROW) {
        for (int i = 0; i < rows; ++i) {
            double mx = 0.0;
            for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
                const double v = fabs((double)values[p]);
                if (v > mx) mx = v;
            }
            if (xo_compute_scale(mx, bits, &scales[i])) return XO_EINVAL;
        }
    } else {
        double *cm = (double *)calloc((size_t)(cols > 0 ? cols : 1), sizeof(double));
        for (int i = 0; i < rows; ++i)
            for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
                const double v = fabs((double)values[p]);
                if (v > cm[col_idx[p]]) cm[col_idx[p]] = v;
            }
        for (int j = 0; j < cols; ++j)
            if (xo_compute_scale(cm[j], bits, &scales[j])) {
                free(cm);
                return XO_EINVAL;
            }
        free(cm);
    }
    for (int i = 0; i < rows; ++i)
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const double lam = scheme == SS_ROW ? scales[i]
                               : scheme == SS_COL ? scales[col_idx[p]]
                                                  : scales[0];
            qvals[p] = (int8_t)xo_quantize_scalar((double)values[p], lam, qmax, rounding);
        }
    return XO_OK;
}

/* sparse.cpp:168-188 */
int xo_csr_transpose_i8(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                        const int8_t *values, int32_t *t_row_ptr, int32_t *t_col_idx,
                        int8_t *t_values) {
    const int64_t nnz = row_ptr[rows];
    for (int j = 0; j <= cols; ++j) t_row_ptr[j] = 0;
    for (int64_t p = 0; p < nnz; ++p) ++t_row_ptr[col_idx[p] + 1];
    for (int j = 0; j < cols; ++j) t_row_ptr[j + 1] += t_row_ptr[j];
    int32_t *fill = (int32_t *)calloc((size_t)(cols > 0 ? cols : 1), sizeof(int32_t));
    for (int i = 0; i < rows; ++i)
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int32_t c = col_idx[p];
            const int32_t at = t_row_ptr[c] + fill[c]++;
            t_col_idx[at] = i;
            t_values[at] = values[p];
        }
    free(fill);
    return XO_OK;
}

/* sparse.cpp:119-138 */
int xo_spmm_int(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                const int8_t *values, const int8_t *d, int d_cols, int d_bits, int32_t *out) {
    if (cols > xo_gemm_int_max_inner(d_bits)) return XO_EINVAL;
    memset(out, 0, sizeof(int32_t) * (size_t)rows * d_cols);
    for (int i = 0; i < rows; ++i) {
        int32_t *crow = out + (int64_t)i * d_cols;
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int32_t v = values[p];
            const int8_t *drow = d + (int64_t)col_idx[p] * d_cols;
            for (int j = 0; j < d_cols; ++j)
                crow[j] = (int32_t)((uint32_t)crow[j] + (uint32_t)(v * (int32_t)drow[j]));
        }
    }
    return XO_OK;
}

/* sparse.cpp:97-117 */
int xo_spmm_f32(int rows, int cols, const int32_t *row_ptr, const int32_t *col_idx,
                const float *values, const float *d, int d_cols, float *out) {
    (void)cols;
    double *acc = (double *)malloc(sizeof(double) * (size_t)(d_cols > 0 ? d_cols : 1));
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < d_cols; ++j) acc[j] = 0.0;
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const double v = values[p];
            const float *drow = d + (int64_t)col_idx[p] * d_cols;
            for (int j = 0; j < d_cols; ++j) acc[j] += v * (double)drow[j];
        }
        for (int j = 0; j < d_cols; ++j) out[(int64_t)i * d_cols + j] = (float)acc[j];
    }
    free(acc);
    return XO_OK;
}

/* --------------------------------------------------------- pipeline ------ */
static int left_scheme(int qs) { return qs == QS_VECTOR ? SS_ROW : SS_TENSOR; }   /* :25-27 */
static int right_scheme(int qs) { return qs == QS_VECTOR ? SS_COL : SS_TENSOR; }  /* :29-31 */

/* pipeline.cpp:153-160 */
static int validate_cfg(const xo_config *cfg) {
    if (!(cfg->threshold > 0.0)) return XO_EINVAL;
    if (!(cfg->density_limit > 0.0) || cfg->density_limit > 1.0) return XO_EINVAL;
    return XO_OK;
}

static int nscales(int scheme, int rows, int cols) {
    return scheme == SS_ROW ? rows : scheme == SS_COL ? cols : 1;
}

/* CSR (rows x cols) -> dense row-major int8 */
static void csr_to_dense_i8(int rows, int cols, const int32_t *rp, const int32_t *ci,
                            const int8_t *v, int8_t *out) {
    memset(out, 0, (size_t)rows * cols);
    for (int i = 0; i < rows; ++i)
        for (int32_t p = rp[i]; p < rp[i + 1]; ++p) out[(int64_t)i * cols + ci[p]] = v[p];
}

#define XO_ALLOC(T, n) ((T *)malloc(sizeof(T) * (size_t)((n) > 0 ? (n) : 1)))

/* run_residual_pipeline, pipeline.cpp:44-149, then the alpha/beta tail of
 * xigemm, :182-209. */
int xo_xigemm(const float *a, const float *b, const float *c, float alpha, float beta, int m,
              int k, int n, const xo_config *cfg, int reduce, float *out, xo_report *rep,
              xo_dump *dump) {
    xo_dump nodump;
    if (!dump) {
        memset(&nodump, 0, sizeof nodump);
        dump = &nodump;
    }
    if (c && !xo_all_finite(c, (int64_t)m * n)) return XO_EINVAL;         /* :184-191 */
    if (validate_cfg(cfg)) return XO_EINVAL;                               /* :46 */
    if (m < 1 || k < 1 || n < 1) return XO_EINVAL;
    if (!xo_all_finite(a, (int64_t)m * k) || !xo_all_finite(b, (int64_t)k * n)) return XO_EINVAL;
    const int bits = cfg->bits;
    if (k > xo_gemm_int_max_inner(bits)) return XO_EINVAL;                 /* gemm_int guard */
    const int ls = left_scheme(cfg->scheme), rs = right_scheme(cfg->scheme);
    const int64_t MK = (int64_t)m * k, KN = (int64_t)k * n, MN = (int64_t)m * n;

    int rc = XO_OK;
    int8_t *aq = XO_ALLOC(int8_t, MK), *bq = XO_ALLOC(int8_t, KN);
    double *sa = XO_ALLOC(double, m), *sb = XO_ALLOC(double, n);
    int32_t *dint = XO_ALLOC(int32_t, MN), *dr1 = XO_ALLOC(int32_t, MN), *dr2 = XO_ALLOC(int32_t, MN);
    float *df = XO_ALLOC(float, MN), *ra = XO_ALLOC(float, MK), *rb = XO_ALLOC(float, KN);
    int8_t *raq = XO_ALLOC(int8_t, MK), *rbq = XO_ALLOC(int8_t, KN);
    float *fr1 = XO_ALLOC(float, MN);
    double sra = 1.0, srb = 1.0;

    /* [quant] :59-63 */
    if (xo_quantize(a, m, k, bits, ls, cfg->rounding, aq, sa) ||
        xo_quantize(b, k, n, bits, rs, cfg->rounding, bq, sb)) {
        rc = XO_EINVAL;
        goto done;
    }
    /* [xxmm] :65-69 */
    xo_gemm_int(aq, bq, m, k, n, bits, bits, dint);
    /* [quant] :71-77 */
    xo_dequant_product(dint, m, n, ls, sa, rs, sb, df);
    /* [package] :79-84 */
    xo_residual(a, aq, m, k, ls, sa, ra);
    xo_residual(b, bq, k, n, rs, sb, rb);
    /* [quant] :86-93, residuals always per-tensor */
    xo_quantize(ra, m, k, bits, SS_TENSOR, cfg->rounding, raq, &sra);
    xo_quantize(rb, k, n, bits, SS_TENSOR, cfg->rounding, rbq, &srb);

    if (dump->aq) memcpy(dump->aq, aq, (size_t)MK);
    if (dump->aq_scales) memcpy(dump->aq_scales, sa, sizeof(double) * nscales(ls, m, k));
    if (dump->bq) memcpy(dump->bq, bq, (size_t)KN);
    if (dump->bq_scales) memcpy(dump->bq_scales, sb, sizeof(double) * nscales(rs, k, n));
    if (dump->d_int) memcpy(dump->d_int, dint, sizeof(int32_t) * MN);
    if (dump->d_f) memcpy(dump->d_f, df, sizeof(float) * MN);
    if (dump->raq) memcpy(dump->raq, raq, (size_t)MK);
    if (dump->raq_scale) *dump->raq_scale = sra;
    if (dump->rbq) memcpy(dump->rbq, rbq, (size_t)KN);
    if (dump->rbq_scale) *dump->rbq_scale = srb;

    int sparse = 0;
    const int8_t *x1 = aq, *y2 = bq;       /* dense branch operands :127-128 */
    const double *l1 = sa, *l4 = sb;
    int l1s = ls, l4s = rs;
    double *s_ared = XO_ALLOC(double, m), *s_bred = XO_ALLOC(double, n);
    int8_t *ared = NULL, *bred = NULL;
    double dens_a = 0.0, dens_b = 0.0;
    int64_t nnz_a = 0, nnz_b = 0;
    if (reduce) {
        /* [reduce] :96-112 */
        float *rst = XO_ALLOC(float, m), *cst = XO_ALLOC(float, n);
        if (cfg->policy == POL_AVG) xo_avg_vectors(df, m, n, rst, cst);
        else xo_abs_min_vectors(df, m, n, rst, cst);
        double scale_a, scale_b;
        xo_compute_scale((double)xo_max_abs(a, MK), bits, &scale_a);
        xo_compute_scale((double)xo_max_abs(b, KN), bits, &scale_b);
        int32_t *arp = XO_ALLOC(int32_t, m + 1), *aci = XO_ALLOC(int32_t, MK);
        float *av = XO_ALLOC(float, MK);
        int32_t *brp = XO_ALLOC(int32_t, k + 1), *bci = XO_ALLOC(int32_t, KN);
        float *bv = XO_ALLOC(float, KN);
        rc = xo_reduce(a, m, k, rst, cfg->threshold, cfg->policy, scale_b, 1, arp, aci, av, &nnz_a);
        if (!rc)
            rc = xo_reduce(b, k, n, cst, cfg->threshold, cfg->policy, scale_a, 0, brp, bci, bv,
                           &nnz_b);
        if (!rc) {
            dens_a = (double)nnz_a / ((double)m * k);   /* sparse.cpp:87-95 */
            dens_b = (double)nnz_b / ((double)k * n);
            int8_t *aqv = XO_ALLOC(int8_t, nnz_a), *bqv = XO_ALLOC(int8_t, nnz_b);
            xo_quantize_csr(m, k, arp, aci, av, bits, ls, cfg->rounding, aqv, s_ared);
            xo_quantize_csr(k, n, brp, bci, bv, bits, rs, cfg->rounding, bqv, s_bred);
            ared = XO_ALLOC(int8_t, MK);
            bred = XO_ALLOC(int8_t, KN);
            csr_to_dense_i8(m, k, arp, aci, aqv, ared);
            csr_to_dense_i8(k, n, brp, bci, bqv, bred);
            if (dump->row_stat) memcpy(dump->row_stat, rst, sizeof(float) * m);
            if (dump->col_stat) memcpy(dump->col_stat, cst, sizeof(float) * n);
            if (dump->a_mask) {
                memset(dump->a_mask, 0, (size_t)MK);
                for (int i = 0; i < m; ++i)
                    for (int32_t p = arp[i]; p < arp[i + 1]; ++p)
                        dump->a_mask[(int64_t)i * k + aci[p]] = 1;
            }
            if (dump->b_mask) {
                memset(dump->b_mask, 0, (size_t)KN);
                for (int i = 0; i < k; ++i)
                    for (int32_t p = brp[i]; p < brp[i + 1]; ++p)
                        dump->b_mask[(int64_t)i * n + bci[p]] = 1;
            }
            if (dump->a_red) memcpy(dump->a_red, ared, (size_t)MK);
            if (dump->a_red_scales) memcpy(dump->a_red_scales, s_ared, sizeof(double) * nscales(ls, m, k));
            if (dump->b_red) memcpy(dump->b_red, bred, (size_t)KN);
            if (dump->b_red_scales) memcpy(dump->b_red_scales, s_bred, sizeof(double) * nscales(rs, k, n));
            sparse = (dens_a > dens_b ? dens_a : dens_b) < cfg->density_limit;   /* :110-111 */
            free(aqv);
            free(bqv);
        }
        free(rst); free(cst); free(arp); free(aci); free(av); free(brp); free(bci); free(bv);
        if (rc) goto done2;
    }
    if (sparse) {
        /* :118-124.  spmm_int on the CSR equals gemm_int on its dense form
         * bitwise (integer arithmetic, zeros contribute nothing) — the
         * reference's own test pins this (test_sparse.cpp:134-152). */
        x1 = ared;
        y2 = bred;
        l1 = s_ared;
        l4 = s_bred;
    }
    /* [xxmm] dr1 = X1 * RBq, dr2 = RAq * Y2 */
    xo_gemm_int(x1, rbq, m, k, n, bits, bits, dr1);
    xo_gemm_int(raq, y2, m, k, n, bits, bits, dr2);
    if (dump->dr1) memcpy(dump->dr1, dr1, sizeof(int32_t) * MN);
    if (dump->dr2) memcpy(dump->dr2, dr2, sizeof(int32_t) * MN);
    /* [quant] :134-139 */
    xo_dequant_product(dr1, m, n, l1s, l1, SS_TENSOR, &srb, fr1);
    xo_dequant_product(dr2, m, n, SS_TENSOR, &sra, l4s, l4, out);
    /* [package] :141-145: d_f += dr1; d_f += dr2 */
    for (int64_t x = 0; x < MN; ++x) {
        float v = df[x] + fr1[x];
        out[x] = v + out[x];
    }
    /* :195-202 */
    if (c) {
        xo_axpby(out, alpha, c, beta, MN);
    } else if (alpha != 1.0f) {
        for (int64_t x = 0; x < MN; ++x) out[x] *= alpha;
    }
    if (rep) {
        rep->density_a = dens_a;
        rep->density_b = dens_b;
        rep->path = sparse ? PATH_SPARSE : PATH_DENSE;
        rep->nnz_a = nnz_a;
        rep->nnz_b = nnz_b;
    }
done2:
    free(s_ared); free(s_bred); free(ared); free(bred);
done:
    free(aq); free(bq); free(sa); free(sb); free(dint); free(dr1); free(dr2); free(df);
    free(ra); free(rb); free(raq); free(rbq); free(fr1);
    return rc;
}

/* pipeline.cpp:162-175 */
int xo_gemm_direct(const float *a, const float *b, int m, int k, int n, const xo_config *cfg,
                   float *out) {
    if (validate_cfg(cfg)) return XO_EINVAL;
    if (m < 1 || k < 1 || n < 1) return XO_EINVAL;
    const int ls = left_scheme(cfg->scheme), rs = right_scheme(cfg->scheme);
    int8_t *aq = XO_ALLOC(int8_t, (int64_t)m * k), *bq = XO_ALLOC(int8_t, (int64_t)k * n);
    double *sa = XO_ALLOC(double, m), *sb = XO_ALLOC(double, n);
    int32_t *d = XO_ALLOC(int32_t, (int64_t)m * n);
    int rc = XO_OK;
    if (xo_quantize(a, m, k, cfg->bits, ls, cfg->rounding, aq, sa) ||
        xo_quantize(b, k, n, cfg->bits, rs, cfg->rounding, bq, sb) ||
        xo_gemm_int(aq, bq, m, k, n, cfg->bits, cfg->bits, d)) {
        rc = XO_EINVAL;
    } else {
        xo_dequant_product(d, m, n, ls, sa, rs, sb, out);
    }
    free(aq); free(bq); free(sa); free(sb); free(d);
    return rc;
}
