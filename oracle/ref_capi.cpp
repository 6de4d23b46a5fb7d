// TEST INFRASTRUCTURE ONLY — extern "C" shim over the *unmodified* reference
// library, compiled from /root/reference/proj/src/*.cpp by oracle/Makefile with
// -Dxigemm=xigemm_ref so its symbols can live next to the product's xigemm::
// symbols in one process.  Used by tests/ to pin the C restatement
// (xigemm_oracle.c) and by bench.py's reference arm / cpu_baseline leg.
// Nothing from the reference is copied here; this file only calls its public
// API (proj/include/xigemm/*.hpp).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "xigemm/matrix.hpp"
#include "xigemm/pipeline.hpp"
#include "xigemm/quantize.hpp"
#include "xigemm/random_matrix.hpp"
#include "xigemm/sparse.hpp"

#include "xigemm_oracle.h"  // xo_config / xo_report / xo_dump layouts

using namespace xigemm;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 2;
    }
}

DenseMatrix dense(const float* p, int r, int c) {
    DenseMatrix m;
    m.rows = r;
    m.cols = c;
    m.data.assign(p, p + static_cast<size_t>(r) * c);
    return m;
}

ScaleFactors scales(int scheme, const double* v, int n) {
    ScaleFactors s;
    s.scheme = static_cast<ScaleScheme>(scheme);
    s.values.assign(v, v + n);
    return s;
}

int nsc(int scheme, int rows, int cols) { return scheme == 1 ? rows : scheme == 2 ? cols : 1; }

QuantizedMatrix qmat(const int8_t* p, int r, int c, int bits, int scheme, const double* sv) {
    QuantizedMatrix q;
    q.rows = r;
    q.cols = c;
    q.data.assign(p, p + static_cast<size_t>(r) * c);
    q.bits = static_cast<QuantBits>(bits);
    q.scales = scales(scheme, sv, nsc(scheme, r, c));
    return q;
}

XigemmConfig cfg_of(const xo_config* c) {
    XigemmConfig cfg;
    cfg.bits = static_cast<QuantBits>(c->bits);
    cfg.threshold = c->threshold;
    cfg.density_limit = c->density_limit;
    cfg.scheme = static_cast<QuantScheme>(c->scheme);
    cfg.policy = static_cast<ReductionPolicy>(c->policy);
    cfg.rounding = static_cast<RoundingMode>(c->rounding);
    return cfg;
}

template <class T>
SparseCsr<T> csr(int rows, int cols, const int32_t* rp, const int32_t* ci, const T* v) {
    SparseCsr<T> s;
    s.rows = rows;
    s.cols = cols;
    s.row_ptr.assign(rp, rp + rows + 1);
    const int64_t nnz = rp[rows];
    s.col_idx.assign(ci, ci + nnz);
    s.values.assign(v, v + nnz);
    return s;
}

}  // namespace

extern "C" {

int xr_version(void) { return 1; }

int xr_xigemm(const float* a, const float* b, const float* c, float alpha, float beta, int m,
              int k, int n, const xo_config* xc, int reduce, float* out, xo_report* rep) {
    return guarded([&] {
        const DenseMatrix A = dense(a, m, k), B = dense(b, k, n);
        const XigemmConfig cfg = cfg_of(xc);
        if (!reduce) {
            const DenseMatrix d = quantized_gemm_full_residual(A, B, cfg);
            std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
            return;
        }
        GemmReport r;
        if (c) {
            const DenseMatrix C = dense(c, m, n);
            r = xigemm::xigemm(A, B, &C, alpha, beta, cfg);
        } else {
            r = xigemm::xigemm(A, B, nullptr, alpha, beta, cfg);
        }
        std::memcpy(out, r.result.data.data(), sizeof(float) * r.result.data.size());
        if (rep) {
            rep->density_a = r.density_a;
            rep->density_b = r.density_b;
            rep->path = r.path == GemmPath::SparseResidual ? 0 : 1;
            rep->nnz_a = -1;
            rep->nnz_b = -1;
        }
    });
}

int xr_gemm_direct(const float* a, const float* b, int m, int k, int n, const xo_config* xc,
                   float* out) {
    return guarded([&] {
        const DenseMatrix d = quantized_gemm_direct(dense(a, m, k), dense(b, k, n), cfg_of(xc));
        std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
    });
}

int xr_quantize(const float* a, int rows, int cols, int bits, int scheme, int rounding, int8_t* q,
                double* sc) {
    return guarded([&] {
        const QuantizedMatrix r = quantize(dense(a, rows, cols), static_cast<QuantBits>(bits),
                                           static_cast<ScaleScheme>(scheme),
                                           static_cast<RoundingMode>(rounding));
        std::memcpy(q, r.data.data(), r.data.size());
        std::memcpy(sc, r.scales.values.data(), sizeof(double) * r.scales.values.size());
    });
}

int xr_quantize_with_scales(const float* a, int rows, int cols, int bits, int scheme,
                            const double* sv, int rounding, int8_t* q) {
    return guarded([&] {
        const QuantizedMatrix r = quantize_with_scales(
            dense(a, rows, cols), static_cast<QuantBits>(bits),
            scales(scheme, sv, nsc(scheme, rows, cols)), static_cast<RoundingMode>(rounding));
        std::memcpy(q, r.data.data(), r.data.size());
    });
}

int xr_dequantize(const int8_t* q, int rows, int cols, int scheme, const double* sv, float* out) {
    return guarded([&] {
        const DenseMatrix d = dequantize(qmat(q, rows, cols, 8, scheme, sv));
        std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
    });
}

int xr_residual(const float* a, const int8_t* q, int rows, int cols, int scheme, const double* sv,
                float* out) {
    return guarded([&] {
        const DenseMatrix d = residual(dense(a, rows, cols), qmat(q, rows, cols, 8, scheme, sv));
        std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
    });
}

int xr_dequant_product(const int32_t* p, int rows, int cols, int sa_scheme, const double* sa,
                       int sb_scheme, const double* sb, float* out) {
    return guarded([&] {
        IntMatrix P(rows, cols);
        std::memcpy(P.data.data(), p, sizeof(int32_t) * P.data.size());
        const DenseMatrix d = dequant_product(P, scales(sa_scheme, sa, nsc(sa_scheme, rows, 1)),
                                              scales(sb_scheme, sb, nsc(sb_scheme, 1, cols)));
        std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
    });
}

int xr_gemm_int(const int8_t* a, const int8_t* b, int m, int k, int n, int bits_a, int bits_b,
                int32_t* c) {
    return guarded([&] {
        const double one = 1.0;
        const IntMatrix r = gemm_int(qmat(a, m, k, bits_a, 0, &one), qmat(b, k, n, bits_b, 0, &one));
        std::memcpy(c, r.data.data(), sizeof(int32_t) * r.data.size());
    });
}

int xr_gemm_f32(const float* a, const float* b, int m, int k, int n, float* c) {
    return guarded([&] {
        const DenseMatrix r = gemm_f32(dense(a, m, k), dense(b, k, n));
        std::memcpy(c, r.data.data(), sizeof(float) * r.data.size());
    });
}

int xr_axpby(float* d, float alpha, const float* c, float beta, int rows, int cols) {
    return guarded([&] {
        DenseMatrix D = dense(d, rows, cols);
        axpby_inplace(D, alpha, dense(c, rows, cols), beta);
        std::memcpy(d, D.data.data(), sizeof(float) * D.data.size());
    });
}

int xr_avg_vectors(const float* d, int rows, int cols, float* row, float* col) {
    return guarded([&] {
        const auto [r, c] = get_avg_vectors(dense(d, rows, cols));
        std::memcpy(row, r.data(), sizeof(float) * r.size());
        std::memcpy(col, c.data(), sizeof(float) * c.size());
    });
}

int xr_abs_min_vectors(const float* d, int rows, int cols, float* row, float* col) {
    return guarded([&] {
        const auto [r, c] = get_abs_min_vectors(dense(d, rows, cols));
        std::memcpy(row, r.data(), sizeof(float) * r.size());
        std::memcpy(col, c.data(), sizeof(float) * c.size());
    });
}

int xr_reduce(const float* m, int rows, int cols, const float* stat, int nstat, double thr,
              int policy, double scale_other, int per_row, int32_t* row_ptr, int32_t* col_idx,
              float* values, int64_t* nnz) {
    return guarded([&] {
        const std::vector<float> st(stat, stat + nstat);
        const SparseCsrF32 s =
            per_row ? reduce_a(dense(m, rows, cols), st, thr,
                               static_cast<ReductionPolicy>(policy), scale_other)
                    : reduce_b(dense(m, rows, cols), st, thr,
                               static_cast<ReductionPolicy>(policy), scale_other);
        std::memcpy(row_ptr, s.row_ptr.data(), sizeof(int32_t) * s.row_ptr.size());
        std::memcpy(col_idx, s.col_idx.data(), sizeof(int32_t) * s.col_idx.size());
        std::memcpy(values, s.values.data(), sizeof(float) * s.values.size());
        *nnz = s.nnz();
    });
}

int xr_quantize_csr(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v,
                    int bits, int scheme, int rounding, int8_t* qv, double* sc) {
    return guarded([&] {
        const QuantizedCsr q = quantize_csr(csr<float>(rows, cols, rp, ci, v),
                                            static_cast<QuantBits>(bits),
                                            static_cast<ScaleScheme>(scheme),
                                            static_cast<RoundingMode>(rounding));
        std::memcpy(qv, q.matrix.values.data(), q.matrix.values.size());
        std::memcpy(sc, q.scales.values.data(), sizeof(double) * q.scales.values.size());
    });
}

int xr_csr_transpose_i8(int rows, int cols, const int32_t* rp, const int32_t* ci, const int8_t* v,
                        int32_t* trp, int32_t* tci, int8_t* tv) {
    return guarded([&] {
        const SparseCsrI8 t = csr_transpose(csr<int8_t>(rows, cols, rp, ci, v));
        std::memcpy(trp, t.row_ptr.data(), sizeof(int32_t) * t.row_ptr.size());
        std::memcpy(tci, t.col_idx.data(), sizeof(int32_t) * t.col_idx.size());
        std::memcpy(tv, t.values.data(), t.values.size());
    });
}

int xr_spmm_int(int rows, int cols, const int32_t* rp, const int32_t* ci, const int8_t* v,
                const int8_t* d, int d_cols, int d_bits, int32_t* out) {
    return guarded([&] {
        const double one = 1.0;
        const IntMatrix r =
            spmm_int(csr<int8_t>(rows, cols, rp, ci, v), qmat(d, cols, d_cols, d_bits, 0, &one));
        std::memcpy(out, r.data.data(), sizeof(int32_t) * r.data.size());
    });
}

int xr_spmm_f32(int rows, int cols, const int32_t* rp, const int32_t* ci, const float* v,
                const float* d, int d_cols, float* out) {
    return guarded([&] {
        const DenseMatrix r = spmm(csr<float>(rows, cols, rp, ci, v), dense(d, cols, d_cols));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int xr_generate(int kind, double p1, double p2, uint64_t seed, int rows, int cols, float* out) {
    return guarded([&] {
        DistributionSpec s{static_cast<DistKind>(kind), p1, p2, seed};
        const DenseMatrix d = generate(s, rows, cols);
        std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
    });
}

uint64_t xr_splitmix_next(uint64_t* state) {
    SplitMix64 r(*state);
    const uint64_t v = r.next();
    *state = r.state;
    return v;
}

// Stage-by-stage replay of run_residual_pipeline (pipeline.cpp:44-149) through
// the reference's own public stage functions, for golden intermediates.
int xr_pipeline_dump(const float* a, const float* b, int m, int k, int n, const xo_config* xc,
                     xo_dump* d) {
    return guarded([&] {
        const DenseMatrix A = dense(a, m, k), B = dense(b, k, n);
        const XigemmConfig cfg = cfg_of(xc);
        const bool vw = cfg.scheme == QuantScheme::VectorWise;
        const ScaleScheme ls = vw ? ScaleScheme::PerRow : ScaleScheme::PerTensor;
        const ScaleScheme rs = vw ? ScaleScheme::PerColumn : ScaleScheme::PerTensor;
        const QuantizedMatrix aq = quantize(A, cfg.bits, ls, cfg.rounding);
        const QuantizedMatrix bq = quantize(B, cfg.bits, rs, cfg.rounding);
        const IntMatrix dint = gemm_int(aq, bq);
        const DenseMatrix df = dequant_product(dint, aq.scales, bq.scales);
        const DenseMatrix ra = subtract(A, dequantize(aq));
        const DenseMatrix rb = subtract(B, dequantize(bq));
        const QuantizedMatrix raq = quantize(ra, cfg.bits, ScaleScheme::PerTensor, cfg.rounding);
        const QuantizedMatrix rbq = quantize(rb, cfg.bits, ScaleScheme::PerTensor, cfg.rounding);
        const auto stat = cfg.policy == ReductionPolicy::AvgRule ? get_avg_vectors(df)
                                                                  : get_abs_min_vectors(df);
        const double scale_a = compute_scale(A.max_abs(), cfg.bits);
        const double scale_b = compute_scale(B.max_abs(), cfg.bits);
        const SparseCsrF32 as = reduce_a(A, stat.first, cfg.threshold, cfg.policy, scale_b);
        const SparseCsrF32 bs = reduce_b(B, stat.second, cfg.threshold, cfg.policy, scale_a);
        const QuantizedCsr ar = quantize_csr(as, cfg.bits, ls, cfg.rounding);
        const QuantizedCsr br = quantize_csr(bs, cfg.bits, rs, cfg.rounding);
        const bool sparse = std::max(density(as), density(bs)) < cfg.density_limit;
        IntMatrix dr1, dr2;
        if (sparse) {
            dr1 = spmm_int(ar.matrix, rbq);
            dr2 = spmm_int(csr_transpose(br.matrix), raq.transposed()).transposed();
        } else {
            dr1 = gemm_int(aq, rbq);
            dr2 = gemm_int(raq, bq);
        }
        auto cp = [](auto* dst, const auto& v) {
            if (dst) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
        };
        cp(d->aq, aq.data);
        cp(d->aq_scales, aq.scales.values);
        cp(d->bq, bq.data);
        cp(d->bq_scales, bq.scales.values);
        cp(d->d_int, dint.data);
        cp(d->d_f, df.data);
        cp(d->raq, raq.data);
        if (d->raq_scale) *d->raq_scale = raq.scales.values[0];
        cp(d->rbq, rbq.data);
        if (d->rbq_scale) *d->rbq_scale = rbq.scales.values[0];
        cp(d->row_stat, stat.first);
        cp(d->col_stat, stat.second);
        auto dense_of = [](const SparseCsrF32& s, const std::vector<int8_t>& qv, uint8_t* mask,
                           int8_t* out) {
            if (mask) std::memset(mask, 0, static_cast<size_t>(s.rows) * s.cols);
            if (out) std::memset(out, 0, static_cast<size_t>(s.rows) * s.cols);
            for (int i = 0; i < s.rows; ++i)
                for (int32_t p = s.row_ptr[i]; p < s.row_ptr[i + 1]; ++p) {
                    const size_t x = static_cast<size_t>(i) * s.cols + s.col_idx[p];
                    if (mask) mask[x] = 1;
                    if (out) out[x] = qv[p];
                }
        };
        dense_of(as, ar.matrix.values, d->a_mask, d->a_red);
        dense_of(bs, br.matrix.values, d->b_mask, d->b_red);
        cp(d->a_red_scales, ar.scales.values);
        cp(d->b_red_scales, br.scales.values);
        cp(d->dr1, dr1.data);
        cp(d->dr2, dr2.data);
    });
}

}  // extern "C"
