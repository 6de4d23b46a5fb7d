// xigemm drop-in: sparse.hpp and pipeline.hpp over the C-ABI.
// Reference: proj/src/sparse.cpp, proj/src/pipeline.cpp.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "dev.hpp"
#include "xigemm/pipeline.hpp"
#include "xigemm/sparse.hpp"

namespace xigemm {

using detail::check;
using detail::DevBuf;
using detail::xs;

// ---------------------------------------------------------------- sparse.hpp
template <typename T>
void SparseCsr<T>::validate() const {
    if (rows < 0 || cols < 0) throw std::invalid_argument("csr: negative dimensions");
    if (row_ptr.size() != static_cast<std::size_t>(rows) + 1 || row_ptr.front() != 0 ||
        row_ptr.back() != nnz() || col_idx.size() != values.size())
        throw std::invalid_argument("csr: inconsistent structure");
    for (int i = 0; i < rows; ++i) {
        if (row_ptr[i] > row_ptr[i + 1]) throw std::invalid_argument("csr: row_ptr not nondecreasing");
        for (std::int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            if (col_idx[p] < 0 || col_idx[p] >= cols) throw std::invalid_argument("csr: column index out of range");
            if (p > row_ptr[i] && col_idx[p] <= col_idx[p - 1])
                throw std::invalid_argument("csr: column indices not strictly increasing");
        }
    }
}
template void SparseCsr<float>::validate() const;
template void SparseCsr<std::int8_t>::validate() const;

namespace {

SparseCsrF32 reduce_dev(const DenseMatrix& m, const std::vector<float>& stat, double thr, ReductionPolicy policy,
                        double scale_other, bool per_row) {
    if (!(thr > 0.0)) throw std::invalid_argument("reduce: threshold M must be positive");
    if (!(scale_other > 0.0) || !std::isfinite(scale_other))
        throw std::invalid_argument("reduce: operand scale must be positive and finite");
    if (stat.size() != static_cast<std::size_t>(per_row ? m.rows : m.cols))
        throw std::invalid_argument("reduce: stat vector length mismatch");
    SparseCsrF32 s;
    s.rows = m.rows;
    s.cols = m.cols;
    DevBuf<float> dm(m.data), dst(stat);
    DevBuf<std::int32_t> drp(static_cast<std::size_t>(m.rows) + 1);
    int64_t nnz = 0;
    check(xg_reduce_count(dm.get(), m.rows, m.cols, dst.get(), thr, static_cast<int>(policy), scale_other,
                          per_row ? 1 : 0, drp.get(), &nnz, xs()));
    DevBuf<std::int32_t> dci(static_cast<std::size_t>(nnz));
    DevBuf<float> dv(static_cast<std::size_t>(nnz));
    check(xg_reduce_fill(dm.get(), m.rows, m.cols, dst.get(), thr, static_cast<int>(policy), scale_other,
                         per_row ? 1 : 0, drp.get(), dci.get(), dv.get(), xs()));
    s.row_ptr = drp.to_vector(drp.size());
    s.col_idx = dci.to_vector(nnz);
    s.values = dv.to_vector(nnz);
    return s;
}

}  // namespace

SparseCsrF32 reduce_a(const DenseMatrix& a, const std::vector<float>& c_row_stat, double m,
                      ReductionPolicy policy, double scale_other) {
    return reduce_dev(a, c_row_stat, m, policy, scale_other, true);
}

SparseCsrF32 reduce_b(const DenseMatrix& b, const std::vector<float>& c_col_stat, double m,
                      ReductionPolicy policy, double scale_other) {
    return reduce_dev(b, c_col_stat, m, policy, scale_other, false);
}

double density(const SparseCsrF32& s) {
    if (s.rows == 0 || s.cols == 0) return 0.0;
    return static_cast<double>(s.nnz()) / (static_cast<double>(s.rows) * s.cols);
}

double density(const SparseCsrI8& s) {
    if (s.rows == 0 || s.cols == 0) return 0.0;
    return static_cast<double>(s.nnz()) / (static_cast<double>(s.rows) * s.cols);
}

DenseMatrix spmm(const SparseCsrF32& s, const DenseMatrix& d) {
    if (s.cols != d.rows) throw std::invalid_argument("spmm: inner dimensions do not match");
    DenseMatrix out(s.rows, d.cols);
    DevBuf<std::int32_t> rp(s.row_ptr), ci(s.col_idx);
    DevBuf<float> v(s.values), dd(d.data), dout(out.data.size());
    check(xg_spmm_f32(s.rows, s.cols, rp.get(), ci.get(), v.get(), dd.get(), d.cols, dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

IntMatrix spmm_int(const SparseCsrI8& s, const QuantizedMatrix& d) {
    if (s.cols != d.rows) throw std::invalid_argument("spmm_int: inner dimensions do not match");
    if (s.cols > gemm_int_max_inner(d.bits))
        throw std::invalid_argument("spmm_int: inner dimension permits 32-bit overflow");
    IntMatrix out(s.rows, d.cols);
    DevBuf<std::int32_t> rp(s.row_ptr), ci(s.col_idx), dout(out.data.size());
    DevBuf<std::int8_t> v(s.values), dd(d.data);
    check(xg_spmm_i8(s.rows, s.cols, rp.get(), ci.get(), v.get(), dd.get(), d.cols, bit_width(d.bits), dout.get(),
                     xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

SparseCsrF32 csr_from_dense(const DenseMatrix& a) {
    SparseCsrF32 s;
    s.rows = a.rows;
    s.cols = a.cols;
    DevBuf<float> da(a.data);
    DevBuf<std::int32_t> drp(static_cast<std::size_t>(a.rows) + 1);
    int64_t nnz = 0;
    check(xg_csr_from_dense_count(da.get(), a.rows, a.cols, drp.get(), &nnz, xs()));
    DevBuf<std::int32_t> dci(static_cast<std::size_t>(nnz));
    DevBuf<float> dv(static_cast<std::size_t>(nnz));
    check(xg_csr_from_dense_fill(da.get(), a.rows, a.cols, drp.get(), dci.get(), dv.get(), xs()));
    s.row_ptr = drp.to_vector(drp.size());
    s.col_idx = dci.to_vector(nnz);
    s.values = dv.to_vector(nnz);
    return s;
}

DenseMatrix densify(const SparseCsrF32& s) {
    DenseMatrix out(s.rows, s.cols);
    DevBuf<std::int32_t> rp(s.row_ptr), ci(s.col_idx);
    DevBuf<float> v(s.values), dout(out.data.size());
    check(xg_densify(s.rows, s.cols, rp.get(), ci.get(), v.get(), dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

template <typename T>
SparseCsr<T> csr_transpose(const SparseCsr<T>& s) {
    SparseCsr<T> t;
    t.rows = s.cols;
    t.cols = s.rows;
    const std::size_t nnz = s.values.size();
    DevBuf<std::int32_t> rp(s.row_ptr), ci(s.col_idx), trp(static_cast<std::size_t>(s.cols) + 1), tci(nnz);
    DevBuf<T> v(s.values), tv(nnz);
    if constexpr (std::is_same_v<T, std::int8_t>)
        check(xg_csr_transpose_i8(s.rows, s.cols, rp.get(), ci.get(), v.get(), (int64_t)nnz, trp.get(), tci.get(),
                                  tv.get(), xs()));
    else
        check(xg_csr_transpose_f32(s.rows, s.cols, rp.get(), ci.get(), v.get(), (int64_t)nnz, trp.get(), tci.get(),
                                   tv.get(), xs()));
    t.row_ptr = trp.to_vector(trp.size());
    t.col_idx = tci.to_vector(nnz);
    t.values = tv.to_vector(nnz);
    return t;
}
template SparseCsr<float> csr_transpose(const SparseCsr<float>&);
template SparseCsr<std::int8_t> csr_transpose(const SparseCsr<std::int8_t>&);

QuantizedCsr quantize_csr(const SparseCsrF32& s, QuantBits bits, ScaleScheme scheme, RoundingMode rounding) {
    QuantizedCsr q;
    q.bits = bits;
    q.scales.scheme = scheme;
    q.matrix.rows = s.rows;
    q.matrix.cols = s.cols;
    q.matrix.row_ptr = s.row_ptr;
    q.matrix.col_idx = s.col_idx;
    const std::size_t nnz = s.values.size();
    const std::size_t ns = scheme == ScaleScheme::PerRow ? s.rows : scheme == ScaleScheme::PerColumn ? s.cols : 1;
    DevBuf<std::int32_t> rp(s.row_ptr), ci(s.col_idx);
    DevBuf<float> v(s.values);
    DevBuf<std::int8_t> qv(nnz);
    DevBuf<double> sc(ns);
    check(xg_quantize_csr(s.rows, s.cols, rp.get(), ci.get(), v.get(), (int64_t)nnz, bit_width(bits),
                          static_cast<int>(scheme), static_cast<int>(rounding), qv.get(), sc.get(), xs()));
    q.matrix.values = qv.to_vector(nnz);
    q.scales.values = sc.to_vector(ns);
    return q;
}

// -------------------------------------------------------------- pipeline.hpp
void XigemmConfig::validate() const {
    if (!(threshold > 0.0)) throw std::invalid_argument("XigemmConfig: threshold M must be positive");
    if (!(density_limit > 0.0) || density_limit > 1.0)
        throw std::invalid_argument("XigemmConfig: density limit must be in (0, 1]");
}

namespace {

xg_config cfg_c(const XigemmConfig& c) {
    xg_config x;
    x.bits = bit_width(c.bits);
    x.threshold = c.threshold;
    x.density_limit = c.density_limit;
    x.scheme = static_cast<int>(c.scheme);
    x.policy = static_cast<int>(c.policy);
    x.rounding = static_cast<int>(c.rounding);
    return x;
}

std::map<std::string, std::chrono::nanoseconds> timings_of(const xg_report& r) {
    using ns = std::chrono::nanoseconds;
    return {{"quant", ns((long long)r.ns_quant)},
            {"xxmm", ns((long long)r.ns_xxmm)},
            {"reduce", ns((long long)r.ns_reduce)},
            {"package", ns((long long)r.ns_package)}};
}

}  // namespace

DenseMatrix quantized_gemm_direct(const DenseMatrix& a, const DenseMatrix& b, const XigemmConfig& cfg) {
    cfg.validate();
    if (a.cols != b.rows) throw std::invalid_argument("quantized_gemm_direct: inner dimensions do not match");
    DenseMatrix out(a.rows, b.cols);
    const xg_config c = cfg_c(cfg);
    check(xg_gemm_direct_host(a.data.data(), b.data.data(), a.rows, a.cols, b.cols, &c, out.data.data()));
    return out;
}

DenseMatrix quantized_gemm_direct(const QuantizedMatrix& aq, const QuantizedMatrix& bq) {
    if (aq.cols != bq.rows) throw std::invalid_argument("gemm_int: inner dimensions do not match");
    DenseMatrix out(aq.rows, bq.cols);
    DevBuf<std::int8_t> da(aq.data), db(bq.data);
    DevBuf<double> sa(aq.scales.values), sb(bq.scales.values);
    DevBuf<float> dout(out.data.size());
    check(xg_gemm_direct_q(da.get(), static_cast<int>(aq.scales.scheme), sa.get(), db.get(),
                           static_cast<int>(bq.scales.scheme), sb.get(), aq.rows, aq.cols, bq.cols,
                           bit_width(aq.bits), bit_width(bq.bits), dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

DenseMatrix quantized_gemm_full_residual(const DenseMatrix& a, const DenseMatrix& b, const XigemmConfig& cfg) {
    cfg.validate();
    if (a.cols != b.rows) throw std::invalid_argument("xigemm: inner dimensions do not match");
    DenseMatrix out(a.rows, b.cols);
    const xg_config c = cfg_c(cfg);
    xg_report rep{};
    check(xg_xigemm_host(a.data.data(), b.data.data(), nullptr, 1.0f, 0.0f, a.rows, a.cols, b.cols, &c, 0,
                         out.data.data(), &rep));
    return out;
}

GemmReport xigemm(const DenseMatrix& a, const DenseMatrix& b, const DenseMatrix* c, float alpha, float beta,
                  const XigemmConfig& cfg) {
    if (c != nullptr && (c->rows != a.rows || c->cols != b.cols))
        throw std::invalid_argument("xigemm: C shape does not match the result");
    cfg.validate();
    if (a.cols != b.rows) throw std::invalid_argument("xigemm: inner dimensions do not match");
    GemmReport report;
    report.result = DenseMatrix(a.rows, b.cols);
    const xg_config xc = cfg_c(cfg);
    xg_report rep{};
    check(xg_xigemm_host(a.data.data(), b.data.data(), c ? c->data.data() : nullptr, alpha, beta, a.rows, a.cols,
                         b.cols, &xc, 1, report.result.data.data(), &rep));
    report.density_a = rep.density_a;
    report.density_b = rep.density_b;
    report.path = rep.path == XG_SPARSE_RESIDUAL ? GemmPath::SparseResidual : GemmPath::DenseResidual;
    report.timings = timings_of(rep);
    return report;
}

GemmReport xigemm(const DenseMatrix& a, const DenseMatrix& b, const XigemmConfig& cfg) {
    return xigemm(a, b, nullptr, 1.0f, 0.0f, cfg);
}

namespace {
std::pair<std::vector<float>, std::vector<float>> stats(const DenseMatrix& d, bool avg) {
    if (d.rows == 0 || d.cols == 0)
        throw std::invalid_argument(avg ? "get_avg_vectors: empty matrix" : "get_abs_min_vectors: empty matrix");
    DevBuf<float> dd(d.data), r(d.rows), c(d.cols);
    check(avg ? xg_avg_vectors(dd.get(), d.rows, d.cols, r.get(), c.get(), xs())
              : xg_abs_min_vectors(dd.get(), d.rows, d.cols, r.get(), c.get(), xs()));
    return {r.to_vector(d.rows), c.to_vector(d.cols)};
}
}  // namespace

std::pair<std::vector<float>, std::vector<float>> get_avg_vectors(const DenseMatrix& d) { return stats(d, true); }
std::pair<std::vector<float>, std::vector<float>> get_abs_min_vectors(const DenseMatrix& d) {
    return stats(d, false);
}

}  // namespace xigemm
