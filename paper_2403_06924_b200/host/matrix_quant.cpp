// xigemm drop-in: matrix.hpp and quantize.hpp.  Containers and scalar helpers
// are host code; every matrix computation runs on the B200 via the C-ABI.
// Reference: proj/src/matrix.cpp, proj/src/quantize.cpp.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <utility>

#include "dev.hpp"
#include "xigemm/matrix.hpp"
#include "xigemm/quantize.hpp"

namespace xigemm {

using detail::check;
using detail::DevBuf;
using detail::xs;

namespace {
void require_dims(int r, int c) {
    if (r < 1 || c < 1) throw std::invalid_argument("matrix dimensions must be >= 1");
}
}  // namespace

// ---------------------------------------------------------------- matrix.hpp
DenseMatrix::DenseMatrix(int r, int c) : rows(r), cols(c) {
    require_dims(r, c);
    data.assign(static_cast<std::size_t>(r) * c, 0.0f);
}

DenseMatrix DenseMatrix::from_data(int r, int c, std::vector<float> values) {
    require_dims(r, c);
    if (values.size() != static_cast<std::size_t>(r) * c)
        throw std::invalid_argument("data length does not match rows*cols");
    DenseMatrix m;
    m.rows = r;
    m.cols = c;
    m.data = std::move(values);
    if (!m.all_finite()) throw std::invalid_argument("matrix entries must be finite");
    return m;
}

DenseMatrix DenseMatrix::identity(int n) {
    DenseMatrix m(n, n);
    for (int i = 0; i < n; ++i) m.at(i, i) = 1.0f;
    return m;
}

// Container invariants checked on the host data the caller handed us (the
// pipeline re-checks on device inside K1).
bool DenseMatrix::all_finite() const {
    return std::all_of(data.begin(), data.end(), [](float v) { return std::isfinite(v); });
}

float DenseMatrix::max_abs() const {
    float m = 0.0f;
    for (float v : data) m = std::fabs(v) > m ? std::fabs(v) : m;
    return m;
}

IntMatrix::IntMatrix(int r, int c) : rows(r), cols(c) {
    require_dims(r, c);
    data.assign(static_cast<std::size_t>(r) * c, 0);
}

IntMatrix IntMatrix::transposed() const {
    IntMatrix t(cols, rows);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) t.at(j, i) = at(i, j);
    return t;
}

DenseMatrix gemm_f32(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols != b.rows) throw std::invalid_argument("gemm_f32: inner dimensions do not match");
    DenseMatrix c(a.rows, b.cols);
    DevBuf<float> da(a.data), db(b.data), dc(c.data.size());
    check(xg_gemm_f32(da.get(), db.get(), a.rows, a.cols, b.cols, dc.get(), xs()));
    dc.download(c.data.data(), c.data.size());
    return c;
}

DenseMatrix& axpby_inplace(DenseMatrix& d, float alpha, const DenseMatrix& c, float beta) {
    if (!d.same_shape(c)) throw std::invalid_argument("axpby_inplace: shape mismatch");
    DevBuf<float> dd(d.data), dc(c.data);
    check(xg_axpby(dd.get(), alpha, dc.get(), beta, (int64_t)d.data.size(), xs()));
    dd.download(d.data.data(), d.data.size());
    return d;
}

DenseMatrix subtract(const DenseMatrix& a, const DenseMatrix& b) {
    if (!a.same_shape(b)) throw std::invalid_argument("subtract: shape mismatch");
    DenseMatrix r(a.rows, a.cols);
    DevBuf<float> da(a.data), db(b.data), dr(r.data.size());
    check(xg_subtract(da.get(), db.get(), dr.get(), (int64_t)a.data.size(), xs()));
    dr.download(r.data.data(), r.data.size());
    return r;
}

DenseMatrix& add_inplace(DenseMatrix& d, const DenseMatrix& x) {
    if (!d.same_shape(x)) throw std::invalid_argument("add_inplace: shape mismatch");
    DevBuf<float> dd(d.data), dx(x.data);
    check(xg_add_inplace(dd.get(), dx.get(), (int64_t)d.data.size(), xs()));
    dd.download(d.data.data(), d.data.size());
    return d;
}

// -------------------------------------------------------------- quantize.hpp
ScaleFactors ScaleFactors::per_tensor(double lambda) { return ScaleFactors{ScaleScheme::PerTensor, {lambda}}; }

void ScaleFactors::validate(int rows, int cols) const {
    const std::size_t want = scheme == ScaleScheme::PerRow      ? static_cast<std::size_t>(rows)
                             : scheme == ScaleScheme::PerColumn ? static_cast<std::size_t>(cols)
                                                                : 1;
    if (values.size() != want) throw std::invalid_argument("ScaleFactors: value count does not match scheme");
    for (double v : values)
        if (!(v > 0.0) || !std::isfinite(v))
            throw std::invalid_argument("ScaleFactors: scales must be positive and finite");
}

QuantizedMatrix QuantizedMatrix::from_ints(int rows, int cols, std::vector<std::int8_t> ints,
                                           QuantBits bits, ScaleFactors scales,
                                           RoundingMode rounding) {
    if (ints.size() != static_cast<std::size_t>(rows) * cols)
        throw std::invalid_argument("QuantizedMatrix: data length does not match rows*cols");
    scales.validate(rows, cols);
    const std::int32_t qmax = quant_max(bits);
    for (std::int8_t v : ints)
        if (v < -qmax || v > qmax) throw std::invalid_argument("QuantizedMatrix: entry outside quantized range");
    QuantizedMatrix q;
    q.rows = rows;
    q.cols = cols;
    q.data = std::move(ints);
    q.bits = bits;
    q.scales = std::move(scales);
    q.rounding = rounding;
    return q;
}

QuantizedMatrix QuantizedMatrix::transposed() const {
    QuantizedMatrix t;
    t.rows = cols;
    t.cols = rows;
    t.bits = bits;
    t.rounding = rounding;
    t.scales = scales;
    if (scales.scheme == ScaleScheme::PerRow) t.scales.scheme = ScaleScheme::PerColumn;
    else if (scales.scheme == ScaleScheme::PerColumn) t.scales.scheme = ScaleScheme::PerRow;
    t.data.resize(data.size());
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) t.data[static_cast<std::size_t>(j) * rows + i] = at(i, j);
    return t;
}

double compute_scale(double max_abs, QuantBits bits) {
    if (!(max_abs >= 0.0) || !std::isfinite(max_abs))
        throw std::invalid_argument("compute_scale: max_abs must be finite and nonnegative");
    return max_abs == 0.0 ? 1.0 : static_cast<double>(quant_max(bits)) / max_abs;
}

// Scalar rule (quantize.cpp:13-24); the kernels carry the same rule on device.
std::int32_t quantize_scalar(double a, double lambda, std::int32_t qmax, RoundingMode mode) {
    double t = a * lambda;
    if (mode == RoundingMode::Floor) t += std::copysign(4.0 * DBL_EPSILON * std::fabs(t), t);
    long long q;
    if (!(std::fabs(t) < 9223372036854775808.0)) q = LLONG_MIN;  // x86-64 conversion result
    else q = mode == RoundingMode::Floor ? static_cast<long long>(std::trunc(t)) : std::llround(t);
    return static_cast<std::int32_t>(std::clamp<long long>(q, -qmax, qmax));
}

int gemm_int_max_inner(QuantBits bits) { return xg_gemm_max_inner(bit_width(bits)); }

namespace {
std::size_t nscales(ScaleScheme s, int rows, int cols) {
    return s == ScaleScheme::PerRow ? rows : s == ScaleScheme::PerColumn ? cols : 1;
}
}  // namespace

QuantizedMatrix quantize(const DenseMatrix& a, QuantBits bits, ScaleScheme scheme,
                         RoundingMode rounding) {
    require_dims(a.rows, a.cols);
    QuantizedMatrix q;
    q.rows = a.rows;
    q.cols = a.cols;
    q.bits = bits;
    q.rounding = rounding;
    q.scales.scheme = scheme;
    DevBuf<float> da(a.data);
    DevBuf<std::int8_t> dq(a.data.size());
    DevBuf<double> ds(nscales(scheme, a.rows, a.cols));
    check(xg_quantize(da.get(), a.rows, a.cols, bit_width(bits), static_cast<int>(scheme),
                      static_cast<int>(rounding), dq.get(), ds.get(), xs()));
    q.data = dq.to_vector(a.data.size());
    q.scales.values = ds.to_vector(ds.size());
    return q;
}

QuantizedMatrix quantize_with_scales(const DenseMatrix& a, QuantBits bits, ScaleFactors scales,
                                     RoundingMode rounding) {
    scales.validate(a.rows, a.cols);
    QuantizedMatrix q;
    q.rows = a.rows;
    q.cols = a.cols;
    q.bits = bits;
    q.rounding = rounding;
    DevBuf<float> da(a.data);
    DevBuf<double> ds(scales.values);
    DevBuf<std::int8_t> dq(a.data.size());
    check(xg_quantize_with_scales(da.get(), a.rows, a.cols, bit_width(bits), static_cast<int>(scales.scheme),
                                  ds.get(), static_cast<int>(rounding), dq.get(), xs()));
    q.data = dq.to_vector(a.data.size());
    q.scales = std::move(scales);
    return q;
}

DenseMatrix dequantize(const QuantizedMatrix& q) {
    DenseMatrix out(q.rows, q.cols);
    DevBuf<std::int8_t> dq(q.data);
    DevBuf<double> ds(q.scales.values);
    DevBuf<float> dout(out.data.size());
    check(xg_dequantize(dq.get(), q.rows, q.cols, static_cast<int>(q.scales.scheme), ds.get(), dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

DenseMatrix residual(const DenseMatrix& a, const QuantizedMatrix& q) {
    if (a.rows != q.rows || a.cols != q.cols) throw std::invalid_argument("residual: shape mismatch");
    DenseMatrix out(q.rows, q.cols);
    DevBuf<float> da(a.data), dout(out.data.size());
    DevBuf<std::int8_t> dq(q.data);
    DevBuf<double> ds(q.scales.values);
    check(xg_residual(da.get(), dq.get(), q.rows, q.cols, static_cast<int>(q.scales.scheme), ds.get(),
                      dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

DenseMatrix dequant_product(const IntMatrix& p, const ScaleFactors& scales_a, const ScaleFactors& scales_b) {
    if (scales_a.scheme == ScaleScheme::PerColumn)
        throw std::invalid_argument("dequant_product: left scales must be PerTensor or PerRow");
    if (scales_b.scheme == ScaleScheme::PerRow)
        throw std::invalid_argument("dequant_product: right scales must be PerTensor or PerColumn");
    scales_a.validate(p.rows, 1);
    scales_b.validate(1, p.cols);
    DenseMatrix out(p.rows, p.cols);
    DevBuf<std::int32_t> dp(p.data);
    DevBuf<double> sa(scales_a.values), sb(scales_b.values);
    DevBuf<float> dout(out.data.size());
    check(xg_dequant_product(dp.get(), p.rows, p.cols, static_cast<int>(scales_a.scheme), sa.get(),
                             static_cast<int>(scales_b.scheme), sb.get(), dout.get(), xs()));
    dout.download(out.data.data(), out.data.size());
    return out;
}

IntMatrix gemm_int(const QuantizedMatrix& a, const QuantizedMatrix& b) {
    if (a.cols != b.rows) throw std::invalid_argument("gemm_int: inner dimensions do not match");
    const int limit = std::min(gemm_int_max_inner(a.bits), gemm_int_max_inner(b.bits));
    if (a.cols > limit) throw std::invalid_argument("gemm_int: inner dimension permits 32-bit overflow");
    IntMatrix c(a.rows, b.cols);
    DevBuf<std::int8_t> da(a.data), db(b.data);
    DevBuf<std::int32_t> dc(c.data.size());
    check(xg_gemm_i8(da.get(), db.get(), a.rows, a.cols, b.cols, bit_width(a.bits), bit_width(b.bits), dc.get(),
                     xs()));
    dc.download(c.data.data(), c.data.size());
    return c;
}

}  // namespace xigemm
