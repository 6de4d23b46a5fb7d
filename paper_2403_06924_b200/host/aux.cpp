// xigemm drop-in: the reference's evaluation-support headers (metrics.hpp,
// random_matrix.hpp, calibrate.hpp, qr.hpp).  These sit outside the hot path
// (OUT OF SCOPE); they are provided so callers and the
// reference's own test suites link unchanged.  Matrix products inside them go
// through the GPU entry points; input generation and error norms are host code.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <stdexcept>
#include <thread>

#include "xigemm/calibrate.hpp"
#include "xigemm_c.h"
#include "xigemm/metrics.hpp"
#include "xigemm/qr.hpp"
#include "xigemm/random_matrix.hpp"
#include "xigemm/sparse.hpp"

#include <cuda_runtime.h>

namespace xigemm {

// ---------------------------------------------------------------- metrics
ErrorReport frobenius_error(const DenseMatrix& x_ref, const DenseMatrix& x) {
    if (!x_ref.same_shape(x)) throw std::invalid_argument("frobenius_error: shape mismatch");
    double diff2 = 0.0, ref2 = 0.0, worst = 0.0;
    for (std::size_t i = 0; i < x_ref.data.size(); ++i) {
        const double r = x_ref.data[i];
        const double d = r - static_cast<double>(x.data[i]);
        diff2 += d * d;
        ref2 += r * r;
        if (std::fabs(r) >= 1e-12) worst = std::max(worst, std::fabs(d) / std::fabs(r));
    }
    ErrorReport rep;
    rep.e_r = std::sqrt(diff2);
    rep.max_elem_rel = worst;
    const double norm = std::sqrt(ref2);
    rep.ref_norm_zero = !(norm > 0.0);
    rep.e_delta = rep.ref_norm_zero ? rep.e_r : rep.e_r / norm;
    return rep;
}

// ---------------------------------------------------------- random_matrix
std::uint64_t SplitMix64::next() {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double SplitMix64::next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

DistributionSpec DistributionSpec::uniform01(std::uint64_t s) { return {DistKind::Uniform01, 0.0, 0.0, s}; }
DistributionSpec DistributionSpec::normal(double mean, double sd, std::uint64_t s) { return {DistKind::Normal, mean, sd, s}; }
DistributionSpec DistributionSpec::exponential(double rate, std::uint64_t s) { return {DistKind::Exponential, rate, 0.0, s}; }
DistributionSpec DistributionSpec::poisson(double rate, std::uint64_t s) { return {DistKind::Poisson, rate, 0.0, s}; }
DistributionSpec DistributionSpec::chi_square(int dof, std::uint64_t s) {
    return {DistKind::ChiSquare, static_cast<double>(dof), 0.0, s};
}

void DistributionSpec::validate() const {
    if (kind == DistKind::Normal && !(param2 > 0.0)) throw std::invalid_argument("normal: stddev must be positive");
    if ((kind == DistKind::Exponential || kind == DistKind::Poisson) && !(param1 > 0.0))
        throw std::invalid_argument("rate must be positive");
    if (kind == DistKind::ChiSquare && !(param1 >= 1.0)) throw std::invalid_argument("chi_square: dof must be >= 1");
}

namespace {
double gauss(SplitMix64& g) {  // Box-Muller, cosine branch (stream layout pinned)
    const double u1 = 1.0 - g.next_unit();
    const double u2 = g.next_unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
}
double draw(SplitMix64& g, const DistributionSpec& s) {
    switch (s.kind) {
        case DistKind::Uniform01: return g.next_unit();
        case DistKind::Normal: return s.param1 + s.param2 * gauss(g);
        case DistKind::Exponential: return -std::log(1.0 - g.next_unit()) / s.param1;
        case DistKind::Poisson: {  // Knuth's product method
            const double limit = std::exp(-s.param1);
            double p = 1.0;
            int k = 0;
            do {
                ++k;
                p *= g.next_unit();
            } while (p > limit);
            return static_cast<double>(k - 1);
        }
        case DistKind::ChiSquare: {
            double acc = 0.0;
            for (int i = 0; i < static_cast<int>(s.param1); ++i) {
                const double z = gauss(g);
                acc += z * z;
            }
            return acc;
        }
    }
    return 0.0;
}
}  // namespace

DenseMatrix generate(const DistributionSpec& spec, int rows, int cols) {
    spec.validate();
    if (rows < 1 || cols < 1) throw std::invalid_argument("generate: rows and cols must be >= 1");
    SplitMix64 g(spec.seed);
    DenseMatrix m(rows, cols);
    for (float& v : m.data) v = static_cast<float>(draw(g, spec));
    return m;
}

// -------------------------------------------------------------- calibrate
double calibrate_eta_from_model(const CostModel& model) {
    constexpr double kMin = 1.0 / 1024.0;
    if (model(1.0) <= 1.0) return 1.0;
    if (model(kMin) >= 1.0) return kMin;
    double lo = kMin, hi = 1.0;
    for (int it = 0; it < 20; ++it) {
        const double mid = 0.5 * (lo + hi);
        (model(mid) <= 1.0 ? lo : hi) = mid;
    }
    return 0.5 * (lo + hi);
}

std::string machine_fingerprint() {
    std::string cpu = "unknown-cpu";
    std::ifstream info("/proc/cpuinfo");
    for (std::string line; std::getline(info, line);) {
        if (line.rfind("model name", 0) == 0) {
            const auto colon = line.find(':');
            if (colon != std::string::npos && colon + 2 <= line.size()) cpu = line.substr(colon + 2);
            break;
        }
    }
    std::string gpu = "no-gpu";
    cudaDeviceProp prop{};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess) gpu = prop.name;
    else cudaGetLastError();
    return gpu + " / " + cpu + " / " + std::to_string(std::thread::hardware_concurrency()) + " threads";
}

// calibrate.cpp:68-100 on the B200: the tcgen05 gemm_int against the CSR
// spmm_int, CUDA-event timed on the device by xg_calibrate_eta (no PCIe or
// host work inside the timings).
EtaCalibration calibrate_eta(int size, QuantBits bits, std::uint64_t seed) {
    if (size < 8) throw std::invalid_argument("calibrate_eta: size too small to time");
    EtaCalibration cal;
    cal.fingerprint = machine_fingerprint();
    double eta = 0.0, ptc = 0.0, psp = 0.0;
    int reps = 0;
    const xg_status st = xg_calibrate_eta(size, bits == QuantBits::Int4 ? 4 : 8, seed, 0, &eta, &reps, &ptc, &psp);
    if (st == XG_EINVAL) throw std::invalid_argument(xg_last_error());
    if (st != XG_OK) throw std::runtime_error(xg_last_error());
    cal.eta = eta;
    cal.repetitions = reps;
    return cal;
}

// --------------------------------------------------------------------- qr
MultiplyBackend MultiplyBackend::float_reference() { return MultiplyBackend{}; }
MultiplyBackend MultiplyBackend::direct_quant(const XigemmConfig& cfg) { return {Kind::DirectQuant, cfg}; }
MultiplyBackend MultiplyBackend::full_residual(const XigemmConfig& cfg) { return {Kind::FullResidual, cfg}; }
MultiplyBackend MultiplyBackend::sparse_residual(const XigemmConfig& cfg) { return {Kind::SparseResidual, cfg}; }

DenseMatrix MultiplyBackend::multiply(const DenseMatrix& a, const DenseMatrix& b) const {
    switch (kind) {
        case Kind::DirectQuant: return quantized_gemm_direct(a, b, cfg);
        case Kind::FullResidual: return quantized_gemm_full_residual(a, b, cfg);
        case Kind::SparseResidual: return xigemm(a, b, cfg).result;
        case Kind::FloatReference: break;
    }
    return gemm_f32(a, b);
}

// Householder QR: reflectors and triangularisation in float with fp64 dot
// products (host), Q accumulated through the backend's GPU multiply.
QrResult householder_qr(const DenseMatrix& a, const MultiplyBackend& backend) {
    if (a.rows < a.cols) throw std::invalid_argument("householder_qr: requires rows >= cols");
    const int m = a.rows, n = a.cols;
    DenseMatrix r = a, q;
    bool have_q = false;
    std::vector<double> v(m);
    for (int k = 0; k < std::min(n, m - 1); ++k) {
        double nrm2 = 0.0;
        for (int i = k; i < m; ++i) nrm2 += static_cast<double>(r.at(i, k)) * r.at(i, k);
        if (nrm2 == 0.0) continue;
        const double x0 = r.at(k, k);
        const double alpha = -std::copysign(std::sqrt(nrm2), x0);
        v[k] = x0 - alpha;
        for (int i = k + 1; i < m; ++i) v[i] = r.at(i, k);
        double vv = 0.0;
        for (int i = k; i < m; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        for (int j = k; j < n; ++j) {
            double dot = 0.0;
            for (int i = k; i < m; ++i) dot += v[i] * r.at(i, j);
            const double f = 2.0 * dot / vv;
            for (int i = k; i < m; ++i) r.at(i, j) = static_cast<float>(r.at(i, j) - f * v[i]);
        }
        DenseMatrix h = DenseMatrix::identity(m);
        for (int i = k; i < m; ++i)
            for (int j = k; j < m; ++j) h.at(i, j) = static_cast<float>(h.at(i, j) - 2.0 * v[i] * v[j] / vv);
        if (have_q) {
            q = backend.multiply(q, h);
        } else {
            q = std::move(h);
            have_q = true;
        }
    }
    if (!have_q) q = DenseMatrix::identity(m);
    return QrResult{std::move(q), std::move(r)};
}

std::vector<QrCell> qr_error_table(const std::vector<int>& sizes, const std::vector<DistributionSpec>& specs,
                                   const std::vector<std::pair<std::string, MultiplyBackend>>& backends) {
    if (sizes.empty() || specs.empty() || backends.empty()) throw std::invalid_argument("qr_error_table: empty inputs");
    std::vector<QrCell> cells;
    for (int size : sizes)
        for (const DistributionSpec& spec : specs) {
            const DenseMatrix a = generate(spec, size, size);
            for (const auto& [label, backend] : backends) {
                const QrResult f = householder_qr(a, backend);
                QrCell cell;
                cell.size = size;
                cell.dist = spec.kind;
                cell.bits = backend.cfg.bits;
                cell.method = label;
                cell.error = frobenius_error(a, backend.multiply(f.q, f.r));
                cells.push_back(std::move(cell));
            }
        }
    return cells;
}

}  // namespace xigemm
