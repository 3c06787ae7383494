// model.cpp -- SeismicModel, build_damping, AcquisitionGeometry and the wavelets of the
// host layer.  Set-up arithmetic in f64 on the host, as in the reference
// (proj/src/model.cpp, proj/src/geometry.cpp, proj/include/sf/wavelet.hpp).
#include <algorithm>
#include <cmath>

#include "sfb/geometry.hpp"
#include "sfb/model.hpp"
#include "sfb200.h"

namespace sfb {

namespace {

// A rank-1..3 field seen as 3-D (unit leading axes), so every sweep below is one
// triple loop with the innermost axis contiguous.
struct View3 {
    long n[3] = {1, 1, 1};
    long stride[3] = {0, 0, 0};
    double* origin = nullptr;  // interior node (0,0,0)

    View3(const FieldBase& f) {
        const int nd = int(f.extents().size()), off = 3 - nd;
        std::vector<long> zero(std::size_t(nd), 0);
        origin = f.values() + f.flat_index(zero);
        for (int a = 0; a < nd; ++a) {
            n[off + a] = f.extents()[std::size_t(a)];
            stride[off + a] = f.stride(a);
        }
    }
    double* row(long i, long j) const { return origin + i * stride[0] + j * stride[1]; }
};

// per-axis table of the physical cell a padded node copies: clamp(i - nbl, 0, n - 1)
std::vector<long> clamp_table(long padded, long nbl, long physical) {
    std::vector<long> t(static_cast<std::size_t>(padded));
    for (long i = 0; i < padded; ++i) t[std::size_t(i)] = std::clamp(i - nbl, 0L, physical - 1);
    return t;
}

}  // namespace

// proj/src/model.cpp:35-56: separable sum over the axes of eta_max_d * ramp(w),
// w = (nbl - dist)/nbl for nodes closer than nbl to a face, eta_max_d = v_max ln(1000) /
// (nbl h_d); exactly zero in the physical interior.
std::shared_ptr<Function> build_damping(const std::shared_ptr<Grid>& grid, long nbl,
                                        double v_max, DampProfile profile, int space_order) {
    if (nbl < 0) throw ParameterError("build_damping: nbl must be >= 0");
    const std::vector<long>& shape = grid->shape();
    for (long e : shape)
        if (nbl >= (e + 1) / 2) throw ParameterError("build_damping: nbl must be < min(shape)/2");
    auto damp = Function::create("damp", grid, space_order);
    if (nbl == 0) return damp;
    const double gain = v_max * std::log(1000.0);
    // one profile per axis, then the sum
    std::vector<std::vector<double>> prof(shape.size());
    for (std::size_t d = 0; d < shape.size(); ++d) {
        const double eta_max = gain / (double(nbl) * grid->spacing()[d]);
        prof[d].assign(std::size_t(shape[d]), 0.0);
        for (long i = 0; i < shape[d]; ++i) {
            const long dist = std::min(i, shape[d] - 1 - i);
            if (dist >= nbl) continue;
            const double w = double(nbl - dist) / double(nbl);
            prof[d][std::size_t(i)] = eta_max * (profile == DampProfile::Linear ? w : w * w);
        }
    }
    const View3 v(*damp);
    const int off = 3 - int(shape.size());
    auto p = [&](int axis, long i) {  // profile of embedded axis `axis`
        return axis < off ? 0.0 : prof[std::size_t(axis - off)][std::size_t(i)];
    };
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < v.n[0]; ++i)
        for (long j = 0; j < v.n[1]; ++j) {
            double* row = v.row(i, j);
            // same left-to-right sum over the axes as the reference
            for (long l = 0; l < v.n[2]; ++l) {
                double eta = 0.0;
                if (off <= 0) eta += p(0, i);
                if (off <= 1) eta += p(1, j);
                eta += p(2, l);
                row[l] = eta;
            }
        }
    return damp;
}

// proj/src/model.cpp:58-78
SeismicModel::SeismicModel(std::vector<long> shape, std::vector<double> spacing,
                           std::vector<double> origin, const std::vector<double>& velocity,
                           long nbl, int space_order, DampProfile profile)
    : box_(std::move(shape)), h_(std::move(spacing)), corner_(std::move(origin)),
      layer_(nbl), order_(space_order) {
    if (box_.empty() || box_.size() != h_.size() || box_.size() != corner_.size())
        throw ParameterError("SeismicModel: rank mismatch");
    if (layer_ < 0) throw ParameterError("SeismicModel: nbl must be >= 0");
    std::vector<long> padded(box_);
    std::vector<double> porigin(corner_);
    for (std::size_t d = 0; d < box_.size(); ++d) {
        padded[d] += 2 * layer_;
        porigin[d] -= double(layer_) * h_[d];
    }
    padded_grid_ = std::make_shared<Grid>(padded, h_, porigin);
    slowness2_ = Function::create("m", padded_grid_, order_);
    set_velocity(velocity);
    absorber_ = build_damping(padded_grid_, layer_, vel_hi_, profile, order_);
}

// edge-clamped extension p = clamp(idx - nbl, 0, n-1), proj/src/model.cpp:92-100
template <typename Fn>
void SeismicModel::extend_into_layer(Fn&& value_of_physical_cell) {
    const View3 v(*slowness2_);
    const int off = 3 - int(box_.size());
    long pn[3] = {1, 1, 1};
    std::vector<long> tab[3];
    for (int a = 0; a < 3; ++a) {
        if (a >= off) pn[a] = box_[std::size_t(a - off)];
        tab[a] = clamp_table(v.n[a], a >= off ? layer_ : 0, pn[a]);
    }
#pragma omp parallel for collapse(2) schedule(static)
    for (long i = 0; i < v.n[0]; ++i)
        for (long j = 0; j < v.n[1]; ++j) {
            double* row = v.row(i, j);
            const std::size_t base =
                (std::size_t(tab[0][std::size_t(i)]) * std::size_t(pn[1]) +
                 std::size_t(tab[1][std::size_t(j)])) * std::size_t(pn[2]);
            for (long l = 0; l < v.n[2]; ++l)
                row[l] = value_of_physical_cell(base + std::size_t(tab[2][std::size_t(l)]));
        }
}

void SeismicModel::set_velocity(const std::vector<double>& velocity) {
    std::size_t n = 1;
    for (long e : box_) n *= std::size_t(e);
    if (velocity.size() != n) throw ParameterError("SeismicModel: velocity size does not match shape");
    for (double v : velocity)
        if (!(v > 0.0)) throw ParameterError("SeismicModel: velocity must be positive");
    auto [lo, hi] = std::minmax_element(velocity.begin(), velocity.end());
    vel_lo_ = *lo;
    vel_hi_ = *hi;
    extend_into_layer([&](std::size_t flat) { return 1.0 / (velocity[flat] * velocity[flat]); });
}

// proj/src/model.cpp:103-111 (arithmetic behind the C-ABI)
double SeismicModel::critical_dt(int space_order, double gamma) const {
    double out = 0;
    int rc = sfb_critical_dt(int(box_.size()), h_.data(), vel_hi_, space_order, &out);
    if (rc == SFB_ERR_PARAMETER) {
        check_space_order(space_order);
        throw OrderError("critical_dt: unsupported space order");
    }
    if (rc != SFB_OK) raise_status(rc, sfb_last_error(nullptr));
    return gamma * out;
}

std::vector<double> SeismicModel::physical_m() const {
    const View3 v(*slowness2_);
    const int off = 3 - int(box_.size());
    long pn[3] = {1, 1, 1}, pad[3] = {0, 0, 0};
    for (int a = off; a < 3; ++a) {
        pn[a] = box_[std::size_t(a - off)];
        pad[a] = layer_;
    }
    std::vector<double> out(std::size_t(pn[0]) * std::size_t(pn[1]) * std::size_t(pn[2]));
    for (long i = 0; i < pn[0]; ++i)
        for (long j = 0; j < pn[1]; ++j) {
            const double* row = v.row(i + pad[0], j + pad[1]) + pad[2];
            std::copy(row, row + pn[2], out.begin() + (std::size_t(i) * pn[1] + j) * pn[2]);
        }
    return out;
}

// proj/src/model.cpp:124-147: values stored verbatim, velocity statistics through sqrt
void SeismicModel::set_physical_m(const std::vector<double>& m_values) {
    std::size_t n = 1;
    for (long e : box_) n *= std::size_t(e);
    if (m_values.size() != n) throw ParameterError("SeismicModel: m size does not match shape");
    for (double mv : m_values)
        if (!(mv > 0.0)) throw ParameterError("SeismicModel: m must be positive");
    vel_lo_ = vel_hi_ = 1.0 / std::sqrt(m_values[0]);
    for (double mv : m_values) {
        const double v = 1.0 / std::sqrt(mv);
        vel_lo_ = std::min(vel_lo_, v);
        vel_hi_ = std::max(vel_hi_, v);
    }
    extend_into_layer([&](std::size_t flat) { return m_values[flat]; });
}

// ---- wavelets (proj/include/sf/wavelet.hpp:12-35) ----------------------------------------

double ricker_value(double f0, double t) {
    const double tau = t - 1.0 / f0;
    const double a = M_PI * M_PI * f0 * f0 * tau * tau;
    return (1.0 - 2.0 * a) * std::exp(-a);
}

std::vector<double> ricker(double f0, double t0, double dt, long nt) {
    if (!(f0 > 0.0)) throw ParameterError("ricker: f0 must be positive");
    if (nt < 1 || !(dt > 0.0)) throw ParameterError("ricker: bad time axis");
    std::vector<double> w(std::size_t(nt), 0.0);
    for (long i = 0; i < nt; ++i) w[std::size_t(i)] = ricker_value(f0, t0 + double(i) * dt);
    return w;
}

double dgauss4_value(double fp, double t) {
    double a = 2.0 * M_PI * fp;
    a = a * a / 8.0;
    const double tau = t - 2.0 / fp;
    const double x2 = a * tau * tau;
    return (16.0 * x2 * x2 - 48.0 * x2 + 12.0) * std::exp(-x2) / 12.0;
}

// ---- geometry (proj/src/geometry.cpp:10-34) -----------------------------------------------

AcquisitionGeometry::AcquisitionGeometry(const SeismicModel& model, std::vector<double> src_coords,
                                         std::vector<double> rec_coords, double t0, double tn,
                                         double dt, double f0)
    : axis_{t0, tn, dt, 0}, peak_freq_(f0) {
    if (!(dt > 0.0) || !(tn > t0)) throw ParameterError("AcquisitionGeometry: bad time axis");
    if (dt > model.critical_dt() * (1.0 + 1e-12))
        throw StabilityError("AcquisitionGeometry: dt exceeds the stable limit " +
                             std::to_string(model.critical_dt()));
    const std::size_t rank = model.grid()->shape().size();
    if (src_coords.empty() || src_coords.size() % rank != 0 || rec_coords.empty() ||
        rec_coords.size() % rank != 0)
        throw ParameterError("AcquisitionGeometry: coordinate list rank mismatch");
    count_[0] = long(src_coords.size() / rank);
    count_[1] = long(rec_coords.size() / rank);
    axis_.nt = long(std::floor((tn - t0) / dt)) + 1;
    cloud_[0] = SparseFunction::create("src", model.grid(), std::move(src_coords), axis_.nt);
    cloud_[1] = SparseFunction::create("rec", model.grid(), std::move(rec_coords), axis_.nt);
    cloud_[0]->locate();
    cloud_[1]->locate();
    const std::vector<double> w = ricker(f0, t0, dt, axis_.nt);
    for (long t = 0; t < axis_.nt; ++t)
        for (long p = 0; p < count_[0]; ++p) cloud_[0]->trace(t, p) = w[std::size_t(t)];
}

}  // namespace sfb
