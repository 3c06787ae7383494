// data.cpp -- Grid, dense fields and point clouds of the host layer (include/sfb/*.hpp).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sfb/function.hpp"
#include "sfb/sparse.hpp"
#include "sfb200.h"

namespace sfb {

void raise_status(int code, const std::string& message) {
    switch (code) {
    case SFB_ERR_PARAMETER: throw ParameterError(message);
    case SFB_ERR_STABILITY: throw StabilityError(message);
    case SFB_ERR_LOCATION: throw LocationError(message);
    case SFB_ERR_CAPABILITY: throw CapabilityError(message);
    case SFB_ERR_BINDING: throw BindingError(message);
    case SFB_ERR_ORDER: throw OrderError(message);
    default: throw Error(message);
    }
}

// ---- Grid (proj/include/sf/grid.hpp:32-47) --------------------------------------------

Grid::Grid(std::vector<long> shape, std::vector<double> spacing, std::vector<double> origin)
    : shape_(std::move(shape)), spacing_(std::move(spacing)), origin_(std::move(origin)) {
    if (shape_.empty() || shape_.size() > 3) throw ParameterError("grid rank must be 1, 2 or 3");
    if (spacing_.size() != shape_.size() || origin_.size() != shape_.size())
        throw ParameterError("grid shape/spacing/origin rank mismatch");
    for (std::size_t d = 0; d < shape_.size(); ++d) {
        if (shape_[d] < 2) throw ParameterError("grid extent must be >= 2 nodes");
        if (!(spacing_[d] > 0.0)) throw ParameterError("grid spacing must be positive");
    }
}

std::size_t Grid::points() const {
    std::size_t n = 1;
    for (long e : shape_) n *= std::size_t(e);
    return n;
}

// ---- fields (proj/include/sf/function.hpp:35-73,113-167) --------------------------------

void check_space_order(int space_order) {
    if (space_order < 2 || space_order % 2 != 0)
        throw OrderError("space order must be a positive even number");
}

FieldBase::FieldBase(std::string name, std::shared_ptr<const Grid> grid, int space_order,
                     std::vector<long> extents, std::vector<long> halos, bool has_time,
                     bool time_buffered, long time_slots)
    : name_(std::move(name)), grid_(std::move(grid)), space_order_(space_order),
      extents_(std::move(extents)), halos_(std::move(halos)), has_time_(has_time),
      time_buffered_(time_buffered), time_slots_(time_slots) {
    size_ = 1;
    for (std::size_t d = 0; d < extents_.size(); ++d) size_ *= std::size_t(padded_extent(int(d)));
    const std::size_t bytes = (size_ * sizeof(double) + 63) / 64 * 64;
    data_ = static_cast<double*>(std::aligned_alloc(64, bytes));
    if (!data_) throw std::bad_alloc();
    std::memset(data_, 0, bytes);
}

FieldBase::~FieldBase() { std::free(data_); }

long FieldBase::stride(int d) const {
    long s = 1;
    for (std::size_t k = std::size_t(d) + 1; k < extents_.size(); ++k) s *= padded_extent(int(k));
    return s;
}

std::size_t FieldBase::flat_index(const std::vector<long>& coords) const {
    if (coords.size() != extents_.size()) throw ParameterError(name_ + ": coordinate rank mismatch");
    std::size_t off = 0;
    for (std::size_t d = 0; d < coords.size(); ++d)
        off += std::size_t(coords[d] + halos_[d]) * std::size_t(stride(int(d)));
    return off;
}

void FieldBase::zero() { std::memset(data_, 0, size_ * sizeof(double)); }

std::shared_ptr<Function> Function::create(std::string name, std::shared_ptr<const Grid> grid,
                                           int space_order) {
    check_space_order(space_order);
    if (!grid) throw ParameterError("field needs a grid");
    std::vector<long> ext = grid->shape();
    std::vector<long> halos(ext.size(), space_order / 2);
    return std::shared_ptr<Function>(new Function(std::move(name), std::move(grid), space_order,
                                                  std::move(ext), std::move(halos), false, false,
                                                  0));
}

std::shared_ptr<TimeFunction> TimeFunction::create(std::string name,
                                                   std::shared_ptr<const Grid> grid,
                                                   int space_order, int time_order,
                                                   std::optional<long> save) {
    check_space_order(space_order);
    if (!grid) throw ParameterError("field needs a grid");
    if (time_order < 1) throw OrderError("time order must be >= 1");
    const long slots = save ? *save : time_order + 1;
    if (slots < time_order + 1)
        throw ParameterError("saved history must hold at least time_order+1 slots");
    std::vector<long> ext{slots};
    for (long s : grid->shape()) ext.push_back(s);
    std::vector<long> halos(ext.size(), space_order / 2);
    halos[0] = 0;
    auto tf = std::shared_ptr<TimeFunction>(
        new TimeFunction(std::move(name), std::move(grid), space_order, std::move(ext),
                         std::move(halos), true, !save.has_value(), slots));
    tf->time_order_ = time_order;
    return tf;
}

// ---- point clouds (proj/src/sparse.cpp:14-70) --------------------------------------------

std::shared_ptr<SparseFunction> SparseFunction::create(std::string name,
                                                       std::shared_ptr<const Grid> grid,
                                                       std::vector<double> coords, long nt) {
    if (!grid) throw ParameterError("point cloud '" + name + "': no grid given");
    const std::size_t rank = std::size_t(grid->ndim());
    if (coords.empty() || coords.size() % rank)
        throw ParameterError("point cloud '" + name + "': " + std::to_string(coords.size()) +
                             " coordinates do not form points of rank " + std::to_string(rank));
    if (nt < 1) throw ParameterError("point cloud '" + name + "': traces need at least one sample");
    std::shared_ptr<SparseFunction> cloud(
        new SparseFunction(std::move(name), std::move(grid), std::move(coords), nt));
    return cloud;
}

SparseFunction::SparseFunction(std::string name, std::shared_ptr<const Grid> grid,
                               std::vector<double> coords, long nt)
    : name_(std::move(name)), grid_(std::move(grid)), coords_(std::move(coords)),
      npoints_(long(coords_.size() / std::size_t(grid_->ndim()))), nt_(nt) {
    traces_.assign(std::size_t(nt_) * std::size_t(npoints_), 0.0);
    weights_.assign(std::size_t(npoints_) * std::size_t(corners()), 0.0);
}

void SparseFunction::locate() {
    if (located_) return;
    // the arithmetic lives behind the C-ABI (sfb_locate restates proj/src/sparse.cpp:36-70)
    sfb_plan_desc d{};
    d.ndim = grid_->ndim();
    for (int a = 0; a < d.ndim; ++a) {
        d.shape[a] = grid_->shape()[std::size_t(a)];
        d.spacing[a] = grid_->spacing()[std::size_t(a)];
    }
    std::vector<int64_t> base(std::size_t(npoints_) * std::size_t(d.ndim));
    int rc = sfb_locate(&d, grid_->origin().data(), npoints_, coords_.data(), base.data(),
                        weights_.data());
    if (rc != SFB_OK) raise_status(rc, name_ + " " + sfb_last_error(nullptr));
    base_.assign(base.begin(), base.end());
    located_ = true;
}

}  // namespace sfb
