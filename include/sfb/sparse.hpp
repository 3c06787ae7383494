// sparse.hpp -- off-lattice point clouds (sources, receivers).  Mirrors SparseFunction
// (proj/include/sf/sparse.hpp:30-95): coordinates [np][ndim], traces [nt][np], and after
// locate() the enclosing-cell table [np][ndim] plus multilinear weights [np][2^ndim]
// with axis 0 as the least-significant corner bit.  interpolate()/inject() of the
// reference return symbolic equations; here the operators apply them on the GPU.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "sfb/grid.hpp"

namespace sfb {

class SparseFunction {
public:
    static std::shared_ptr<SparseFunction> create(std::string name,
                                                  std::shared_ptr<const Grid> grid,
                                                  std::vector<double> coords, long nt);

    const std::string& name() const { return name_; }
    const std::shared_ptr<const Grid>& grid() const { return grid_; }
    long npoints() const { return npoints_; }
    long nt() const { return nt_; }
    int corners() const { return 1 << grid_->ndim(); }
    double coord(long p, std::size_t d) const { return coords_[p * grid_->ndim() + d]; }
    const std::vector<double>& coords() const { return coords_; }

    double& trace(long t, long p) { return traces_[std::size_t(t) * npoints_ + p]; }
    double trace(long t, long p) const { return traces_[std::size_t(t) * npoints_ + p]; }
    std::vector<double>& traces() { return traces_; }
    const std::vector<double>& traces() const { return traces_; }

    const std::vector<double>& weight_table() const { return weights_; }
    const std::vector<long>& base_table() const { return base_; }

    // resolves bases and weights; idempotent; LocationError when a point lies outside
    void locate();
    bool located() const { return located_; }

private:
    SparseFunction(std::string name, std::shared_ptr<const Grid> grid,
                   std::vector<double> coords, long nt);

    std::string name_;
    std::shared_ptr<const Grid> grid_;
    std::vector<double> coords_;
    long npoints_ = 0, nt_ = 0;
    std::vector<double> traces_, weights_;
    std::vector<long> base_;
    bool located_ = false;
};

}  // namespace sfb
