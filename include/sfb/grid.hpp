// grid.hpp -- structured Cartesian grid (mirrors Grid, proj/include/sf/grid.hpp:30-71;
// the symbolic Dim machinery of the reference is not part of the propagator path).
#pragma once

#include <cstddef>
#include <vector>

#include "sfb/error.hpp"

namespace sfb {

class Grid {
public:
    // shape counts nodes per axis; node i of axis d sits at origin[d] + i*spacing[d]
    Grid(std::vector<long> shape, std::vector<double> spacing, std::vector<double> origin);

    int ndim() const { return int(shape_.size()); }
    const std::vector<long>& shape() const { return shape_; }
    const std::vector<double>& spacing() const { return spacing_; }
    const std::vector<double>& origin() const { return origin_; }
    double extent(int d) const { return double(shape_[d] - 1) * spacing_[d]; }
    std::size_t points() const;

private:
    std::vector<long> shape_;
    std::vector<double> spacing_, origin_;
};

}  // namespace sfb
