// gridio.hpp -- the wire formats on either side of the propagator path (SURVEY.md 8f,
// rank 2): the SFGD binary grid container (proj/include/sf/gridio.hpp:8-18) and the trace
// / coordinate CSV tables (proj/include/sf/sparse.hpp:97-104, proj/src/gridio.cpp:71-87).
// Files written here are byte-identical to the reference's for the same data.
#pragma once

#include <string>
#include <vector>

#include "sfb/sparse.hpp"

namespace sfb {

// ---- SFGD grids ------------------------------------------------------------------------
// layout (little-endian): "SFGD" | u8 rank | u8 dtype (0 = f64) | u16 0 | u32 extent[rank] |
// f64 payload, row-major
struct GridData {
    std::vector<long> shape;
    std::vector<double> data;
};
GridData read_grid(const std::string& path);
void write_grid(const std::string& path, const std::vector<long>& shape, const std::vector<double>& data);

// ---- trace tables: header "t,p0,p1,...", one row per time sample, %.17g values ---------
void write_traces_csv(const std::string& path, long nt, long npts, const std::vector<double>& traces,
                      double t0, double dt);
void write_traces_csv(const std::string& path, const SparseFunction& s, const std::vector<double>& times);
void read_traces_csv(const std::string& path, SparseFunction& s, std::vector<double>* times = nullptr);

// ---- point coordinates: header "x[,y[,z]]", one row per point --------------------------
std::vector<double> read_coords_csv(const std::string& path, std::size_t ndim);
void write_coords_csv(const std::string& path, const SparseFunction& s);

}  // namespace sfb
