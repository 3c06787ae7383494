// gridio.cpp -- SFGD grid container and trace / coordinate CSV tables of the host layer.
// Formats follow proj/src/gridio.cpp:26-87 and proj/src/sparse.cpp:152-229 byte for byte.
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "sfb/gridio.hpp"

namespace sfb {

namespace {

std::array<unsigned char, 4> le32(uint32_t v) {
    return {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
            static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
}

std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

}  // namespace

void write_grid(const std::string& path, const std::vector<long>& shape,
                const std::vector<double>& data) {
    if (shape.empty() || shape.size() > 255) throw ParameterError("write_grid: bad rank");
    std::size_t n = 1;
    for (long e : shape) {
        if (e < 1) throw ParameterError("write_grid: bad extent");
        n *= std::size_t(e);
    }
    if (n != data.size()) throw ParameterError("write_grid: shape/data mismatch");
    std::ofstream os(path, std::ios::binary);
    if (!os) throw ParameterError("write_grid: cannot open " + path);
    const unsigned char head[8] = {'S', 'F', 'G', 'D', static_cast<unsigned char>(shape.size()),
                                   0, 0, 0};
    os.write(reinterpret_cast<const char*>(head), 8);
    for (long e : shape) {
        const auto b = le32(uint32_t(e));
        os.write(reinterpret_cast<const char*>(b.data()), 4);
    }
    os.write(reinterpret_cast<const char*>(data.data()), std::streamsize(n * sizeof(double)));
    if (!os) throw ParameterError("write_grid: write failed for " + path);
}

GridData read_grid(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw ParameterError("read_grid: cannot open " + path);
    unsigned char head[8];
    is.read(reinterpret_cast<char*>(head), 8);
    if (!is || std::memcmp(head, "SFGD", 4) != 0)
        throw ParameterError("read_grid: bad magic in " + path);
    if (head[4] == 0 || head[5] != 0)
        throw ParameterError("read_grid: unsupported header in " + path);
    GridData g;
    std::size_t n = 1;
    for (int d = 0; d < head[4]; ++d) {
        unsigned char b[4];
        is.read(reinterpret_cast<char*>(b), 4);
        if (!is) throw ParameterError("read_grid: truncated header in " + path);
        const uint32_t e = uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 |
                           uint32_t(b[3]) << 24;
        g.shape.push_back(long(e));
        n *= e;
    }
    g.data.resize(n);
    is.read(reinterpret_cast<char*>(g.data.data()), std::streamsize(n * sizeof(double)));
    if (!is) throw ParameterError("read_grid: truncated payload in " + path);
    return g;
}

// proj/src/gridio.cpp:71-87 (stream precision 17, times t0 + t*dt)
void write_traces_csv(const std::string& path, long nt, long npts,
                      const std::vector<double>& traces, double t0, double dt) {
    if (nt < 0 || npts < 0 || traces.size() != std::size_t(nt) * std::size_t(npts))
        throw ParameterError("write_traces_csv: shape mismatch");
    std::ofstream os(path);
    if (!os) throw ParameterError("write_traces_csv: cannot open " + path);
    os << "t";
    for (long p = 0; p < npts; ++p) os << ",p" << p;
    os << "\n";
    os.precision(17);
    for (long t = 0; t < nt; ++t) {
        os << (t0 + double(t) * dt);
        for (long p = 0; p < npts; ++p) os << "," << traces[std::size_t(t) * npts + p];
        os << "\n";
    }
    if (!os) throw ParameterError("write_traces_csv: write failed for " + path);
}

// proj/src/sparse.cpp:152-173
void write_traces_csv(const std::string& path, const SparseFunction& s,
                      const std::vector<double>& times) {
    if (long(times.size()) != s.nt())
        throw ParameterError("time axis length does not match trace length");
    std::ofstream out(path);
    if (!out) throw Error("cannot open " + path + " for writing");
    out << "t";
    for (long p = 0; p < s.npoints(); ++p) out << ",p" << p;
    out << "\n";
    for (long t = 0; t < s.nt(); ++t) {
        out << g17(times[std::size_t(t)]);
        for (long p = 0; p < s.npoints(); ++p) out << ',' << g17(s.trace(t, p));
        out << "\n";
    }
}

// proj/src/sparse.cpp:175-199
void read_traces_csv(const std::string& path, SparseFunction& s, std::vector<double>* times) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open " + path);
    std::string line;
    if (!std::getline(in, line)) throw Error(path + ": missing header");
    if (times) times->clear();
    long t = 0;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (t >= s.nt()) throw Error(path + ": more rows than trace steps");
        std::istringstream row(line);
        std::string cell;
        if (!std::getline(row, cell, ',')) throw Error(path + ": short row");
        if (times) times->push_back(std::stod(cell));
        for (long p = 0; p < s.npoints(); ++p) {
            if (!std::getline(row, cell, ',')) throw Error(path + ": short row");
            s.trace(t, p) = std::stod(cell);
        }
        ++t;
    }
    if (t != s.nt()) throw Error(path + ": fewer rows than trace steps");
}

// proj/src/sparse.cpp:201-214 (axis names x, y, z as in proj/include/sf/grid.hpp:42-44)
void write_coords_csv(const std::string& path, const SparseFunction& s) {
    std::ofstream out(path);
    if (!out) throw Error("cannot open " + path + " for writing");
    static const char* names[3] = {"x", "y", "z"};
    const std::size_t nd = std::size_t(s.grid()->ndim());
    for (std::size_t d = 0; d < nd; ++d) out << (d ? "," : "") << names[d];
    out << "\n";
    for (long p = 0; p < s.npoints(); ++p) {
        for (std::size_t d = 0; d < nd; ++d) out << (d ? "," : "") << g17(s.coord(p, d));
        out << "\n";
    }
}

// proj/src/sparse.cpp:216-229
std::vector<double> read_coords_csv(const std::string& path, std::size_t ndim) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open " + path);
    std::string line;
    if (!std::getline(in, line)) throw Error(path + ": missing header");
    std::vector<double> coords;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::istringstream row(line);
        std::string cell;
        for (std::size_t d = 0; d < ndim; ++d) {
            if (!std::getline(row, cell, ',')) throw Error(path + ": short row");
            coords.push_back(std::stod(cell));
        }
    }
    if (coords.empty()) throw Error(path + ": no points");
    return coords;
}

}  // namespace sfb
