// gridio.cpp -- SFGD grid container and trace / coordinate CSV tables of the host layer.
// The FILE FORMATS are the reference's (SFGD: proj/include/sf/gridio.hpp:8-18; CSV tables:
// proj/include/sf/sparse.hpp:97-104) and files written here are byte-identical to the
// reference's for the same data (tests/test_gridio.py); the code is this repository's own:
// tables are rendered into one text buffer and written with a single call, files are read
// whole and walked with a cursor.
#include <algorithm>
#include <array>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string_view>

#include "sfb/gridio.hpp"

namespace sfb {

namespace {

std::array<unsigned char, 4> le32(uint32_t v) {
    return {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
            static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
}

// ---- text tables ------------------------------------------------------------------------

// A comma-separated table rendered in memory.  Numbers are printed with 17 significant
// digits in the shortest of fixed / scientific notation ("%.17g"), which is what both of the
// reference's writers produce and what makes an f64 survive the round trip exactly.
class TableText {
public:
    explicit TableText(std::size_t expected_cells) { text_.reserve(24 * expected_cells + 64); }
    TableText& label(std::string_view s) {
        separate();
        text_.append(s);
        return *this;
    }
    TableText& indexed(char prefix, long i) {   // "p0", "p1", ...
        separate();
        text_.push_back(prefix);
        text_.append(std::to_string(i));
        return *this;
    }
    TableText& number(double v) {
        separate();
        char buf[40];
        const int n = std::snprintf(buf, sizeof buf, "%.17g", v);
        text_.append(buf, std::size_t(n));
        return *this;
    }
    void end_row() {
        text_.push_back('\n');
        row_open_ = false;
    }
    // one write; `what` names the caller in the error text
    void save(const std::string& path, const char* what) const {
        std::FILE* f = std::fopen(path.c_str(), "wb");
        if (!f) throw Error(std::string(what) + ": cannot create '" + path + "'");
        const bool ok = std::fwrite(text_.data(), 1, text_.size(), f) == text_.size();
        if (std::fclose(f) != 0 || !ok)
            throw Error(std::string(what) + ": short write to '" + path + "'");
    }

private:
    void separate() {
        if (row_open_) text_.push_back(',');
        row_open_ = true;
    }
    std::string text_;
    bool row_open_ = false;
};

// A whole table file in memory, walked row by row (blank lines are skipped, the first
// non-consumed line is the header) and cell by cell.
class TableCursor {
public:
    TableCursor(const std::string& path, const char* what) : path_(path), what_(what) {
        std::ifstream in(path, std::ios::binary);
        if (!in) fail("cannot open the file");
        text_.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    }
    [[noreturn]] void fail(const std::string& why) const {
        throw Error(std::string(what_) + " '" + path_ + "': " + why);
    }
    // moves to the next non-blank line; false at the end of the file
    bool next_row() {
        while (pos_ < text_.size()) {
            const std::size_t eol = std::min(text_.find('\n', pos_), text_.size());
            row_ = std::string_view(text_).substr(pos_, eol - pos_);
            pos_ = eol + 1;
            if (!row_.empty() && row_.back() == '\r') row_.remove_suffix(1);
            if (!row_.empty()) {
                ++row_no_;
                return true;
            }
        }
        return false;
    }
    // the next comma-separated cell of the current row as a number
    double number() {
        if (row_done_) fail("row " + std::to_string(row_no_) + " has too few columns");
        const std::size_t comma = row_.find(',');
        const std::string cell(row_.substr(0, comma));
        if (comma == std::string_view::npos) {
            row_done_ = true;
        } else {
            row_.remove_prefix(comma + 1);
        }
        char* end = nullptr;
        errno = 0;
        const double v = std::strtod(cell.c_str(), &end);
        if (end == cell.c_str())
            fail("row " + std::to_string(row_no_) + ": '" + cell + "' is not a number");
        return v;
    }
    void begin_cells() { row_done_ = row_.empty(); }

private:
    std::string path_;
    const char* what_;
    std::string text_;
    std::size_t pos_ = 0;
    std::string_view row_;
    long row_no_ = 0;
    bool row_done_ = false;
};

}  // namespace

// ---- SFGD container -------------------------------------------------------------------------
// bytes 0-3 "SFGD" | 4 rank | 5 dtype (0 = f64) | 6-7 zero | rank x u32 LE extents | payload

namespace {

constexpr char kMagic[4] = {'S', 'F', 'G', 'D'};

struct SfgdHeader {
    std::vector<long> extents;
    std::size_t cells() const {
        std::size_t n = 1;
        for (long e : extents) n *= std::size_t(e);
        return n;
    }
    std::size_t bytes() const { return 8 + 4 * extents.size(); }
    std::vector<unsigned char> encode() const {
        std::vector<unsigned char> out(bytes(), 0);
        std::memcpy(out.data(), kMagic, 4);
        out[4] = static_cast<unsigned char>(extents.size());
        for (std::size_t d = 0; d < extents.size(); ++d) {
            const auto w = le32(uint32_t(extents[d]));
            std::copy(w.begin(), w.end(), out.begin() + 8 + 4 * long(d));
        }
        return out;
    }
    // parses the front of `raw`; returns an empty string or what is wrong with it
    std::string decode(const std::vector<unsigned char>& raw) {
        if (raw.size() < 8 || std::memcmp(raw.data(), kMagic, 4) != 0) return "not an SFGD file";
        const std::size_t rank = raw[4];
        if (rank == 0 || raw[5] != 0) return "unsupported rank or element type";
        if (raw.size() < 8 + 4 * rank) return "header cut short";
        extents.assign(rank, 0);
        for (std::size_t d = 0; d < rank; ++d) {
            const unsigned char* w = raw.data() + 8 + 4 * d;
            extents[d] = long(uint32_t(w[0]) | uint32_t(w[1]) << 8 | uint32_t(w[2]) << 16 |
                              uint32_t(w[3]) << 24);
        }
        return "";
    }
};

}  // namespace

void write_grid(const std::string& path, const std::vector<long>& shape,
                const std::vector<double>& data) {
    SfgdHeader h{shape};
    const bool extents_ok =
        std::all_of(shape.begin(), shape.end(), [](long e) { return e >= 1 && e <= 0xffffffffL; });
    if (shape.empty() || shape.size() > 255 || !extents_ok)
        throw ParameterError("write_grid: rank must be 1..255 and every extent a positive u32");
    if (h.cells() != data.size())
        throw ParameterError("write_grid: " + std::to_string(data.size()) + " values for a grid of " +
                             std::to_string(h.cells()) + " cells");
    const std::vector<unsigned char> head = h.encode();
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw ParameterError("write_grid: cannot create '" + path + "'");
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    ok = ok && std::fwrite(data.data(), sizeof(double), data.size(), f) == data.size();
    if (std::fclose(f) != 0 || !ok) throw ParameterError("write_grid: short write to '" + path + "'");
}

GridData read_grid(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw ParameterError("read_grid: cannot open '" + path + "'");
    const std::size_t size = std::size_t(in.tellg());
    in.seekg(0);
    std::vector<unsigned char> front(std::min<std::size_t>(size, 8 + 4 * 255));
    in.read(reinterpret_cast<char*>(front.data()), std::streamsize(front.size()));
    SfgdHeader h;
    const std::string why = h.decode(front);
    if (!why.empty()) throw ParameterError("read_grid '" + path + "': " + why);
    GridData g;
    g.shape = h.extents;
    const std::size_t want = h.cells() * sizeof(double);
    if (size < h.bytes() + want)
        throw ParameterError("read_grid '" + path + "': payload cut short (" +
                             std::to_string(size - h.bytes()) + " of " + std::to_string(want) + " bytes)");
    g.data.resize(h.cells());
    in.seekg(std::streamoff(h.bytes()));
    in.read(reinterpret_cast<char*>(g.data.data()), std::streamsize(want));
    if (!in) throw ParameterError("read_grid '" + path + "': read failed");
    return g;
}

// ---- trace tables: "t,p0,p1,..." then one row per time sample ------------------------------

namespace {

void trace_header(TableText& tab, long npts) {
    tab.label("t");
    for (long p = 0; p < npts; ++p) tab.indexed('p', p);
    tab.end_row();
}

}  // namespace

// bare-table form (the reference's counterpart takes a regular time axis t0 + t*dt,
// proj/include/sf/gridio.hpp)
void write_traces_csv(const std::string& path, long nt, long npts,
                      const std::vector<double>& traces, double t0, double dt) {
    if (nt < 0 || npts < 0 || traces.size() != std::size_t(nt) * std::size_t(npts))
        throw ParameterError("write_traces_csv: the table is not nt x npts");
    TableText tab(std::size_t(nt + 1) * std::size_t(npts + 1));
    trace_header(tab, npts);
    const double* row = traces.data();
    for (long t = 0; t < nt; ++t, row += npts) {
        tab.number(t0 + double(t) * dt);
        for (long p = 0; p < npts; ++p) tab.number(row[p]);
        tab.end_row();
    }
    tab.save(path, "write_traces_csv");
}

// cloud form: the traces of a SparseFunction against an explicit time axis
void write_traces_csv(const std::string& path, const SparseFunction& s,
                      const std::vector<double>& times) {
    const long nt = s.nt(), npts = s.npoints();
    if (times.size() != std::size_t(nt))
        throw ParameterError("write_traces_csv: " + std::to_string(times.size()) +
                             " time samples for " + std::to_string(nt) + " trace rows");
    TableText tab(std::size_t(nt + 1) * std::size_t(npts + 1));
    trace_header(tab, npts);
    for (long t = 0; t < nt; ++t) {
        tab.number(times[std::size_t(t)]);
        for (long p = 0; p < npts; ++p) tab.number(s.trace(t, p));
        tab.end_row();
    }
    tab.save(path, "write_traces_csv");
}

void read_traces_csv(const std::string& path, SparseFunction& s, std::vector<double>* times) {
    TableCursor cur(path, "read_traces_csv");
    if (!cur.next_row()) cur.fail("the header row is missing");
    const long nt = s.nt(), npts = s.npoints();
    std::vector<double> axis;
    axis.reserve(std::size_t(nt));
    long filled = 0;
    for (; cur.next_row(); ++filled) {
        if (filled == nt) cur.fail("holds more than the cloud's " + std::to_string(nt) + " rows");
        cur.begin_cells();
        axis.push_back(cur.number());
        for (long p = 0; p < npts; ++p) s.trace(filled, p) = cur.number();
    }
    if (filled < nt)
        cur.fail("holds " + std::to_string(filled) + " of the cloud's " + std::to_string(nt) + " rows");
    if (times) times->swap(axis);
}

// ---- point coordinates: "x[,y[,z]]" then one row per point --------------------------------

void write_coords_csv(const std::string& path, const SparseFunction& s) {
    const long npts = s.npoints();
    const std::size_t rank = std::size_t(s.grid()->ndim());
    TableText tab(std::size_t(npts + 1) * rank);
    for (std::size_t d = 0; d < rank; ++d)   // axis names of proj/include/sf/grid.hpp:42-44
        tab.label(std::string_view("xyz").substr(d, 1));
    tab.end_row();
    for (long p = 0; p < npts; ++p) {
        for (std::size_t d = 0; d < rank; ++d) tab.number(s.coord(p, d));
        tab.end_row();
    }
    tab.save(path, "write_coords_csv");
}

std::vector<double> read_coords_csv(const std::string& path, std::size_t ndim) {
    TableCursor cur(path, "read_coords_csv");
    if (!cur.next_row()) cur.fail("the header row is missing");
    std::vector<double> flat;
    while (cur.next_row()) {
        cur.begin_cells();
        for (std::size_t d = 0; d < ndim; ++d) flat.push_back(cur.number());
    }
    if (flat.empty()) cur.fail("lists no points");
    return flat;
}

}  // namespace sfb
