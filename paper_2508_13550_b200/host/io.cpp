// CSV / report I/O of the B200 front-end.  The interface is the reference's (csfs/io.hpp,
// /root/reference/proj/src/io.cpp:47-220): the same headers select the particle format,
// numbers are written "%.17g" (exact round trip), malformed input is E_CSV with the file
// and line, unreadable / unwritable paths are E_IO, a potentials file with the wrong row
// count is E_DIM — byte-identical messages, so scripts that parse them keep working.
//
// The implementation is a small streaming design of its own: CsvSource hands out the
// non-blank lines already split into trimmed fields, CsvSink writes rows of numbers, and
// the readers are thin field-mapping loops on top of them.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string_view>

#include "io.hpp"

namespace csfs_b200::host {

namespace {

constexpr double kPi = 3.14159265358979323846;

// ---- reading ------------------------------------------------------------------------------

// Blanks around a field: leading spaces, trailing spaces and carriage returns.
std::string_view strip(std::string_view f) {
    std::size_t b = 0, e = f.size();
    while (b < e && f[b] == ' ') ++b;
    while (e > b && (f[e - 1] == ' ' || f[e - 1] == '\r')) --e;
    return f.substr(b, e - b);
}

// Fields of one line with std::getline(',') semantics: "a,,b" has an empty middle field,
// a trailing comma adds no field, an empty line has none.
void split_fields(std::string_view rest, std::vector<std::string>& fields) {
    fields.clear();
    while (!rest.empty()) {
        const std::size_t comma = rest.find(',');
        fields.emplace_back(strip(rest.substr(0, comma)));
        if (comma == std::string_view::npos) break;
        rest.remove_prefix(comma + 1);
    }
}

// One CSV file, line by line: next() skips blank lines and returns the fields of the next
// one with its 1-based line number; first() returns line 1 whatever it holds.
class CsvSource {
public:
    explicit CsvSource(const std::string& path) : in_(path) {
        if (!in_) throw_cli("E_IO", "cannot open input file: " + path);
    }
    bool next(std::size_t& line_no, std::vector<std::string>& fields) {
        while (std::getline(in_, buf_)) {
            ++no_;
            if (buf_.empty()) continue;
            split_fields(buf_, fields);
            line_no = no_;
            return true;
        }
        return false;
    }
    bool first(std::vector<std::string>& fields) {
        if (no_ != 0 || !std::getline(in_, buf_)) return false;
        ++no_;
        split_fields(buf_, fields);
        return true;
    }

private:
    std::ifstream in_;
    std::string buf_;
    std::size_t no_ = 0;
};

// The whole field must be a number (strtod's grammar, as std::stod accepts it); anything
// else — empty, trailing characters, out of range — is E_CSV.
double to_number(const std::string& f, const std::string& path, std::size_t line_no) {
    const char* s = f.c_str();
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(s, &end);
    if (end == s || *end != '\0' || errno == ERANGE)
        throw_cli("E_CSV", path + ": malformed number '" + f + "' on line " + std::to_string(line_no));
    return v;
}

std::string joined(const std::vector<std::string>& fields) {
    std::string h;
    for (std::size_t i = 0; i < fields.size(); ++i) h += (i ? "," : "") + fields[i];
    return h;
}

// Header + numeric rows of exactly `width` columns.  Line 1 is the header whatever it
// holds; when line 1 is blank there is no header, every later line is data, and the
// missing header is reported after the rows were read.
struct Sheet {
    std::string header;  // the header fields joined with ','
    bool has_header = false;
    std::vector<double> cells;  // row-major, width per row
};

Sheet read_sheet(const std::string& path, std::size_t width) {
    CsvSource src(path);
    Sheet sh;
    std::vector<std::string> f;
    std::size_t line_no = 0;
    while (src.next(line_no, f)) {
        if (line_no == 1) {
            sh.header = joined(f);
            sh.has_header = true;
            continue;
        }
        if (f.size() != width)
            throw_cli("E_CSV", path + ": expected " + std::to_string(width) + " columns on line " +
                                   std::to_string(line_no));
        for (const std::string& cell : f) sh.cells.push_back(to_number(cell, path, line_no));
    }
    if (!sh.has_header) throw_cli("E_CSV", path + ": missing header line");
    return sh;
}

// ---- writing ------------------------------------------------------------------------------

class CsvSink {
public:
    CsvSink(const std::string& path, const char* header) : out_(path) {
        if (!out_) throw_cli("E_IO", "cannot open output file: " + path);
        out_ << header << '\n';
    }
    // one row: the values, comma separated, %.17g
    void row(std::initializer_list<double> head, const double* tail = nullptr, int n_tail = 0) {
        const char* sep = "";
        for (double v : head) {
            out_ << sep << format_double(v);
            sep = ",";
        }
        for (int i = 0; i < n_tail; ++i) out_ << ',' << format_double(tail[i]);
        out_ << '\n';
    }

private:
    std::ofstream out_;
};

}  // namespace

void throw_cli(const std::string& code, const std::string& message) { throw CliError{code, message}; }

int exit_code_for(const std::string& code) {
    static const char* const kCodes[] = {"E_FLAGS", "E_KERNEL", "E_CONFIG", "E_CSV", "E_DIM", "E_IO"};
    for (int i = 0; i < 6; ++i)
        if (code == kCodes[i]) return 2 + i;
    return 1;
}

std::string format_double(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

Particles read_particles_csv(const std::string& path) {
    const Sheet sh = read_sheet(path, 4);
    const bool xyz = sh.header == "x,y,z,weight";
    if (!xyz && sh.header != "lon,lat,area,value")
        throw_cli("E_CSV", path + ": header must be 'x,y,z,weight' or 'lon,lat,area,value'");
    Particles p;
    const std::size_t rows = sh.cells.size() / 4;
    p.positions.resize(rows);
    p.weights.resize(rows);
    for (std::size_t r = 0; r < rows; ++r) {
        const double* c = &sh.cells[4 * r];
        if (xyz) {  // normalized((x, y, z)), weight as given
            const double len = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
            p.positions[r] = {c[0] / len, c[1] / len, c[2] / len};
            p.weights[r] = c[3];
        } else {  // degrees -> unit vector, weight = value * area
            const double lon = c[0] * kPi / 180.0, lat = c[1] * kPi / 180.0;
            p.positions[r] = {std::cos(lat) * std::cos(lon), std::cos(lat) * std::sin(lon), std::sin(lat)};
            p.weights[r] = c[3] * c[2];
        }
    }
    return p;
}

std::vector<double> read_potentials_csv(const std::string& path, std::size_t expected_rows, int& out_dim) {
    CsvSource src(path);
    std::vector<std::string> f;
    if (!src.first(f)) throw_cli("E_CSV", path + ": missing header line");
    const std::string h = joined(f);
    if (h == "x,y,z,phi") out_dim = 1;
    else if (h == "x,y,z,phi,phi_y,phi_z") out_dim = 3;
    else throw_cli("E_CSV", path + ": unrecognized potentials header");
    std::vector<double> vals;
    std::size_t line_no = 0;
    while (src.next(line_no, f)) {
        if (f.size() != std::size_t(3 + out_dim))
            throw_cli("E_CSV", path + ": bad column count on line " + std::to_string(line_no));
        for (int d = 0; d < out_dim; ++d) vals.push_back(to_number(f[3 + d], path, line_no));
    }
    const std::size_t rows = vals.size() / out_dim;
    if (rows != expected_rows)
        throw_cli("E_DIM", path + ": has " + std::to_string(rows) + " rows, expected " + std::to_string(expected_rows));
    return vals;
}

void write_grid_csv(const std::string& path, const Grid& g) {
    CsvSink out(path, "x,y,z,area");
    for (std::size_t i = 0; i < g.size(); ++i) out.row({g.centers[i].x, g.centers[i].y, g.centers[i].z, g.areas[i]});
}

void write_potentials_csv(const std::string& path, const std::vector<Vec3>& pts, const std::vector<double>& phi,
                          int out_dim) {
    CsvSink out(path, out_dim == 1 ? "x,y,z,phi" : "x,y,z,phi,phi_y,phi_z");
    for (std::size_t i = 0; i < pts.size(); ++i) out.row({pts[i].x, pts[i].y, pts[i].z}, &phi[i * out_dim], out_dim);
}

// ---- JSON -------------------------------------------------------------------------------

Json& Json::set(const std::string& key, Json v) {
    for (auto& kv : items_)
        if (kv.first == key) {
            kv.second = std::move(v);
            return *this;
        }
    items_.emplace_back(key, std::move(v));
    return *this;
}

Json& Json::push(Json v) {
    items_.emplace_back(std::string(), std::move(v));
    return *this;
}

namespace {
void quote(std::string& out, const std::string& s) {
    out += '"';
    for (const char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            default:
                if ((unsigned char)c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", c);
                    out += b;
                } else {
                    out += c;
                }
        }
    }
    out += '"';
}
}  // namespace

void Json::dump_to(std::string& out, int indent, int depth) const {
    const std::string pad = indent > 0 ? std::string(size_t(indent) * (depth + 1), ' ') : "";
    const std::string close = indent > 0 ? std::string(size_t(indent) * depth, ' ') : "";
    const char* nl = indent > 0 ? "\n" : "";
    switch (kind_) {
        case Null: out += "null"; break;
        case Number:
            // JSON has no inf/nan
            out += (num_ == "inf" || num_ == "-inf" || num_ == "nan" || num_ == "-nan") ? "null" : num_;
            break;
        case Bool: out += num_; break;
        case String: quote(out, str_); break;
        case Object:
        case Array: {
            const bool obj = kind_ == Object;
            out += obj ? '{' : '[';
            if (items_.empty()) {
                out += obj ? '}' : ']';
                break;
            }
            out += nl;
            for (std::size_t i = 0; i < items_.size(); ++i) {
                out += pad;
                if (obj) {
                    quote(out, items_[i].first);
                    out += indent > 0 ? ": " : ":";
                }
                items_[i].second.dump_to(out, indent, depth + 1);
                if (i + 1 < items_.size()) out += ',';
                out += nl;
            }
            out += close;
            out += obj ? '}' : ']';
        }
    }
}

std::string Json::dump(int indent) const {
    std::string s;
    dump_to(s, indent, 0);
    return s;
}

}  // namespace csfs_b200::host
