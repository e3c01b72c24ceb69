// CSV / report I/O of the B200 front-end, with the reference's formats and error codes
// (/root/reference/proj/src/io.cpp:47-220): headers select the particle format, numbers are
// written with "%.17g" (exact round trip), malformed input raises E_CSV with the file and
// line, unreadable / unwritable paths raise E_IO, a potentials file with the wrong row
// count raises E_DIM.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "io.hpp"

namespace csfs_b200::host {

namespace {

constexpr double kPi = 3.14159265358979323846;

std::ofstream create(const std::string& path) {
    std::ofstream f(path);
    if (!f) throw_cli("E_IO", "cannot open output file: " + path);
    return f;
}

std::string trim(std::string s) {
    std::size_t b = 0, e = s.size();
    while (b < e && s[b] == ' ') ++b;
    while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\r')) --e;
    return s.substr(b, e - b);
}

// comma-separated fields, blanks trimmed; like std::getline on ',' a trailing empty
// field is not reported
std::vector<std::string> fields_of(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream in(line);
    for (std::string f; std::getline(in, f, ',');) out.push_back(trim(f));
    return out;
}

double number(const std::string& s, const std::string& path, std::size_t line) {
    std::size_t used = 0;
    double v = 0.0;
    bool ok = true;
    try {
        v = std::stod(s, &used);
    } catch (const std::exception&) {
        ok = false;
    }
    if (!ok || used != s.size())
        throw_cli("E_CSV", path + ": malformed number '" + s + "' on line " + std::to_string(line));
    return v;
}

bool is_header(const std::vector<std::string>& h, std::initializer_list<const char*> names) {
    if (h.size() != names.size()) return false;
    std::size_t i = 0;
    for (const char* n : names)
        if (h[i++] != n) return false;
    return true;
}

struct Table {
    std::vector<std::string> header;
    std::vector<std::vector<double>> rows;
};

// first line = header; every other non-blank line holds exactly `cols` numbers
Table read_table(const std::string& path, std::size_t cols) {
    std::ifstream in(path);
    if (!in) throw_cli("E_IO", "cannot open input file: " + path);
    Table t;
    std::string line;
    for (std::size_t no = 1; std::getline(in, line); ++no) {
        if (line.empty()) continue;
        std::vector<std::string> f = fields_of(line);
        if (no == 1) {
            t.header = std::move(f);
            continue;
        }
        if (f.size() != cols)
            throw_cli("E_CSV", path + ": expected " + std::to_string(cols) + " columns on line " + std::to_string(no));
        std::vector<double> row(cols);
        for (std::size_t c = 0; c < cols; ++c) row[c] = number(f[c], path, no);
        t.rows.push_back(std::move(row));
    }
    if (t.header.empty()) throw_cli("E_CSV", path + ": missing header line");
    return t;
}

Vec3 lonlat_deg(double lon, double lat) {
    const double lo = lon * kPi / 180.0, la = lat * kPi / 180.0;
    return {std::cos(la) * std::cos(lo), std::cos(la) * std::sin(lo), std::sin(la)};
}

}  // namespace

void throw_cli(const std::string& code, const std::string& message) { throw CliError{code, message}; }

int exit_code_for(const std::string& code) {
    static const std::map<std::string, int> codes = {{"E_FLAGS", 2}, {"E_KERNEL", 3}, {"E_CONFIG", 4},
                                                     {"E_CSV", 5},   {"E_DIM", 6},    {"E_IO", 7}};
    const auto it = codes.find(code);
    return it == codes.end() ? 1 : it->second;
}

std::string format_double(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

Particles read_particles_csv(const std::string& path) {
    const Table t = read_table(path, 4);
    Particles p;
    p.positions.reserve(t.rows.size());
    p.weights.reserve(t.rows.size());
    if (is_header(t.header, {"x", "y", "z", "weight"})) {
        for (const auto& r : t.rows) {
            const double n = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
            p.positions.push_back({r[0] / n, r[1] / n, r[2] / n});
            p.weights.push_back(r[3]);
        }
    } else if (is_header(t.header, {"lon", "lat", "area", "value"})) {
        for (const auto& r : t.rows) {
            p.positions.push_back(lonlat_deg(r[0], r[1]));
            p.weights.push_back(r[3] * r[2]);
        }
    } else {
        throw_cli("E_CSV", path + ": header must be 'x,y,z,weight' or 'lon,lat,area,value'");
    }
    return p;
}

std::vector<double> read_potentials_csv(const std::string& path, std::size_t expected_rows, int& out_dim) {
    std::ifstream in(path);
    if (!in) throw_cli("E_IO", "cannot open input file: " + path);
    std::string line;
    if (!std::getline(in, line)) throw_cli("E_CSV", path + ": missing header line");
    const std::vector<std::string> h = fields_of(line);
    if (is_header(h, {"x", "y", "z", "phi"})) out_dim = 1;
    else if (is_header(h, {"x", "y", "z", "phi", "phi_y", "phi_z"})) out_dim = 3;
    else throw_cli("E_CSV", path + ": unrecognized potentials header");
    std::vector<double> vals;
    for (std::size_t no = 2; std::getline(in, line); ++no) {
        if (line.empty()) continue;
        const std::vector<std::string> f = fields_of(line);
        if (int(f.size()) != 3 + out_dim)
            throw_cli("E_CSV", path + ": bad column count on line " + std::to_string(no));
        for (int d = 0; d < out_dim; ++d) vals.push_back(number(f[3 + d], path, no));
    }
    const std::size_t rows = vals.size() / out_dim;
    if (rows != expected_rows)
        throw_cli("E_DIM", path + ": has " + std::to_string(rows) + " rows, expected " + std::to_string(expected_rows));
    return vals;
}

void write_grid_csv(const std::string& path, const Grid& g) {
    std::ofstream f = create(path);
    f << "x,y,z,area\n";
    for (std::size_t i = 0; i < g.size(); ++i)
        f << format_double(g.centers[i].x) << ',' << format_double(g.centers[i].y) << ','
          << format_double(g.centers[i].z) << ',' << format_double(g.areas[i]) << '\n';
}

void write_potentials_csv(const std::string& path, const std::vector<Vec3>& pts, const std::vector<double>& phi,
                          int out_dim) {
    std::ofstream f = create(path);
    f << (out_dim == 1 ? "x,y,z,phi" : "x,y,z,phi,phi_y,phi_z") << '\n';
    for (std::size_t i = 0; i < pts.size(); ++i) {
        f << format_double(pts[i].x) << ',' << format_double(pts[i].y) << ',' << format_double(pts[i].z);
        for (int d = 0; d < out_dim; ++d) f << ',' << format_double(phi[i * out_dim + d]);
        f << '\n';
    }
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
