// Host-side I/O and input generation for the B200 front-end (csfs_b200 CLI): the
// reference's csfs/io.hpp (CSV formats, %.17g, CLI error codes; io.cpp:47-220) and the
// pieces of geometry/applications the `sum` / `bench` workflows need (build_grid
// geometry.cpp:97-213, real_sph_harm applications.cpp:20-49, relative_l2_error :51-67),
// on plain std::vector data so the CLI links only against libcsfs_b200.so.
#pragma once

#include <cstddef>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace csfs_b200::host {

struct Vec3 {
    double x, y, z;
};

// CLI-facing error with a machine-readable code (io.hpp:15-18).
struct CliError {
    std::string code;
    std::string message;
};
[[noreturn]] void throw_cli(const std::string& code, const std::string& message);
// E_FLAGS 2, E_KERNEL 3, E_CONFIG 4, E_CSV 5, E_DIM 6, E_IO 7, anything else 1 (io.cpp:51-59)
int exit_code_for(const std::string& code);

// 17 significant digits, "%.17g" (io.cpp:61-65)
std::string format_double(double v);

struct Grid {
    std::string kind;
    int level = 0;
    std::vector<Vec3> centers;
    std::vector<double> areas;
    std::size_t size() const { return centers.size(); }
};
// icosahedral (levels 0..9), cubed_sphere (0..10), latlon (4..9); throws
// std::invalid_argument with the reference's messages.
Grid build_grid(const std::string& kind, int level);

double real_sph_harm(int l, int m, const Vec3& p);

// sqrt(sum A (phi1 - phi2)^2 / sum A phi_exact^2) over out_dim components
double relative_l2_error(const std::vector<double>& phi1, const std::vector<double>& phi2,
                         const std::vector<double>& phi_exact, const std::vector<double>& areas, int out_dim);

struct Particles {
    std::vector<Vec3> positions;
    std::vector<double> weights;
    std::size_t size() const { return positions.size(); }
};

// `x,y,z,weight` (positions normalized) or `lon,lat,area,value` (degrees; weight =
// value * area), chosen by the header (io.cpp:166-185).
Particles read_particles_csv(const std::string& path);
// potentials written by write_potentials_csv; out_dim from the header; row count checked
// (E_DIM) (io.cpp:190-220).
std::vector<double> read_potentials_csv(const std::string& path, std::size_t expected_rows, int& out_dim);

void write_grid_csv(const std::string& path, const Grid& grid);
void write_potentials_csv(const std::string& path, const std::vector<Vec3>& points, const std::vector<double>& phi,
                          int out_dim);

// Minimal ordered JSON value for the reports (objects keep insertion order).
class Json {
public:
    Json() : kind_(Null) {}
    Json(double v) : kind_(Number), num_(format_double(v)) {}
    Json(int v) : kind_(Number), num_(std::to_string(v)) {}
    Json(long long v) : kind_(Number), num_(std::to_string(v)) {}
    Json(unsigned long long v) : kind_(Number), num_(std::to_string(v)) {}
    Json(std::size_t v, int) : kind_(Number), num_(std::to_string(v)) {}
    Json(bool v) : kind_(Bool), num_(v ? "true" : "false") {}
    Json(const char* s) : kind_(String), str_(s) {}
    Json(std::string s) : kind_(String), str_(std::move(s)) {}
    static Json object() { Json j; j.kind_ = Object; return j; }
    static Json array() { Json j; j.kind_ = Array; return j; }
    static Json count(std::size_t v) { return Json(v, 0); }
    Json& set(const std::string& key, Json v);
    Json& push(Json v);
    std::string dump(int indent = 2) const;

private:
    enum Kind { Null, Number, Bool, String, Object, Array } kind_;
    std::string num_, str_;
    std::vector<std::pair<std::string, Json>> items_;  // object members / array elements (key unused)
    void dump_to(std::string& out, int indent, int depth) const;
};

}  // namespace csfs_b200::host
