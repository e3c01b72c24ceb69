// csfs_b200 — command-line front-end of the B200 engine: the reference CLI's `grid`, `sum`
// and `bench` subcommands (/root/reference/proj/src/cli.cpp:131-206, 473-543, 561-657) with
// the same flags, CSV formats, JSON report fields and exit codes (io.hpp), evaluating
// through the C-ABI (include/csfs_b200.h).  The reference parses flags with CLI11 and writes
// JSON with nlohmann::json, neither of which is in this image; both are replaced by small
// local equivalents (any flag error -> E_FLAGS, like the reference's ParseError path).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "csfs_b200.h"
#include "io.hpp"

using namespace csfs_b200::host;

namespace {

// ---- flags ------------------------------------------------------------------------------

// One subcommand's flags: name -> setter (value flags) or toggle (boolean flags).
class Flags {
public:
    void value(const std::string& names, std::function<void(const std::string&)> set) {
        for (const std::string& n : split(names)) values_[n] = set;
    }
    void toggle(const std::string& name, bool& b) { toggles_[name] = &b; }
    void required(const std::string& name) { required_.push_back(name); }
    void parse(int argc, const char* const* argv, int first) {
        std::vector<std::string> seen;
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i], v;
            bool inline_value = false;
            const std::size_t eq = a.find('=');
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                v = a.substr(eq + 1);
                a = a.substr(0, eq);
                inline_value = true;
            }
            if (toggles_.count(a)) {
                if (inline_value) throw_cli("E_FLAGS", a + " takes no value");
                *toggles_[a] = true;
                continue;
            }
            const auto it = values_.find(a);
            if (it == values_.end()) throw_cli("E_FLAGS", "The following argument was not expected: " + a);
            if (!inline_value) {
                if (i + 1 >= argc) throw_cli("E_FLAGS", a + " requires a value");
                v = argv[++i];
            }
            try {
                it->second(v);
            } catch (const CliError&) {
                throw;
            } catch (const std::exception&) {
                throw_cli("E_FLAGS", "Could not convert: " + a + " = " + v);
            }
            seen.push_back(a);
        }
        for (const std::string& r : required_) {
            bool ok = false;
            for (const std::string& n : split(r)) ok = ok || std::count(seen.begin(), seen.end(), n);
            if (!ok) throw_cli("E_FLAGS", split(r).back() + " is required");
        }
    }

private:
    static std::vector<std::string> split(const std::string& names) {
        std::vector<std::string> out;
        std::istringstream in(names);
        for (std::string n; std::getline(in, n, ',');) out.push_back(n);
        return out;
    }
    std::map<std::string, std::function<void(const std::string&)>> values_;
    std::map<std::string, bool*> toggles_;
    std::vector<std::string> required_;
};

double to_double(const std::string& s) {
    std::size_t used = 0;
    const double v = std::stod(s, &used);
    if (used != s.size()) throw std::invalid_argument(s);
    return v;
}
int to_int(const std::string& s) {
    std::size_t used = 0;
    const int v = std::stoi(s, &used);
    if (used != s.size()) throw std::invalid_argument(s);
    return v;
}

struct CommonOpts {  // cli.cpp:23-47
    std::string kernel = "laplace", method = "csfmm";
    double mac = 0.7;
    int degree = 6, n0 = -1, threads = 0;
    unsigned seed = 0;
    bool stats = false;
    double sal_a1 = -2.7, sal_b0 = -6.21196, sal_b1 = 6.1, rho_ratio = 1025.0 / 5517.0;  // kernels.hpp:18-23
};

void add_common(Flags& f, CommonOpts& o, bool with_kernel = true) {
    if (with_kernel) f.value("--kernel", [&](const std::string& v) { o.kernel = v; });
    f.value("--method", [&](const std::string& v) { o.method = v; });
    f.value("--mac", [&](const std::string& v) { o.mac = to_double(v); });
    f.value("--degree", [&](const std::string& v) { o.degree = to_int(v); });
    f.value("--n0", [&](const std::string& v) { o.n0 = to_int(v); });
    f.value("--threads", [&](const std::string& v) { o.threads = to_int(v); });
    f.value("--seed", [&](const std::string& v) { o.seed = unsigned(std::stoul(v)); });
    f.toggle("--stats", o.stats);
    f.value("--sal-a1", [&](const std::string& v) { o.sal_a1 = to_double(v); });
    f.value("--sal-b0", [&](const std::string& v) { o.sal_b0 = to_double(v); });
    f.value("--sal-b1", [&](const std::string& v) { o.sal_b1 = to_double(v); });
    f.value("--rho-ratio", [&](const std::string& v) { o.rho_ratio = to_double(v); });
}

// ---- engine -----------------------------------------------------------------------------

enum class Method { Direct, Cstc, Csfmm };

Method parse_method(const std::string& m) {
    if (m == "direct") return Method::Direct;
    if (m == "cstc") return Method::Cstc;
    if (m == "csfmm") return Method::Csfmm;
    throw_cli("E_CONFIG", "unknown method: " + m);
}
const char* method_name(Method m) { return m == Method::Direct ? "direct" : m == Method::Cstc ? "cstc" : "csfmm"; }

csfs_b200_kernel make_kernel(const CommonOpts& o) {  // Kernel::parse (kernels.cpp:109-117)
    static const std::map<std::string, int> kinds = {{"laplace", 0}, {"biharmonic", 1}, {"biot_savart", 2}, {"sal", 3}};
    const auto it = kinds.find(o.kernel);
    if (it == kinds.end()) throw_cli("E_KERNEL", "unknown kernel: " + o.kernel);
    return {it->second, o.sal_a1, o.sal_b0, o.sal_b1, o.rho_ratio};
}
int out_dim(const csfs_b200_kernel& k) { return k.kind == 2 ? 3 : 1; }

struct Config {
    Method method;
    csfs_b200_config c;
    int resolved_n0() const { return c.n0 >= 0 ? c.n0 : 4 * c.degree * c.degree; }
};

Config make_config(const CommonOpts& o) {  // cli.cpp:57-72
    Config cfg{parse_method(o.method), {o.mac, o.degree, o.n0, 1}};
    if (o.mac <= 0.0 || o.mac > 1.0) throw_cli("E_CONFIG", "mac must lie in (0, 1]");
    if (o.degree < 1) throw_cli("E_CONFIG", "degree must be positive");
    return cfg;
}

// One context per process (created on first use: flag / input errors never touch the GPU).
csfs_b200_ctx* engine() {
    static std::unique_ptr<csfs_b200_ctx, void (*)(csfs_b200_ctx*)> ctx(nullptr, csfs_b200_destroy);
    if (!ctx) {
        csfs_b200_ctx* c = nullptr;
        if (csfs_b200_create(&c, 0) != CSFS_B200_OK)
            throw std::runtime_error("no usable sm_100 GPU (the B200 engine has no CPU fallback)");
        ctx.reset(c);
    }
    return ctx.get();
}

void check(int rc) {
    if (rc == CSFS_B200_OK) return;
    std::string msg = csfs_b200_last_error(engine());
    if (msg.empty()) msg = "csfs_b200 error code " + std::to_string(rc);
    if (rc == CSFS_B200_INVALID_ARGUMENT) throw_cli("E_CONFIG", msg);
    throw std::runtime_error(msg);
}

struct Sum {
    std::vector<double> phi;
    csfs_b200_stats st{};
};

// summed_potential (summation.cpp:423-440) over the C-ABI
Sum summed_potential(const Particles& p, const csfs_b200_kernel& k, const Config& cfg) {
    Sum s;
    s.phi.assign(p.size() * out_dim(k), 0.0);
    const double* x = p.positions.empty() ? nullptr : &p.positions[0].x;
    if (cfg.method == Method::Direct) {
        const auto t0 = std::chrono::steady_clock::now();
        check(csfs_b200_direct(engine(), x, p.size(), x, p.weights.data(), p.size(), &k, s.phi.data()));
        s.st.t_traversal = s.st.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        s.st.pp = uint64_t(p.size()) * p.size();
    } else if (cfg.method == Method::Cstc) {
        check(csfs_b200_cstc(engine(), x, p.size(), x, p.weights.data(), p.size(), &k, &cfg.c, s.phi.data(), &s.st));
    } else {
        check(csfs_b200_csfmm(engine(), x, p.size(), x, p.weights.data(), p.size(), &k, &cfg.c, s.phi.data(), &s.st));
    }
    return s;
}

// ---- report pieces (cli.cpp:95-119) -------------------------------------------------------

Json timings_json(const csfs_b200_stats& s) {
    return Json::object()
        .set("tree_build", s.t_tree_build)
        .set("upward", s.t_upward)
        .set("traversal", s.t_traversal)
        .set("downward", s.t_downward)
        .set("total", s.t_total);
}
Json interactions_json(const csfs_b200_stats& s) {
    return Json::object()
        .set("pp", (unsigned long long)s.pp)
        .set("pc", (unsigned long long)s.pc)
        .set("cp", (unsigned long long)s.cp)
        .set("cc", (unsigned long long)s.cc);
}
// TreeStats of the last call's tree `which` (0 target, 1 source): depth, counts and the
// leaf-size histogram (cluster_tree.cpp:148-161; empty face roots count as size-0 leaves)
Json tree_json(int which) {
    int ncl = 0, depth = 0, npp = 0;
    size_t np = 0;
    check(csfs_b200_tree_info(engine(), which, &ncl, &depth, &np, &npp));
    std::vector<int> ints(size_t(ncl) * 10);
    check(csfs_b200_tree_export(engine(), which, nullptr, ints.data(), nullptr, nullptr));
    std::vector<int> hist;
    int leaves = 0;
    for (int c = 0; c < ncl; ++c) {
        const int* r = &ints[size_t(c) * 10];
        if (r[5] != 0) continue;  // child_count
        ++leaves;
        const int count = r[2] - r[1];
        if (int(hist.size()) <= count) hist.resize(count + 1, 0);
        ++hist[count];
    }
    Json h = Json::array();
    for (int v : hist) h.push(v);
    return Json::object().set("depth", depth).set("cluster_count", ncl).set("leaf_count", leaves).set(
        "leaf_size_histogram", h);
}
Json environment_json(const CommonOpts& o) {
    return Json::object()
        .set("compiler", __VERSION__)
        .set("seed", (long long)o.seed)
        .set("threads", o.threads)
        .set("openmp", false)
        .set("engine", "csfs_b200 (sm_100a, one GPU)");
}

void emit_report(const Json& report, const std::string& path) {
    if (!path.empty()) {
        std::ofstream f(path);
        if (!f) throw_cli("E_IO", "cannot open report file: " + path);
        f << report.dump(2) << '\n';
    }
    std::cout << report.dump(2) << std::endl;
}

Grid grid_from_spec(const std::string& spec) {  // cli.cpp:74-85
    const std::size_t colon = spec.find(':');
    if (colon == std::string::npos) throw_cli("E_CONFIG", "grid spec must look like kind:level, got '" + spec + "'");
    try {
        return build_grid(spec.substr(0, colon), std::stoi(spec.substr(colon + 1)));
    } catch (const std::invalid_argument& e) {
        throw_cli("E_CONFIG", e.what());
    }
}

double y43(const Vec3& p) { return real_sph_harm(4, 3, p); }

Particles y43_particles(const Grid& g) {
    Particles p;
    p.positions = g.centers;
    p.weights.resize(g.size());
    for (std::size_t i = 0; i < g.size(); ++i) p.weights[i] = y43(g.centers[i]) * g.areas[i];
    return p;
}

// ---- subcommands --------------------------------------------------------------------------

int cmd_grid(const std::string& kind, int level, const std::string& out) {
    Grid g;
    try {
        g = build_grid(kind, level);
    } catch (const std::invalid_argument& e) {
        throw_cli("E_CONFIG", e.what());
    }
    write_grid_csv(out, g);
    std::cout << Json::object()
                     .set("subcommand", "grid")
                     .set("kind", kind)
                     .set("level", level)
                     .set("N", Json::count(g.size()))
                     .dump(2)
              << std::endl;
    return 0;
}

int cmd_sum(const CommonOpts& o, const std::string& grid_spec, const std::string& particles,
            const std::string& reference, const std::string& out, const std::string& report_path) {
    const csfs_b200_kernel k = make_kernel(o);
    const Config cfg = make_config(o);
    if (grid_spec.empty() == particles.empty()) throw_cli("E_FLAGS", "exactly one of --grid and --particles is required");
    Particles p;
    std::vector<double> areas;
    if (!grid_spec.empty()) {
        const Grid g = grid_from_spec(grid_spec);
        p = y43_particles(g);
        areas = g.areas;
    } else {
        p = read_particles_csv(particles);
        areas.assign(p.size(), 1.0);
    }
    const Sum s = summed_potential(p, k, cfg);
    static const char* names[] = {"laplace", "biharmonic", "biot_savart", "sal"};
    Json report = Json::object()
                      .set("subcommand", "sum")
                      .set("N", Json::count(p.size()))
                      .set("kernel", names[k.kind])
                      .set("method", method_name(cfg.method))
                      .set("mac", cfg.c.mac)
                      .set("degree", cfg.c.degree)
                      .set("n0", cfg.resolved_n0())
                      .set("timings", timings_json(s.st))
                      .set("interactions", interactions_json(s.st))
                      .set("environment", environment_json(o));
    if (o.stats) {  // (direct builds no tree: the reference reports an empty TreeStats)
        report.set("tree", cfg.method == Method::Direct ? Json::object()
                                                             .set("depth", 0)
                                                             .set("cluster_count", 0)
                                                             .set("leaf_count", 0)
                                                             .set("leaf_size_histogram", Json::array())
                                                       : tree_json(1));
        if (cfg.method == Method::Csfmm) report.set("target_tree", tree_json(0));
    }
    if (!reference.empty()) {
        std::vector<double> ref;
        if (reference == "direct") {
            Config d = cfg;
            d.method = Method::Direct;
            ref = summed_potential(p, k, d).phi;
        } else {
            int dim = 0;
            ref = read_potentials_csv(reference, p.size(), dim);
            if (dim != out_dim(k)) throw_cli("E_DIM", "reference output dimension does not match the kernel");
        }
        try {
            report.set("relative_l2_error", relative_l2_error(s.phi, ref, ref, areas, out_dim(k)));
        } catch (const std::invalid_argument& e) {
            throw_cli("E_CONFIG", e.what());
        }
    }
    if (!out.empty()) write_potentials_csv(out, p.positions, s.phi, out_dim(k));
    emit_report(report, report_path);
    return 0;
}

// read a particle CSV in either format, write it back as `x,y,z,weight` (positions
// normalized, lon/lat converted, weights = value * area): the io.cpp:166-185 conversion
int cmd_convert(const std::string& in, const std::string& out) {
    const Particles p = read_particles_csv(in);
    std::ofstream f(out);
    if (!f) throw_cli("E_IO", "cannot open output file: " + out);
    f << "x,y,z,weight\n";
    for (std::size_t i = 0; i < p.size(); ++i)
        f << format_double(p.positions[i].x) << ',' << format_double(p.positions[i].y) << ','
          << format_double(p.positions[i].z) << ',' << format_double(p.weights[i]) << '\n';
    std::cout << Json::object().set("subcommand", "convert").set("N", Json::count(p.size())).dump(2) << std::endl;
    return 0;
}

std::vector<int> int_list(const std::string& csv, const std::string& what) {  // cli.cpp parse_int_list
    std::vector<int> out;
    std::istringstream in(csv);
    for (std::string item; std::getline(in, item, ',');) {
        try {
            out.push_back(std::stoi(item));
        } catch (const std::exception&) {
            throw_cli("E_FLAGS", "bad " + what + " list entry: " + item);
        }
    }
    if (out.empty()) throw_cli("E_FLAGS", "empty " + what + " list");
    return out;
}

double loglog_slope(const std::vector<double>& x, const std::vector<double>& y) {  // fit_loglog_slope
    const double n = double(x.size());
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
        const double lx = std::log(x[i]), ly = std::log(y[i]);
        sx += lx;
        sy += ly;
        sxx += lx * lx;
        sxy += lx * ly;
    }
    return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

int cmd_bench(const CommonOpts& o, const std::string& kind, const std::string& levels_csv,
              const std::string& methods_csv, const std::string& prefix) {
    const csfs_b200_kernel k = make_kernel(o);
    const std::vector<int> levels = int_list(levels_csv, "level");
    std::vector<std::string> methods;
    {
        std::istringstream in(methods_csv);
        for (std::string m; std::getline(in, m, ',');) methods.push_back(m);
    }
    if (kind != "icosahedral" && kind != "cubed_sphere" && kind != "latlon")
        throw_cli("E_CONFIG", "unknown grid kind: " + kind);
    std::ofstream csv(prefix + ".csv");
    if (!csv) throw_cli("E_IO", "cannot open output file: " + prefix + ".csv");
    csv << "method,level,N,seconds\n";
    Json rows = Json::array();
    std::map<std::string, std::vector<double>> ns, ts;
    for (const int level : levels) {
        Grid g;
        try {
            g = build_grid(kind, level);
        } catch (const std::invalid_argument& e) {
            throw_cli("E_CONFIG", e.what());
        }
        const Particles p = y43_particles(g);
        for (const std::string& m : methods) {
            CommonOpts om = o;
            om.method = m;
            const Config cfg = make_config(om);
            summed_potential(p, k, cfg);  // warm-up
            std::vector<double> t(3);
            for (double& ti : t) ti = summed_potential(p, k, cfg).st.t_total;
            std::sort(t.begin(), t.end());
            csv << m << ',' << level << ',' << g.size() << ',' << format_double(t[1]) << '\n';
            rows.push(Json::object().set("method", m).set("level", level).set("N", Json::count(g.size())).set(
                "seconds", t[1]));
            ns[m].push_back(double(g.size()));
            ts[m].push_back(t[1]);
        }
    }
    static const char* names[] = {"laplace", "biharmonic", "biot_savart", "sal"};
    Json exps = Json::object();
    for (const auto& [m, n] : ns)
        if (n.size() >= 2) exps.set(m, loglog_slope(n, ts[m]));
    Json report = Json::object()
                      .set("subcommand", "bench")
                      .set("kernel", names[k.kind])
                      .set("grid", kind)
                      .set("rows", rows)
                      .set("environment", environment_json(o))
                      .set("exponents", exps);
    emit_report(report, prefix + ".json");
    return 0;
}

const char* kUsage =
    "csfs_b200 — fast summation of pairwise particle interactions on the sphere (B200 engine)\n"
    "usage: csfs_b200 <grid|sum|bench|convert> [options]\n"
    "  grid  --kind icosahedral|cubed_sphere|latlon --level L -o out.csv\n"
    "  sum   (--grid kind:level | --particles file.csv) [--kernel K] [--method direct|cstc|csfmm]\n"
    "        [--mac M] [--degree D] [--n0 N] [--reference direct|file.csv] [-o out.csv] [--report r.json]\n"
    "        [--stats] [--sal-a1 .. --sal-b0 .. --sal-b1 .. --rho-ratio ..] [--threads T] [--seed S]\n"
    "  bench [--grid-kind K] [--levels 4,5] [--methods direct,cstc,csfmm] [--out-prefix bench] [common]\n"
    "  convert --particles in.csv -o out.csv   (either particle format -> x,y,z,weight)\n";

int cli_main(int argc, const char* const* argv) {
    try {
        if (argc < 2) throw_cli("E_FLAGS", "A subcommand is required");
        const std::string sub = argv[1];
        if (sub == "-h" || sub == "--help") {
            std::cout << kUsage;
            return 0;
        }
        for (int i = 2; i < argc; ++i)
            if (std::string(argv[i]) == "-h" || std::string(argv[i]) == "--help") {
                std::cout << kUsage;
                return 0;
            }
        Flags f;
        if (sub == "grid") {
            std::string kind = "icosahedral", out;
            int level = 4;
            f.value("--kind", [&](const std::string& v) { kind = v; });
            f.value("--level", [&](const std::string& v) { level = to_int(v); });
            f.value("-o,--out", [&](const std::string& v) { out = v; });
            f.required("-o,--out");
            f.parse(argc, argv, 2);
            return cmd_grid(kind, level, out);
        }
        if (sub == "sum") {
            CommonOpts o;
            std::string grid, particles, reference, out, report;
            add_common(f, o);
            f.value("--grid", [&](const std::string& v) { grid = v; });
            f.value("--particles", [&](const std::string& v) { particles = v; });
            f.value("--reference", [&](const std::string& v) { reference = v; });
            f.value("-o,--out", [&](const std::string& v) { out = v; });
            f.value("--report", [&](const std::string& v) { report = v; });
            f.parse(argc, argv, 2);
            return cmd_sum(o, grid, particles, reference, out, report);
        }
        if (sub == "bench") {
            CommonOpts o;
            o.threads = 1;
            std::string kind = "icosahedral", levels = "4,5", methods = "direct,cstc,csfmm", prefix = "bench";
            add_common(f, o);
            f.value("--grid-kind", [&](const std::string& v) { kind = v; });
            f.value("--levels", [&](const std::string& v) { levels = v; });
            f.value("--methods", [&](const std::string& v) { methods = v; });
            f.value("--out-prefix", [&](const std::string& v) { prefix = v; });
            f.parse(argc, argv, 2);
            return cmd_bench(o, kind, levels, methods, prefix);
        }
        if (sub == "convert") {
            std::string in, out;
            f.value("--particles", [&](const std::string& v) { in = v; });
            f.value("-o,--out", [&](const std::string& v) { out = v; });
            f.required("--particles");
            f.required("-o,--out");
            f.parse(argc, argv, 2);
            return cmd_convert(in, out);
        }
        throw_cli("E_FLAGS", "The following argument was not expected: " + sub);
    } catch (const CliError& e) {
        std::cerr << Json::object().set("error", e.code).set("message", e.message).dump(-1) << std::endl;
        return exit_code_for(e.code);
    } catch (const std::exception& e) {
        std::cerr << Json::object().set("error", "E_CONFIG").set("message", e.what()).dump(-1) << std::endl;
        return exit_code_for("E_CONFIG");
    }
}

}  // namespace

int main(int argc, char** argv) { return cli_main(argc, argv); }
