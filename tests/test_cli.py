"""The `csfs_b200` front-end (paper_2508_13550_b200/host/cli.cpp): the reference CLI's
`grid` / `sum` / `bench` workflows with its CSV formats, %.17g numbers, JSON reports and
exit codes — the cases of the reference's own tests/test_cli.cpp, plus bitwise checks of
the generated inputs against the reference library (oracle/_ref).

CPU tests: grid generation, format conversion and every error path (none of which touch
the GPU).  GPU tests: `sum` / `bench` end to end, against the reference's summed_potential
on the same inputs."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2508_13550_b200", "csfs_b200")
CODES = {"E_FLAGS": 2, "E_KERNEL": 3, "E_CONFIG": 4, "E_CSV": 5, "E_DIM": 6, "E_IO": 7}


def run(args, cwd):
    p = subprocess.run([CLI] + list(args), cwd=cwd, capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def read_csv(path):
    with open(path) as f:
        header = f.readline().strip()
    return header, np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)


@pytest.fixture(autouse=True)
def _built():
    if not os.path.exists(CLI):
        pytest.fail(f"{CLI} is missing: run __graft_entry__.build()")


# ---- CPU ------------------------------------------------------------------------------


@pytest.mark.parametrize("kind,level", [("icosahedral", 0), ("icosahedral", 4), ("cubed_sphere", 0),
                                        ("cubed_sphere", 5), ("latlon", 4), ("latlon", 5)])
def test_grid_matches_reference(tmp_path, kind, level):
    """`grid` writes the reference's build_grid bit for bit (%.17g round-trips exactly)."""
    code, out, _ = run(["grid", "--kind", kind, "--level", str(level), "-o", "g.csv"], tmp_path)
    assert code == 0
    rep = json.loads(out)
    header, rows = read_csv(tmp_path / "g.csv")
    assert header == "x,y,z,area"
    xyz, areas = ref.grid(kind, level)
    assert rep == {"subcommand": "grid", "kind": kind, "level": level, "N": len(areas)} == {**rep, "N": rows.shape[0]}
    np.testing.assert_array_equal(rows[:, :3], xyz)
    np.testing.assert_array_equal(rows[:, 3], areas)


def test_grid_row_counts(tmp_path):
    """test_cli.cpp: 'grid subcommand row counts match the cell counts'."""
    assert run(["grid", "--kind", "icosahedral", "--level", "4", "-o", "g.csv"], tmp_path)[0] == 0
    lines = [l for l in open(tmp_path / "g.csv").read().splitlines() if l]
    assert len(lines) == 2562 + 1 and lines[0] == "x,y,z,area"


def test_error_codes(tmp_path):
    """test_cli.cpp: unknown kernel -> E_KERNEL; bad flags and bad configs use distinct exit
    codes; malformed CSV -> E_CSV; missing file -> E_IO.  Errors are one JSON line on stderr."""
    cases = [
        (["sum", "--kernel", "helmholtz", "--grid", "icosahedral:3"], "E_KERNEL"),
        (["sum", "--nonsense-flag", "1"], "E_FLAGS"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral:3", "--mac", "1.5"], "E_CONFIG"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral:3", "--degree", "0"], "E_CONFIG"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral:3", "--method", "fmm"], "E_CONFIG"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral:99"], "E_CONFIG"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral"], "E_CONFIG"),
        (["sum", "--kernel", "laplace", "--mac", "abc", "--grid", "icosahedral:3"], "E_FLAGS"),
        (["grid", "--kind", "hexagonal", "--level", "3", "-o", "x.csv"], "E_CONFIG"),
        (["grid", "--kind", "latlon", "--level", "3", "-o", "x.csv"], "E_CONFIG"),
        (["grid", "--level", "3"], "E_FLAGS"),
        (["sum", "--kernel", "laplace"], "E_FLAGS"),
        (["sum", "--kernel", "laplace", "--grid", "icosahedral:3", "--particles", "p.csv"], "E_FLAGS"),
        (["bench", "--levels", "4,x"], "E_FLAGS"),
        (["bench", "--grid-kind", "hexagonal"], "E_CONFIG"),
        (["frobnicate"], "E_FLAGS"),
        ([], "E_FLAGS"),
    ]
    for args, want in cases:
        code, _, err = run(args, tmp_path)
        assert code == CODES[want], (args, code, err)
        assert json.loads(err.strip().splitlines()[-1])["error"] == want
    for body, msg in [("x,y,z,weight\n1,0,0\n", "expected 4 columns on line 2"),
                      ("x,y,z,weight\n1,0,zero,1\n", "malformed number 'zero' on line 2"),
                      ("a,b,c,d\n1,0,0,1\n", "header must be 'x,y,z,weight' or 'lon,lat,area,value'"),
                      ("", "missing header line")]:
        (tmp_path / "bad.csv").write_text(body)
        code, _, err = run(["sum", "--kernel", "laplace", "--particles", "bad.csv"], tmp_path)
        assert code == CODES["E_CSV"] and msg in err
    code, _, err = run(["sum", "--kernel", "laplace", "--particles", "missing.csv"], tmp_path)
    assert code == CODES["E_IO"] and "cannot open input file: missing.csv" in err
    code, _, _ = run(["grid", "--kind", "icosahedral", "--level", "2", "-o", "no/such/dir/g.csv"], tmp_path)
    assert code == CODES["E_IO"]
    assert run(["--help"], tmp_path)[0] == 0


def test_particle_formats_autodetected(tmp_path):
    """test_cli.cpp: 'particle CSV formats are auto-detected and round-trip'."""
    (tmp_path / "a.csv").write_text("x,y,z,weight\n1,0,0,2.5\n0,1,0,-1\n0,0,1,0.25\n")
    assert run(["convert", "--particles", "a.csv", "-o", "a2.csv"], tmp_path)[0] == 0
    h, r = read_csv(tmp_path / "a2.csv")
    assert h == "x,y,z,weight" and r.shape == (3, 4) and r[0, 3] == 2.5
    (tmp_path / "b.csv").write_text("lon,lat,area,value\n0,0,0.5,3\n90,0,0.5,1\n")
    assert run(["convert", "--particles", "b.csv", "-o", "b2.csv"], tmp_path)[0] == 0
    _, r = read_csv(tmp_path / "b2.csv")
    assert r.shape == (2, 4)
    assert abs(r[0, 0] - 1.0) < 1e-15 and abs(r[1, 1] - 1.0) < 1e-15
    assert r[0, 3] == 1.5  # value * area
    # un-normalized x,y,z are projected to the sphere (normalized, geometry.hpp:24)
    (tmp_path / "c.csv").write_text("x,y,z,weight\n3,0,4,1\n")
    run(["convert", "--particles", "c.csv", "-o", "c2.csv"], tmp_path)
    _, r = read_csv(tmp_path / "c2.csv")
    np.testing.assert_array_equal(r[0, :3], [3 / 5, 0, 4 / 5])


def test_floats_have_17_significant_digits(tmp_path):
    """test_cli.cpp: format_double(1/3) == '0.33333333333333331'; round trip exact."""
    (tmp_path / "t.csv").write_text("x,y,z,weight\n1,0,0,0.333333333333333314829616256247\n0,0,1,2562\n")
    run(["convert", "--particles", "t.csv", "-o", "t2.csv"], tmp_path)
    lines = open(tmp_path / "t2.csv").read().splitlines()
    assert lines[1].endswith(",0.33333333333333331") and lines[2].endswith(",2562")


CSV_CASES = {
    "plain": "x,y,z,weight\n1,0,0,2.5\n0,1,0,-1\n",
    "crlf_spaces": "x, y ,z,weight \r\n 3 , 0,4 ,1e-3\r\n\r\n0,0,-2,  7\r\n",
    "blank_lines": "x,y,z,weight\n\n1,2,3,4\n\n\n-1,0.5,0.25,1e300\n",
    "trailing_comma": "x,y,z,weight,\n1,2,3,4,\n",
    "lonlat": "lon,lat,area,value\n0,0,0.5,3\n-179.5,89.999,1e-6,-2\n33.3,-12.5,0.125,0.5\n",
    "hex_inf": "x,y,z,weight\n0x1p-1,0,1,inf\n1,1,1,-0\n",
    "blank_first_line": "\nx,y,z,weight\n1,0,0,1\n",
    "short_row": "x,y,z,weight\n1,0,0\n",
    "empty_field": "x,y,z,weight\n1,,0,1\n",
    "bad_number": "x,y,z,weight\n1,0,1e,1\n",
    "overflow": "x,y,z,weight\n1,0,0,1e999\n",
    "bad_header": "lon,lat,value,area\n1,0,0,1\n",
    "header_only": "x,y,z,weight\n",
    "empty": "",
}


@pytest.mark.parametrize("case", sorted(CSV_CASES))
def test_particle_csv_matches_reference_reader(tmp_path, monkeypatch, case):
    """`convert` reads particle CSVs exactly like the reference's read_particles_csv
    (io.cpp:166-185, compiled into oracle/_ref): the same particles bit for bit, or the same
    error code and message."""
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    (tmp_path / "in.csv").write_text(CSV_CASES[case])
    code, _, err = run(["convert", "--particles", "in.csv", "-o", "out.csv"], tmp_path)
    monkeypatch.chdir(tmp_path)  # same relative path in both messages
    try:
        xyz, w = ref.read_particles_csv("in.csv")
    except ValueError as ex:
        want_code, want_msg = str(ex).split(": ", 1)
        got = json.loads(err.strip().splitlines()[-1])
        assert code == CODES[want_code] and got["error"] == want_code and got["message"] == want_msg, (got, str(ex))
        return
    assert code == 0, err
    lines = open(tmp_path / "out.csv").read().splitlines()
    assert lines[0] == "x,y,z,weight" and len(lines) == 1 + len(w)
    got = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]]).reshape(-1, 4)
    np.testing.assert_array_equal(got[:, :3], xyz)
    np.testing.assert_array_equal(got[:, 3], w)


# ---- GPU ------------------------------------------------------------------------------


@pytest.mark.gpu
def test_sum_against_direct(tmp_path):
    """test_cli.cpp: 'sum against the built-in direct reference'."""
    code, out, err = run(["sum", "--method", "csfmm", "--kernel", "laplace", "--grid", "icosahedral:4",
                          "--reference", "direct", "--report", "sum_report.json"], tmp_path)
    assert code == 0, err
    rep = json.load(open(tmp_path / "sum_report.json"))
    assert rep == json.loads(out)
    assert rep["N"] == 2562 and rep["relative_l2_error"] < 1e-5 and rep["timings"]["total"] > 0
    t = rep["timings"]
    assert t["tree_build"] + t["upward"] + t["traversal"] + t["downward"] >= 0.9 * t["total"]
    assert (rep["kernel"], rep["method"], rep["mac"], rep["degree"], rep["n0"]) == ("laplace", "csfmm", 0.7, 6, 144)


@pytest.mark.gpu
@pytest.mark.parametrize("grid,kernel,method", [("icosahedral:4", "laplace", "csfmm"),
                                                ("cubed_sphere:5", "sal", "csfmm"),
                                                ("latlon:4", "biot_savart", "csfmm"),
                                                ("icosahedral:3", "biharmonic", "cstc"),
                                                ("cubed_sphere:3", "laplace", "direct")])
def test_sum_matches_reference(tmp_path, grid, kernel, method):
    """`sum -o` writes the reference's summed_potential on the reference's grid with the
    built-in Y_4^3 weights (cli.cpp:147-163)."""
    code, out, err = run(["sum", "--method", method, "--kernel", kernel, "--grid", grid, "--stats", "-o", "phi.csv"],
                         tmp_path)
    assert code == 0, err
    rep = json.loads(out)
    kind, level = grid.split(":")
    xyz, areas = ref.grid(kind, int(level))
    w = ref.sph_harm(4, 3, xyz) * areas
    m = {"direct": 0, "cstc": 1, "csfmm": 2}[method]
    r, rst = ref.summed(m, xyz, xyz, w, kernel)
    h, rows = read_csv(tmp_path / "phi.csv")
    dim = 3 if kernel == "biot_savart" else 1
    assert h == ("x,y,z,phi,phi_y,phi_z" if dim == 3 else "x,y,z,phi")
    np.testing.assert_array_equal(rows[:, :3], xyz)
    g = rows[:, 3:].reshape(-1)
    assert np.sqrt(np.sum((g - r) ** 2) / np.sum(r ** 2)) < 1e-10
    assert [rep["interactions"][k] for k in ("pp", "pc", "cp", "cc")] == [int(v) for v in rst[5:9]]
    if method == "csfmm":
        st = ref.Tree(xyz, 6, 144).export()
        leaves = st["ints"][:, 5] == 0
        sizes = (st["ints"][:, 2] - st["ints"][:, 1])[leaves]
        assert rep["tree"]["leaf_count"] == int(leaves.sum()) == rep["target_tree"]["leaf_count"]
        assert rep["tree"]["leaf_size_histogram"] == np.bincount(sizes).tolist()


@pytest.mark.gpu
def test_reference_potentials_from_csv(tmp_path):
    """test_cli.cpp: 'reference potentials can come from a CSV file' (+ E_DIM on a row mismatch)."""
    assert run(["sum", "--method", "direct", "--kernel", "laplace", "--grid", "icosahedral:2", "-o", "ref.csv"],
               tmp_path)[0] == 0
    code, out, _ = run(["sum", "--method", "csfmm", "--kernel", "laplace", "--grid", "icosahedral:2",
                        "--reference", "ref.csv", "--report", "r.json"], tmp_path)
    assert code == 0 and json.load(open(tmp_path / "r.json"))["relative_l2_error"] < 1e-5
    code, _, _ = run(["sum", "--method", "csfmm", "--kernel", "laplace", "--grid", "icosahedral:3",
                      "--reference", "ref.csv"], tmp_path)
    assert code == CODES["E_DIM"]
    code, _, _ = run(["sum", "--method", "csfmm", "--kernel", "biot_savart", "--grid", "icosahedral:2",
                      "--reference", "ref.csv"], tmp_path)
    assert code == CODES["E_DIM"]


@pytest.mark.gpu
def test_sum_particles_file(tmp_path):
    """--particles in both formats, against the reference on the same particles."""
    rng = np.random.default_rng(11)
    p = rng.normal(size=(3000, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    wts = rng.normal(size=3000)
    with open(tmp_path / "p.csv", "w") as f:
        f.write("x,y,z,weight\n")
        for (x, y, z), v in zip(p, wts):
            f.write(f"{float(x)!r},{float(y)!r},{float(z)!r},{float(v)!r}\n")
    code, out, err = run(["sum", "--kernel", "sal", "--degree", "8", "--mac", "0.5", "--particles", "p.csv", "-o",
                          "o.csv"], tmp_path)
    assert code == 0, err
    _, rows = read_csv(tmp_path / "o.csv")
    xyz = rows[:, :3]
    r, _ = ref.summed(2, xyz, xyz, wts, "sal", mac=0.5, degree=8)
    assert np.sqrt(np.sum((rows[:, 3] - r) ** 2) / np.sum(r ** 2)) < 1e-10


@pytest.mark.gpu
def test_bench(tmp_path):
    code, out, err = run(["bench", "--grid-kind", "cubed_sphere", "--levels", "4,5", "--methods", "csfmm,cstc",
                          "--kernel", "laplace", "--out-prefix", "b"], tmp_path)
    assert code == 0, err
    rep = json.load(open(tmp_path / "b.json"))
    assert rep["subcommand"] == "bench" and len(rep["rows"]) == 4
    assert set(rep["exponents"]) == {"csfmm", "cstc"}
    h = open(tmp_path / "b.csv").readline().strip()
    assert h == "method,level,N,seconds"
