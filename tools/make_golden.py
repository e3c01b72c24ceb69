"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the unmodified
/root/reference library built by `make -C oracle ref`).  Run in this container:

    python tools/make_golden.py

The fixtures pin the C restatement (oracle/csfmm_oracle.c) and the B200 engine when the
reference is not available (GPU box, fresh checkouts).  Inputs are regenerated in the
tests from grids.cubed_sphere (bit-identical to the reference's build_grid, see
tests/test_grids.py) except the icosahedral points, which are stored.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2508_13550_b200 import configs  # noqa: E402
from paper_2508_13550_b200.grids import cubed_sphere  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
KERNELS = ["laplace", "biharmonic", "biot_savart", "sal"]


def kernels_fixture():
    rng = np.random.Generator(np.random.MT19937(7))
    x = rng.standard_normal((64, 3))
    x /= np.linalg.norm(x, axis=1)[:, None]
    y = rng.standard_normal((64, 3))
    y /= np.linalg.norm(y, axis=1)[:, None]
    special = np.array([[0, 0, 1], [0, 0, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    xs = np.vstack([np.repeat(special[:1], 5, 0), x, x[:8]])
    ys = np.vstack([special, y, x[:8] * (1 + 1e-16)])  # near-coincident pairs hit the guard
    out = {"x": xs, "y": ys}
    for k in KERNELS:
        ok = np.zeros(len(xs), bool)
        val = np.zeros((len(xs), 3))
        for i in range(len(xs)):
            ok[i], val[i] = ref.kernel_try_eval(k, xs[i], ys[i])
        out[f"{k}_ok"] = ok
        out[f"{k}_val"] = val
    u = np.concatenate([np.linspace(-1.0, 1.0, 2001), [0.0, 0.5, 1.0, 1 - 1e-16, 1 - 1e-8, 0.5 + 1e-12, -1e-16],
                        1.0 - np.logspace(-15, -0.3, 400)])
    out["dilog_u"] = u
    out["dilog_v"] = np.array([ref.dilog(v) for v in u])
    bx = np.concatenate([np.linspace(-1, 1, 41), [1 - 1e-15, -1 + 5e-15, 0.3]])
    for deg in (4, 6, 10):
        out[f"bary{deg}_x"] = bx
        out[f"bary{deg}"] = np.array([ref.bary_basis_1d(deg, v) for v in bx])
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def tree_fixture():
    xyz, a = cubed_sphere(4)
    w = ref.sph_harm(4, 3, xyz) * a
    out = {}
    for tag, deg, n0, shrink in [("s", 6, 32, True), ("ns", 4, 25, False)]:
        t = ref.Tree(xyz, deg, n0, shrink)
        e = t.export()
        for k in ("perm", "ints", "dbls", "proxy"):
            out[f"{tag}_{k}"] = e[k]
        out[f"{tag}_pw"] = t.upward(w)
        lists = ref.lists(t, t, 0.7, n0)
        for k, v in lists.items():
            out[f"{tag}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "tree_cs4.npz"), **out)


def csfmm_fixture():
    out = {}
    ico, ia = ref.grid("icosahedral", 3)
    out["ico3_xyz"], out["ico3_area"] = ico, ia
    cs4, ca = cubed_sphere(4)
    cases = []
    for gname, xyz, a in (("ico3", ico, ia), ("cs4", cs4, ca)):
        w = ref.sph_harm(4, 3, xyz) * a
        for k in KERNELS:
            for deg, mac, n0 in ((6, 0.7, -1), (8, 0.6, 40)):
                tag = f"{gname}_{k}_{deg}"
                v, st = ref.csfmm(xyz, xyz, w, k, mac=mac, degree=deg, n0=n0)
                out[f"{tag}_phi"] = v
                out[f"{tag}_counts"] = st[5:9].astype(np.int64)
                out[f"{tag}_params"] = np.array([deg, mac, n0], float)
                cases.append(tag)
        out[f"{gname}_direct_sal"] = ref.direct(xyz, xyz, w, "sal")
        out[f"{gname}_direct_bs"] = ref.direct(xyz, xyz, w, "biot_savart")
    # targets != sources (test_summation.cpp:285-296 shape)
    v, st = ref.csfmm(cs4, ico, ref.sph_harm(4, 3, ico) * ia, "laplace")
    out["cross_phi"], out["cross_counts"] = v, st[5:9].astype(np.int64)
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(OUT, "csfmm_small.npz"), **out)


def c1_fixture():
    wl = configs.make("c1")
    v, st = ref.csfmm(wl.xyz, wl.xyz, wl.weights, wl.kernel, mac=wl.mac, degree=wl.degree, n0=wl.n0)
    d = ref.direct(wl.xyz, wl.xyz, wl.weights, wl.kernel)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), phi=v, counts=st[5:9].astype(np.int64),
                        tree=st[9:15].astype(np.int64), direct=d)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    kernels_fixture()
    tree_fixture()
    csfmm_fixture()
    c1_fixture()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
