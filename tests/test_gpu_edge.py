"""GPU parity on the inputs grids never produce — the edge cases of the reference's own
tests (test_cluster_tree.cpp / test_summation.cpp) and the ones the B200 design has to
get right by construction: irregular clustered point sets (deep, unbalanced trees, empty
face roots), tiny sets, duplicate / near-coincident points (the coincidence guard and the
extent stop), points exactly on cube-face edges and corners (face ties), n0 = 1, the
highest supported degree, target sets much smaller or larger than the source set, SAL
with non-default parameters (including c1 = 1 - b0 = 0, the log-only functor), and the
symmetric-pair paths with every kernel.  Each case: the reference's own csfmm_sum
(oracle/_ref) on the same inputs, potentials within the 1e-10 bar, lists bit-exact."""
import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200 import Kernel, ParticleSet, SalParams, SumStats, TraversalConfig

pytestmark = pytest.mark.gpu

PARITY = 1e-10


def rel_l2(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b ** 2), 1e-300)))


def unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def blobs(n, seed, k=5, spread=0.05):
    """k Gaussian blobs + 10% uniform background: strongly non-uniform density."""
    rng = np.random.default_rng(seed)
    centres = unit(rng.normal(size=(k, 3)))
    m = int(0.9 * n)
    pts = centres[rng.integers(0, k, m)] + spread * rng.normal(size=(m, 3))
    pts = np.concatenate([pts, rng.normal(size=(n - m, 3))])
    return unit(pts), rng.normal(size=n)


def check(engine, txyz, sxyz, sw, kernel, sal=None, **cfg):
    c = TraversalConfig(**cfg)
    st = SumStats()
    k = Kernel.parse(kernel, sal) if sal else Kernel.parse(kernel)
    g = engine.csfmm_sum(ParticleSet(txyz, np.zeros(len(txyz))), ParticleSet(sxyz, sw), k, c, st).values
    sal_v = None if sal is None else [sal.a1, sal.b0, sal.b1, sal.rho_ratio]
    r, rst = ref.csfmm(txyz, sxyz, sw, kernel, mac=c.mac, degree=c.degree, n0=c.n0, shrink=c.shrink, sal=sal_v)
    assert rel_l2(g, r) < PARITY, (kernel, cfg, rel_l2(g, r))
    assert (st.pp, st.pc, st.cp, st.cc) == tuple(int(v) for v in rst[5:9])
    return st


@pytest.mark.parametrize("kernel", ["laplace", "biharmonic", "biot_savart", "sal"])
def test_clustered_points(engine, kernel):
    """Deep, unbalanced trees with PC entries and symmetric pairs of every size <= 256."""
    x, w = blobs(40000, 1)
    st = check(engine, x, x, w, kernel, degree=7, mac=0.6, n0=48)
    assert st.pc > 0 and st.tgt_depth >= 6
    if kernel != "biot_savart":
        assert st.symmetric_pairs > 0


def test_blobs_on_one_face(engine):
    """All points near +z: five of the six face roots are empty (kept, never split)."""
    rng = np.random.default_rng(2)
    x = unit(np.array([0, 0, 1.0]) + 0.2 * rng.normal(size=(5000, 3)) * [1, 1, 0.1])
    check(engine, x, x, rng.normal(size=len(x)), "sal", degree=6, n0=20)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 33])
def test_tiny_sets(engine, n):
    x, w = blobs(n, 3 + n)
    for kernel in ("laplace", "biot_savart"):
        check(engine, x, x, w, kernel, degree=4, n0=2)


def test_duplicates_and_near_coincident(engine):
    """Exact duplicates (guard skips them; the extent stop ends the split) and pairs closer
    than the 1e-14 guard threshold, next to ordinary points."""
    rng = np.random.default_rng(4)
    base = unit(rng.normal(size=(3000, 3)))
    dup = base[:400].copy()                                   # exact duplicates
    near = unit(base[400:600] + 1e-9 * rng.normal(size=(200, 3)))  # omc ~ 1e-18..1e-17: guarded
    mid = unit(base[600:800] + 3e-7 * rng.normal(size=(200, 3)))   # omc ~ 1e-13: evaluated
    x = np.concatenate([base, dup, near, mid])
    w = rng.normal(size=len(x))
    for kernel in ("laplace", "biharmonic", "biot_savart", "sal"):
        check(engine, x, x, w, kernel, degree=6, n0=16)
    # many copies of one point: a leaf that cannot be split (extent < 1e-13)
    x2 = np.concatenate([np.repeat(base[:1], 300, axis=0), base[1:500]])
    check(engine, x2, x2, rng.normal(size=len(x2)), "laplace", degree=5, n0=8)


def test_face_edges_and_corners(engine):
    """Points exactly on the cube-face boundaries (|x| = |y|, |x| = |z|, corners): the
    face_project argmax ties go to the lowest face id in both implementations."""
    s = 1 / np.sqrt(2)
    t = 1 / np.sqrt(3)
    pts = []
    for a in (-1, 1):
        for b in (-1, 1):
            pts += [[a * s, b * s, 0], [a * s, 0, b * s], [0, a * s, b * s]]
            for c in (-1, 1):
                pts.append([a * t, b * t, c * t])
    edge = np.array(pts)
    rng = np.random.default_rng(6)
    x = np.concatenate([edge, unit(rng.normal(size=(2000, 3)))])
    check(engine, x, x, rng.normal(size=len(x)), "laplace", degree=6, n0=10)
    check(engine, x, x, rng.normal(size=len(x)), "sal", degree=8, n0=40, mac=0.5)


def test_n0_one_and_high_degree(engine):
    x, w = blobs(3000, 7)
    check(engine, x, x, w, "laplace", degree=3, n0=1)
    check(engine, x, x, w, "sal", degree=20, n0=600, mac=0.5)


def test_asymmetric_target_source_sizes(engine):
    sx, sw = blobs(30000, 8)
    tx, _ = blobs(1, 9)
    check(engine, tx, sx, sw, "sal", degree=6)
    tx, _ = blobs(50000, 10)
    sx, sw = blobs(500, 11)
    check(engine, tx, sx, sw, "biot_savart", degree=6, n0=30)


@pytest.mark.parametrize("sal", [SalParams(a1=-1.0, b0=0.3, b1=2.0, rho_ratio=0.2),
                                 SalParams(b0=1.0),               # c1 = 0: the log-only functor
                                 SalParams(a1=6.1, b1=6.1)])      # c2 = 0: no log term
def test_sal_parameters(engine, sal):
    x, w = blobs(20000, 12)
    check(engine, x, x, w, "sal", sal=sal, degree=8, mac=0.6, n0=64)


@pytest.mark.parametrize("kernel", ["laplace", "sal", "biot_savart"])
def test_points_off_the_unit_sphere(engine, kernel):
    """Radii scattered in [0.98, 1.02]: the coincidence-guard elision assumes unit vectors, so
    the engine keeps the guard on every entry (k_face flags the tree) and matches the
    reference, which skips pairs with 1 - x.y < 1e-14 whatever their distance."""
    rng = np.random.default_rng(11)
    x = unit(rng.normal(size=(20000, 3))) * rng.uniform(0.98, 1.02, size=(20000, 1))
    x[:50] = x[50:100] * (1.0 / np.einsum("ij,ij->i", x[50:100], x[50:100]))[:, None]  # x.y = 1 exactly-ish
    w = rng.normal(size=20000)
    check(engine, x, x, w, kernel, degree=6, mac=0.7, n0=64)
