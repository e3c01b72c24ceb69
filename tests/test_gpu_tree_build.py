"""GPU: the label-then-sort tree build (tree.cu build_tree, the default) against the
level-synchronous build it replaced (CSFS_B200_TREE=levels): the same trees bit for bit —
perm, topology, bounds, centres, radii, proxy points — the same lists and the same
potentials, on inputs that stress the parts that changed: particles in random input order
(the per-quadrant atomics see no coherence), clustered blobs (deep unbalanced trees, more
than one batch of speculative levels), duplicates (the extent stop), n0 = 1, tiny sets,
empty face roots, targets != sources (two trees per call).  The reference comparisons of
the new build are the rest of the -m gpu suite (test_gpu_parity / _edge / _fullsize)."""
import os

import numpy as np
import pytest

from paper_2508_13550_b200 import Kernel, ParticleSet, SumStats, TraversalConfig, configs

pytestmark = pytest.mark.gpu


def unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def run(engine, txyz, sxyz, w, kernel, mode, **cfg):
    old = os.environ.get("CSFS_B200_TREE")
    if mode:
        os.environ["CSFS_B200_TREE"] = mode
    else:
        os.environ.pop("CSFS_B200_TREE", None)
    try:
        st = SumStats()
        c = TraversalConfig(**cfg)
        phi = engine.csfmm_sum(ParticleSet(txyz, np.zeros(len(txyz))), ParticleSet(sxyz, w), Kernel.parse(kernel),
                               c, st).values
        trees = [engine.tree_export(0)]
        if st.shared_tree == 0:
            trees.append(engine.tree_export(1))
        return phi, trees, engine.lists_export(), st
    finally:
        if old is None:
            os.environ.pop("CSFS_B200_TREE", None)
        else:
            os.environ["CSFS_B200_TREE"] = old


def same(engine, txyz, sxyz, w, kernel="laplace", **cfg):
    a = run(engine, txyz, sxyz, w, kernel, None, **cfg)
    b = run(engine, txyz, sxyz, w, kernel, "levels", **cfg)
    assert np.array_equal(a[0], b[0])  # potentials bitwise
    assert len(a[1]) == len(b[1])
    for ta, tb in zip(a[1], b[1]):
        assert ta["depth"] == tb["depth"]
        for k in ("perm", "ints", "dbls", "proxy"):
            assert np.array_equal(ta[k], tb[k]), k
    for k in ("pp", "pc", "cp", "cc"):
        assert np.array_equal(a[2][k], b[2][k]), k
    return a[3]


def blobs(n, seed, k=5, spread=0.05):
    rng = np.random.default_rng(seed)
    centres = unit(rng.normal(size=(k, 3)))
    m = int(0.9 * n)
    pts = centres[rng.integers(0, k, m)] + spread * rng.normal(size=(m, 3))
    pts = np.concatenate([pts, rng.normal(size=(n - m, 3))])
    return unit(pts), rng.normal(size=n)


def test_grid_in_order_and_shuffled(engine):
    wl = configs.make("c2")
    same(engine, wl.xyz, wl.xyz, wl.weights, "laplace", mac=wl.mac, degree=wl.degree, n0=wl.n0)
    p = np.random.default_rng(5).permutation(wl.n)
    same(engine, wl.xyz[p], wl.xyz[p], wl.weights[p], "laplace", mac=wl.mac, degree=wl.degree, n0=wl.n0)


def test_clustered_deep(engine):
    x, w = blobs(60000, 11, spread=0.01)
    st = same(engine, x, x, w, "sal", degree=6, mac=0.6, n0=8)
    assert st.tgt_depth >= 10


def test_duplicates_n0_1(engine):
    rng = np.random.default_rng(12)
    base = unit(rng.normal(size=(2000, 3)))
    x = np.concatenate([base, base[:300], base[:50]])
    same(engine, x, x, rng.normal(size=len(x)), "laplace", degree=4, n0=1)


@pytest.mark.parametrize("n", [1, 2, 5, 40])
def test_tiny(engine, n):
    x, w = blobs(n, 20 + n)
    same(engine, x, x, w, "biot_savart", degree=4, n0=2)


def test_one_face_and_two_trees(engine):
    rng = np.random.default_rng(13)
    t = unit(np.array([0, 0, 1.0]) + 0.2 * rng.normal(size=(7000, 3)) * [1, 1, 0.1])
    s, w = blobs(20000, 14)
    st = same(engine, t, s, w, "biharmonic", degree=6, n0=20)
    assert st.shared_tree == 0


def test_no_shrink(engine):
    x, w = blobs(30000, 15)
    same(engine, x, x, w, "laplace", degree=5, n0=30, shrink=False)
