"""CPU: the Python input generator (paper_2508_13550_b200/grids.py) against the reference's
own build_grid / real_sph_harm (oracle/_ref).  The benchmark configs hand the same arrays
to both engines, so exact agreement is not required for parity — but the generator is
checked anyway: cubed-sphere centres and areas bit for bit, harmonics to 1e-12."""
import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200.grids import cubed_sphere, real_sph_harm


@pytest.mark.parametrize("level", [0, 3, 5])
def test_cubed_sphere_matches_reference(level):
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    xyz, a = cubed_sphere(level)
    rx, ra = ref.grid("cubed_sphere", level)
    assert xyz.shape == rx.shape
    np.testing.assert_array_equal(xyz, rx)
    np.testing.assert_array_equal(a, ra)
    assert abs(a.sum() - 4 * np.pi) < 1e-12


@pytest.mark.parametrize("l,m", [(0, 0), (1, -1), (4, 3), (12, -7), (32, 32)])
def test_real_sph_harm_matches_reference(l, m):
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    xyz, _ = cubed_sphere(3)
    np.testing.assert_allclose(real_sph_harm(l, m, xyz), ref.sph_harm(l, m, xyz), rtol=1e-12, atol=1e-14)
