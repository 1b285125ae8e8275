"""Seeded input generators (nc_inputs): separation, determinism, table shapes."""
import numpy as np
import pytest

from nc_inputs import CONFIGS, synthetic_tables
from nc_inputs.layouts import fibonacci, haar_rotation, min_arc_distance


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_layouts_separated_and_deterministic(name):
    cfg = CONFIGS[name]
    a = cfg.centers()
    assert a.shape == (cfg.N, 3)
    np.testing.assert_allclose(np.linalg.norm(a, axis=1), 1.0, atol=1e-15)
    # PAPER.md:641-646 (§3): centre arc distance at least 3 eps
    assert min_arc_distance(a) >= 3 * cfg.eps * (1 - 1e-12)
    np.testing.assert_array_equal(a, cfg.centers())


def test_c5_fibonacci_separation():
    cfg = CONFIGS["C5"]
    a = cfg.centers()
    assert min_arc_distance(a) >= 3 * cfg.eps


def test_haar_rotation_is_rotation():
    q = haar_rotation(np.random.default_rng(0))
    np.testing.assert_allclose(q.T @ q, np.eye(3), atol=1e-14)
    assert abs(np.linalg.det(q) - 1) < 1e-14


def test_fibonacci_rotation_preserves_distances():
    a = fibonacci(100)
    b = fibonacci(100, seed=3)
    np.testing.assert_allclose(a @ a.T, b @ b.T, atol=1e-13)


def test_synthetic_tables_shapes():
    t = synthetic_tables(0, 0.02, seed=1)
    assert (t.K, t.Kstar, t.p) == (136, 512, 120)
    # every node lies on the patch: arc distance from the pole <= eps
    assert np.arccos(np.clip(t.zhat[:, 2], -1, 1)).max() <= 0.02 + 1e-15
    assert np.arccos(np.clip(t.shat[:, 2], -1, 1)).max() <= 0.02 + 1e-15
