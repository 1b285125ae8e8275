"""Pins of the oracle's off-surface field (NEXT-3; oracle.green_off / oracle.offsurface).

The off-surface Neumann Green's functions eq:Gintoffsurface / eq:Gextoffsurface are
checked against what the mathematics fixes, not against a retyped formula:
  * the defining Neumann property on the sphere: d/dr G_I(x, x') = -1 and d/dr G_E(x, x') = 0 at |x| = 1, x != x'
    (the interior Neumann function's flux 4 pi / |dOmega| = 1; the exterior one carries no flux through the sphere);
  * G_I(0, x') = 2 for every x' on the sphere (the step behind v(0) = 2 I_sigma);
  * continuity up to the surface: the off-surface form at |x| = 1 equals the on-surface three-term form
    (eq:Gintonsurface / eq:Gextonsurface) that the matvec oracle uses;
  * harmonicity in x (a second-order finite-difference Laplacian vanishes to O(h^2));
  * the exterior far field |x| G_E(x, x') -> 1 (R3 / SURVEY A3), hence |x| u -> sum rho.
A dropped term, a wrong sign or a swapped argument fails at least one of them by orders of magnitude."""
import numpy as np
import pytest

from nc_inputs import make_centers, random_coeffs, synthetic_tables
from oracle import oracle as O


def _unit(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


@pytest.mark.parametrize("kind,expect", [(0, -1.0), (1, 0.0)])
def test_neumann_derivative_on_sphere(kind, expect):
    rng = np.random.default_rng(11)
    e, xp = _unit(rng, 40), _unit(rng, 40)
    h = 1e-5
    # one-sided for the exterior (x must stay outside), central for the interior (formula defined both sides)
    if kind == 0:
        dr = (O.green_off(kind, (1 + h) * e, xp) - O.green_off(kind, (1 - h) * e, xp)) / (2 * h)
    else:
        dr = (-3 * O.green_off(kind, e * (1 + 1e-12), xp) + 4 * O.green_off(kind, (1 + h) * e, xp)
              - O.green_off(kind, (1 + 2 * h) * e, xp)) / (2 * h)
    assert np.max(np.abs(dr - expect)) < 1e-6


def test_interior_value_at_origin():
    rng = np.random.default_rng(12)
    xp = _unit(rng, 50)
    assert np.max(np.abs(O.green_off(0, np.zeros((50, 3)), xp) - 2.0)) < 1e-15


@pytest.mark.parametrize("kind", [0, 1])
def test_continuity_to_on_surface_form(kind):
    rng = np.random.default_rng(13)
    x, xp = _unit(rng, 60), _unit(rng, 60)
    assert np.max(np.abs(O.green_off(kind, x, xp) - O.green(kind, x, xp)) / np.abs(O.green(kind, x, xp))) < 1e-12


@pytest.mark.parametrize("kind,radius", [(0, 0.6), (1, 1.7)])
def test_harmonic_in_x(kind, radius):
    rng = np.random.default_rng(14)
    x, xp = radius * _unit(rng, 20), _unit(rng, 20)
    h = 1e-3
    lap = -6 * O.green_off(kind, x, xp)
    for a in range(3):
        dv = np.zeros(3)
        dv[a] = h
        lap = lap + O.green_off(kind, x + dv, xp) + O.green_off(kind, x - dv, xp)
    lap /= h * h
    assert np.max(np.abs(lap)) < 1e-4   # O(h^2) truncation of a field of size ~1


def test_exterior_far_field():
    rng = np.random.default_rng(15)
    e, xp = _unit(rng, 30), _unit(rng, 30)
    for R, tol in ((1e3, 2e-3), (1e5, 2e-5)):
        assert np.max(np.abs(R * O.green_off(1, R * e, xp) - 1.0)) < tol


def test_offsurface_field_origin_and_far_field():
    """v(0) = 2 sum rho (interior) and |x| u -> sum rho (exterior) for the compressed densities of a layout."""
    c = make_centers("uniform", 25, 0.05, seed=5)
    for kind in (0, 1):
        tab = synthetic_tables(kind, 0.05, seed=8)
        x = random_coeffs(25, tab.K, 9)
        total = float(np.sum(O.outgoing(tab.T, x)))
        if kind == 0:
            v, dmin = O.offsurface(0, c, tab, x, np.zeros((1, 3)))
            assert abs(v[0] - 2 * total) <= 1e-13 * max(1.0, abs(total)) * 50
            assert abs(dmin[0] - 1.0) < 1e-12   # skeleton nodes lie on the unit sphere
        else:
            p = 1e5 * _unit(np.random.default_rng(3), 4)
            u, _ = O.offsurface(1, c, tab, x, p)
            assert np.max(np.abs(1e5 * u - total)) < 1e-4 * max(1.0, abs(total))

# oracle.mfpt_field (eq:vtilde) is pinned by tests/test_mfpt_oracle.py: Delta v-bar = -1 and its ball averages.
