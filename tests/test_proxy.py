"""The step-4 proxy rule of NC_HIER handles (R36; nc_proxy_rule, host arithmetic in libnc, no GPU).

Far levels of step 4 are evaluated at n proxy points per patch and carried to the K* Zernike
nodes by one matrix Int.  Pinned here against what the mathematics fixes: Int reproduces every polynomial of total
degree <= deg in the tangent-plane coordinates exactly (monomials, not the rule's own Chebyshev basis); the
interpolation error of the Green's function of a point source at the calibrated distance kappa h is at most the
requested tolerance, and it falls geometrically with the distance; the proxies lie on the unit sphere inside the
node disk; the Lebesgue constant of the map is small."""
import os

import numpy as np
import pytest

from nc_inputs.tables import load_tables
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


@pytest.fixture(scope="module", params=["C1", "C5"])
def zhat(request):
    return load_tables(os.path.join(ROOT, "tables", "data", f"{request.param}.npz")).zhat


def test_proxy_rule_reproduces_polynomials(zhat):
    deg = 11
    pts, Int, kappa, h = _nc().proxy_rule(zhat, deg=deg, nring=6, cphi=24.0, tol=1e-8)
    n = pts.shape[0]
    assert n == 96 and Int.shape == (zhat.shape[0], n)
    rng = np.random.default_rng(5)
    for _ in range(4):   # a random polynomial of total degree <= deg in (u / h, v / h), monomial basis
        c = rng.standard_normal((deg + 1, deg + 1))
        def f(u, v):
            return sum(c[a, b] * (u / h) ** a * (v / h) ** b for a in range(deg + 1) for b in range(deg + 1 - a))
        fn = f(zhat[:, 0], zhat[:, 1])
        fp = f(pts[:, 0], pts[:, 1])
        assert np.max(np.abs(Int @ fp - fn)) <= 1e-11 * np.max(np.abs(fn))


@pytest.mark.parametrize("rule", [(8, 4, 24.0), (11, 6, 24.0)])
def test_proxy_points_geometry_and_lebesgue(zhat, rule):
    pts, Int, kappa, h = _nc().proxy_rule(zhat, *rule)
    np.testing.assert_allclose(np.linalg.norm(pts, axis=1), 1.0, atol=1e-15)
    assert np.max(np.hypot(pts[:, 0], pts[:, 1])) <= h
    assert np.max(np.hypot(zhat[:, 0], zhat[:, 1])) <= h
    assert np.abs(Int).sum(axis=1).max() < 10.0          # Lebesgue constant of the least-squares map
    assert np.min(pts[:, 2]) > 0.0


@pytest.mark.parametrize("kind", [0, 1])
def test_proxy_rule_green_error_at_kappa(zhat, kind):
    """Point sources at the calibrated distance kappa h (and beyond): the oracle's G (eq:Gintonsurface /
    eq:Gextonsurface, the literal three-term forms) interpolated through the proxies stays within the tolerance
    relative to max G over the nodes; twice as far it is much smaller."""
    tol = 1e-8
    pts, Int, kappa, h = _nc().proxy_rule(zhat, tol=tol)
    assert 2.0 <= kappa <= 8.0
    for D, bound in ((kappa, 2 * tol), (2 * kappa, 2 * tol * 1e-2)):
        th = D * h
        if th >= 2.5:
            continue
        worst = 0.0
        for a in range(7):
            ph = 2 * np.pi * (a + 0.3) / 7
            s = np.array([[np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)]])
            gn = O.green(kind, zhat, np.repeat(s, zhat.shape[0], axis=0))
            gp = O.green(kind, pts, np.repeat(s, pts.shape[0], axis=0))
            worst = max(worst, np.max(np.abs(Int @ gp - gn)) / np.max(np.abs(gn)))
        assert worst <= bound, (D, worst)


def test_proxy_kappa_grows_with_tighter_tolerance(zhat):
    k1 = _nc().proxy_rule(zhat, tol=1e-6)[2]
    k2 = _nc().proxy_rule(zhat, tol=1e-8)[2]
    k3 = _nc().proxy_rule(zhat, tol=1e-10)[2]
    assert k1 < k2 < k3


def test_proxy_rule_rejects_underdetermined():
    z = load_tables(os.path.join(ROOT, "tables", "data", "C5.npz")).zhat
    with pytest.raises(_nc().NcError):
        _nc().proxy_rule(z, deg=14, nring=3, cphi=10.0)   # fewer points than basis functions
