"""Pins of the oracle's MFPT field (oracle.mfpt_field, eq:vtilde PAPER.md:533-536) against what the mathematics fixes.

v-bar = (v - 1) / (3 D) + (1 - |x|^2) / 6 with D = -I_sigma (the Lemma) must solve the MFPT problem
eq:intBVP: Delta v-bar = -1 in the ball; and its ball average is the average MFPT
mu = 1/(3 I_sigma) - 3/5 (eq:avgmfpt PAPER.md:141, eq:mufromsigma2 PAPER.md:617-618).  Both are checked on the
oracle's own solution of C1 (N = 10 patches, eps = 0.1, physical tables), with v from oracle.offsurface:

  * a second-order finite-difference Laplacian of mfpt_field at interior points equals -1 (v is harmonic: the
    off-surface Neumann function is, tests/test_field_oracle.py);
  * the average of mfpt_field over the ball B_R (R <= 0.9, spherical-shell quadrature: Gauss-Legendre in r and cos
    theta, trapezoid in phi) equals (v(0) - 1)/(3 D) + (1 - 3 R^2 / 5)/6 by the mean-value property of harmonic v,
    with v(0) = 2 I_sigma (G_I(0, x') = 2); at R = 1 this is exactly mu of the read-out.

A sign slip on D, on the |x|^2 term or a wrong coefficient of either fails one of them by orders of magnitude."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c1_solution():
    from nc_inputs.tables import load_tables
    cfg = CONFIGS["C1"]
    tab = load_tables(os.path.join(ROOT, "tables", "data", "C1.npz"))
    c = cfg.centers()
    r = O.solve(cfg.kind, c, tab, tol=1e-12)
    return c, tab, r


def _vbar(c, tab, r, pts):
    v, dmin = O.offsurface(0, c, tab, r["x"], pts)
    assert np.all(dmin > 0.05)
    return O.mfpt_field(v, pts, r["I_sigma"])


def test_mfpt_field_laplacian_is_minus_one(c1_solution):
    """Delta v-bar = -1 (eq:intBVP) at 12 interior points, central differences h = 2e-3."""
    c, tab, r = c1_solution
    rng = np.random.default_rng(31)
    d = rng.normal(size=(12, 3))
    p = (0.7 * rng.random(12) ** (1 / 3))[:, None] * d / np.linalg.norm(d, axis=1, keepdims=True)
    h = 2e-3
    pts = [p]
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        pts += [p + e, p - e]
    vb = _vbar(c, tab, r, np.concatenate(pts)).reshape(7, -1)
    lap = (vb[1:].sum(axis=0) - 6.0 * vb[0]) / h ** 2
    np.testing.assert_allclose(lap, -1.0, atol=2e-4)


@pytest.mark.parametrize("R", [0.5, 0.8])
def test_mfpt_field_ball_average(c1_solution, R):
    """(1/|B_R|) int_{B_R} v-bar dV = (2 I_sigma - 1)/(3 D) + (1 - 3 R^2/5)/6 with D = -I_sigma; R -> 1 gives the
    read-out mu = 1/(3 I_sigma) - 3/5 (eq:avgmfpt, eq:mufromsigma2)."""
    c, tab, r = c1_solution
    Is = r["I_sigma"]
    xr, wr = np.polynomial.legendre.leggauss(4)          # r in [0, R]: shell averages are polynomials of degree 2
    rr, wr = 0.5 * R * (xr + 1.0), 0.5 * R * wr * (0.5 * R * (xr + 1.0)) ** 2
    xt, wt = np.polynomial.legendre.leggauss(64)          # cos theta
    nph = 128
    ph = 2.0 * np.pi * np.arange(nph) / nph
    st = np.sqrt(1.0 - xt ** 2)
    dirs = np.stack([np.outer(st, np.cos(ph)), np.outer(st, np.sin(ph)), np.outer(xt, np.ones(nph))], -1).reshape(-1, 3)
    wd = np.repeat(wt, nph) * (2.0 * np.pi / nph)          # sums to 4 pi
    pts = (rr[:, None, None] * dirs[None]).reshape(-1, 3)
    vb = _vbar(c, tab, r, pts).reshape(len(rr), -1)
    avg = np.sum(wr[:, None] * wd[None, :] * vb) / (4.0 * np.pi * R ** 3 / 3.0)
    D = -Is
    expect = (2.0 * Is - 1.0) / (3.0 * D) + (1.0 - 3.0 * R ** 2 / 5.0) / 6.0
    assert abs(avg - expect) <= 1e-10 * abs(expect)
    # the same closed form at R = 1 is the read-out's average MFPT
    mu = O.readout(0, tab.I, r["x"])[1]
    assert abs(((2.0 * Is - 1.0) / (3.0 * D) + (1.0 - 3.0 / 5.0) / 6.0) - mu) <= 1e-13 * abs(mu)
