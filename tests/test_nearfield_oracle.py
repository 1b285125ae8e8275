"""Pins of the oracle's near-surface potential (NEXT-3: oracle.near_patch / oracle.nearfield; PAPER.md:2069-2097 plot
the MFPT on the sphere of radius 1 - eps/5, eq:vtilde PAPER.md:533-536).

near_patch integrates one patch's density sigma = B fhat (eq:recoversig) against the off-surface
Neumann function by adaptive quadrature.  What pins it, independently of the CUDA path and of its own formula:
  * the one-patch integral equation: the potential of the basis density sigma_a ON the patch is its Zernike datum q_a
    (S sigma_a = q_a; the solver's residual eq:patcherrl2 is 1.5e-12 at eps = 0.1), and the
    solver's own singular quadrature of S sigma_a at the residual grid (res_S) is an independent rule for the same
    integral: the off-surface potential at height h over a patch point extrapolates (h -> 0, cubic Richardson) to both;
  * the compressed skeleton (eq:outgoingcompressed, a different representation of the same field) agrees with it
    wherever both hold (3 to 6 eps from the patch);
  * the solved system's boundary condition: v -> 1 on an absorbing patch (eq:intBVP2 PAPER.md:525-531), and the
    MFPT v-bar solves Delta v-bar = -1 right next to the patches (eq:intBVP PAPER.md:131-139)."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c1():
    from nc_inputs.tables import load_tables
    tab = load_tables(os.path.join(ROOT, "tables", "data", "C1.npz"))
    assert tab.near_sigma is not None
    c = CONFIGS["C1"].centers()
    r = O.solve(0, c, tab, tol=1e-12)
    return tab, c, r


def _zernike(n, m, cs, r, th):
    """Orthonormal Zernike function of the table basis (R6: flat measure on the unit disk, r = t / eps)."""
    from math import factorial
    k = (n - m) // 2
    R = sum((-1) ** s * factorial(n - s) / (factorial(s) * factorial((n + m) // 2 - s) * factorial((n - m) // 2 - s))
            * r ** (n - 2 * s) for s in range(k + 1))
    norm = np.sqrt((2 * n + 2) / (2 * np.pi if m == 0 else np.pi))
    return norm * R * (np.cos(m * th) if cs > 0 else np.sin(m * th))


@pytest.mark.parametrize("a", [0, 4, 17, 60, 131])
def test_basis_density_potential_on_the_patch(c1, a):
    """The potential of the basis density sigma_a ON the patch, reached from inside: the near quadrature at heights
    eps/200 .. eps/1600 over a patch point, extrapolated to the surface (cubic Richardson: the potential is smooth up
    to the surface from one side, away from the patch edge), equals
      * res_S[k, a]: S sigma_a at the residual-grid point k computed by the one-patch solver's own singular
        quadrature (nc_tables/residual.py, an independent rule for the same on-surface integral), and
      * for the low orders, the Zernike datum q_a itself (S sigma_a = q_a up to the solver residual eq:patcherrl2)."""
    tab, _, _ = c1
    from nc_tables import zernike
    n, m, cs = zernike.basis_indices(tab.M)[a]
    eps = tab.eps
    x = np.zeros(tab.K)
    x[a] = 1.0
    t_all = np.arccos(np.clip(tab.res_rhat[:, 2], -1, 1))
    for k in (np.argmin(np.abs(t_all - 0.3 * eps) + 0.01 * np.arange(len(t_all)) / len(t_all)),
              np.argmin(np.abs(t_all - 0.5 * eps) + 0.01 * np.arange(len(t_all)) / len(t_all))):
        on = tab.res_rhat[k]
        hs = eps / np.array([200.0, 400.0, 800.0, 1600.0])
        v = np.array([O.near_patch(0, tab, x, (1.0 - h) * on) for h in hs])
        v0 = np.polyval(np.polyfit(hs, v, 3), 0.0)
        # (the extrapolation's own error, ~h^4 times the 4th normal derivative, is ~1e-9 for the high orders)
        assert abs(v0 - tab.res_S[k, a]) <= 2e-9 * max(1.0, abs(v0)), (v0, tab.res_S[k, a])
        if n <= 4:
            q = _zernike(n, m, cs, t_all[k] / eps, np.arctan2(on[1], on[0]))
            assert abs(v0 - q) <= 1e-10 * max(1.0, abs(q)), (v0, q)


def test_near_quadrature_matches_compressed_skeleton(c1):
    tab, c, r = c1
    rng = np.random.default_rng(3)
    for d_rel in (4.0, 5.0, 6.0):
        for h_rel in (0.2, 1.0):
            az = 2 * np.pi * rng.random()
            ang = d_rel * tab.eps
            p = (1.0 - h_rel * tab.eps) * np.array([np.sin(ang) * np.cos(az), np.sin(ang) * np.sin(az), np.cos(ang)])
            vq = O.near_patch(0, tab, r["x"][0], p)
            vc, dm = O.offsurface(0, c[:1] * 0 + np.array([[0.0, 0.0, 1.0]]), tab, r["x"][:1], p[None])
            assert dm[0] > 2.5 * tab.eps
            assert abs(vq - vc[0]) <= 1e-11 * abs(vc[0]), (d_rel, h_rel, vq, vc[0])


def test_solution_meets_boundary_condition_on_patches(c1):
    """v -> 1 on the absorbing patches: cubic extrapolation of v at heights eps/100 .. eps/800 over patch points."""
    tab, c, r = c1
    eps = tab.eps
    R = O.frames(c)
    for j, (t_rel, th) in ((0, (0.0, 0.0)), (3, (0.5, 1.0)), (7, (0.85, 4.0))):
        t = t_rel * eps
        loc = np.array([np.sin(t) * np.cos(th), np.sin(t) * np.sin(th), np.cos(t)])
        on = R[j] @ loc
        hs = eps / np.array([100.0, 200.0, 400.0, 800.0])
        v = O.nearfield(0, c, tab, r["x"], (1.0 - hs)[:, None] * on[None, :])
        v0 = np.polyval(np.polyfit(hs, v, 3), 0.0)
        assert abs(v0 - 1.0) <= 1e-8, (j, v0)


def test_mfpt_laplacian_next_to_a_patch(c1):
    """Delta v-bar = -1 at height eps/5 over a patch (fourth-order central differences, step eps/40)."""
    tab, c, r = c1
    p = (1.0 - tab.eps / 5) * c[2]
    hd = tab.eps / 40
    pts = [p]
    for a in range(3):
        for k in (1, -1, 2, -2):
            e = np.zeros(3)
            e[a] = k * hd
            pts.append(p + e)
    pts = np.array(pts)
    vb = O.mfpt_field(O.nearfield(0, c, tab, r["x"], pts), pts, r["I_sigma"])
    f = vb[1:].reshape(3, 4)                                # per axis: +h, -h, +2h, -2h
    lap = np.sum(16.0 * (f[:, 0] + f[:, 1]) - (f[:, 2] + f[:, 3]) - 30.0 * vb[0]) / (12.0 * hd ** 2)
    assert abs(lap + 1.0) <= 1e-4, lap
