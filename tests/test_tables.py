"""Step-1 table builder (nc_tables) pinned against what the paper and mathematics fix, and the oracle's physics
limits with physical tables (single-patch limit, refinement convergence, bounds)."""
import os

import numpy as np
import pytest

from nc_tables import zernike
from nc_tables.kernel import INTERIOR, EXTERIOR, phi_rule
from nc_tables.onepatch import solve_onepatch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_zernike_count_and_exact_transform():
    # K = (M+1)(M+2)/2 = 136 for M = 15 (PAPER.md:845-847 with :55 "13.6 million" / 100 000)
    M = 15
    assert len(zernike.basis_indices(M)) == 136
    r, th, P = zernike.transform(M)
    Q = zernike.q_eval(M, r, th)
    # P is a left inverse of the synthesis at the nodes (Definition "projectors")
    np.testing.assert_allclose(P @ Q, np.eye(136), atol=2e-13)


def test_zernike_orthogonality_relation():
    # eq:zorthog: int Z Z r dr dtheta = (1 + delta_m0) pi / (2n + 2), checked by an
    # independent fine tensor quadrature (not the sampling grid)
    x, w = np.polynomial.legendre.leggauss(40)
    r = 0.5 * (x + 1)
    wr = 0.5 * w * r
    th = 2 * np.pi * np.arange(64) / 64
    R, TH = np.meshgrid(r, th, indexing="ij")
    W = (wr[:, None] * np.full(64, 2 * np.pi / 64)[None, :]).ravel()
    for (n, m) in [(0, 0), (2, 0), (3, 1), (7, 5), (15, 15), (14, 0)]:
        z = zernike.radial(n, m, R.ravel()) * np.cos(m * TH.ravel())
        assert abs(np.sum(W * z * z) - (1 + (m == 0)) * np.pi / (2 * n + 2)) < 1e-13
    # R_1^1 = r, R_2^0 = 2r^2 - 1 (textbook)
    np.testing.assert_allclose(zernike.radial(1, 1, r), r, atol=1e-15)
    np.testing.assert_allclose(zernike.radial(2, 0, r), 2 * r * r - 1, atol=1e-14)


@pytest.mark.parametrize("t,tp", [(0.1, 0.2), (0.3, 0.7), (0.01, 0.0100001), (1e-3, 0.02), (0.05, 0.05 + 1e-12)])
def test_modal_quadrature_matches_paper_closed_form(t, tp):
    # the paper's closed form for (1/pi) int_0^pi log(2/|x-x'|) cos(n phi) dphi
    phi, w = phi_rule()
    A = 4 * np.sin((t - tp) / 2) ** 2
    B = 4 * np.sin(t) * np.sin(tp)
    d = np.sqrt(A + B * np.sin(phi / 2) ** 2)
    t1, t2 = min(t, tp), max(t, tp)
    for n in range(0, 41):
        g = np.sum(w * np.log(2 / d) * np.cos(n * phi)) / np.pi
        ex = -np.log(np.cos(t1 / 2) * np.sin(t2 / 2)) if n == 0 else (np.tan(t1 / 2) / np.tan(t2 / 2)) ** n / (2 * n)
        assert abs(g - ex) < 1e-14 * max(1.0, abs(ex))


def _I_sigma_single(kind, eps, npan=13, k=20):
    op = solve_onepatch(kind, eps, 15, npan, k)
    g = op.grid
    # data f = 1 = sqrt(pi) q_0; I_sigma = int sigma dS = 2 pi sum_j w_j sigma(t_j)
    return np.sqrt(np.pi) * 2 * np.pi * np.sum(g.w * op.sigma_radial[0])


@pytest.mark.parametrize("kind", [INTERIOR, EXTERIOR])
def test_single_patch_flat_disk_asymptotics(kind):
    """Leading 2/|x-x'| kernel gives the flat-disk charge eps/pi (textbook disk capacitance);
    first-order perturbation by the +-log(2/d) term gives
      I = (eps/pi) [1 -+ (eps/pi)(log(2/eps) + 3/2 - 2 log 2)] + O((eps log eps)^2)."""
    eps = 0.003
    Is = _I_sigma_single(kind, eps)
    sgn = -1.0 if kind == INTERIOR else 1.0
    asym = (eps / np.pi) * (1 + sgn * (eps / np.pi) * (np.log(2 / eps) + 1.5 - 2 * np.log(2)))
    assert abs(Is / asym - 1) < 1e-4
    # the perturbative correction itself is resolved: dropping it is off by far more
    assert abs(Is / (eps / np.pi) - 1) > 5e-3


def test_one_patch_refinement_convergence():
    # convergence under patch-quadrature refinement (Fig. 5 right panel)
    a = _I_sigma_single(INTERIOR, 0.1, 10, 16)
    b = _I_sigma_single(INTERIOR, 0.1, 13, 20)
    c = _I_sigma_single(INTERIOR, 0.1, 16, 24)
    assert abs(b - c) < 1e-12 * abs(c)
    assert abs(a - c) < 1e-9 * abs(c)


def _load(name):
    from nc_inputs.tables import load_tables
    path = os.path.join(ROOT, "tables", "data", f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (python -m nc_tables.build --configs)")
    return load_tables(path)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_config_tables(name):
    from nc_inputs import CONFIGS
    tab = _load(name)
    cfg = CONFIGS[name]
    assert tab.kind == cfg.kind and tab.eps == cfg.eps and tab.K == 136 and tab.Kstar == 248
    meta = eval(tab.meta["repr"], {"__builtins__": {}}) if tab.meta.get("repr", "").startswith("{") else {}
    if meta:
        assert meta["outgoing_rel_err"] < 1e-9        # eq:outgoingcompressed at ID tol 1e-11
    # skeleton nodes are fine-grid points on the patch
    assert np.arccos(np.clip(tab.shat[:, 2], -1, 1)).max() < tab.eps


def test_oracle_single_patch_solve_physical_tables():
    """N = 1 with physical tables: GMRES returns P 1 and mu = 1/(3 I_sigma) - 3/5 (eq:mufromsigma2) with
    I_sigma matching the flat-disk asymptotics; mu > 1/15 (full-coverage bound)."""
    from oracle import oracle as O
    tab = _load("C5")
    r = O.solve(0, np.array([[0.0, 0.0, 1.0]]), tab)
    eps = tab.eps
    asym = (eps / np.pi) * (1 - (eps / np.pi) * (np.log(2 / eps) + 1.5 - 2 * np.log(2)))
    assert r["iters"] <= 1
    assert abs(r["I_sigma"] / asym - 1) < 1e-4
    assert r["value"] == pytest.approx(1 / (3 * r["I_sigma"]) - 0.6, rel=1e-15)
    assert r["value"] > 1 / 15


def test_oracle_physics_bounds_C1():
    """C1 with physical tables: 1/15 < mu; adding patches lowers mu (comparison principle); the exterior flux
    |J| < 4 pi (full-coverage capacitance)."""
    from nc_inputs import CONFIGS
    from oracle import oracle as O
    tab = _load("C1")
    c = CONFIGS["C1"].centers()
    mus = [O.solve(0, c[:n], tab)["value"] for n in (1, 3, 10)]
    assert mus[0] > mus[1] > mus[2] > 1 / 15
    tabE = _load("C2")
    cE = CONFIGS["C2"].centers()[:20]
    rE = O.solve(1, cE, tabE)
    assert -4 * np.pi < rE["value"] < 0


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_per_level_ladder_tables(name):
    """Per-level recompression: rung k compresses the outgoing field on {arc > r_k} with fewer
    skeleton points than the base (valid beyond 2 eps); every rung's compressed field meets its ID tolerance on its
    region to the factor the ID's field error carries (<= 10 x the tolerance, SURVEY.md §8(c) "Skeleton/T")."""
    tab = _load(name)
    meta = eval(tab.meta["repr"], {"__builtins__": {}})
    assert tab.ladder_r is not None
    assert np.all(tab.ladder_p < tab.p) and tab.ladder_p[-1] < tab.ladder_p[0] / 2
    assert max(meta["ladder_err"]) < 10.0 * tab.ladder_tol
    ratio = meta.get("ladder_ratio", 2.0)
    np.testing.assert_allclose(tab.ladder_r / tab.eps, 2.0 * ratio ** np.arange(1, len(tab.ladder_r) + 1), rtol=1e-6)
