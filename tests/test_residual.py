"""NEXT-4: the L2 residual diagnostic eq:l2res.

CPU pins of the residual-grid tables (nc_tables/residual.py) and of the oracle (oracle.residual):
  * the grid's weights integrate the patch area |Gamma| = 2 pi (1 - cos eps) (the normaliser of eq:l2res);
  * the self-patch potential res_S of each basis solution equals the Zernike datum q_a at points the one-patch solve
    never saw -- the paper's one-patch residual eq:patcherrl2, here ~1e-14;
  * a single patch solved exactly (x = P 1: the N = 1 system is the identity) has residual ~0, and a
    perturbed x does not;
  * after the oracle's GMRES solve of C1 the residual is small and falls with the GMRES tolerance.
GPU parity (tests marked gpu): nc_residual against oracle.residual on the same inputs."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, make_centers, random_coeffs, synthetic_residual, synthetic_tables
from nc_inputs.tables import load_tables
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _phys(name):
    return load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))


def _q_at(tab):
    import nc_tables.zernike as Z
    r = np.arccos(np.clip(tab.res_rhat[:, 2], -1, 1)) / tab.eps
    th = np.arctan2(tab.res_rhat[:, 1], tab.res_rhat[:, 0])
    return Z.q_eval(tab.M, r, th)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_residual_tables_physical(name):
    tab = _phys(name)
    assert tab.res_S is not None
    area = 4 * np.pi * np.sin(tab.eps / 2) ** 2          # 2 pi (1 - cos eps) without the cancellation
    assert abs(tab.res_w.sum() - area) <= 1e-13 * area
    # the grid is not the solve's: no residual point coincides with a Zernike sampling node
    dmin = np.min(np.linalg.norm(tab.res_rhat[:, None, :] - tab.zhat[None, :, :], axis=2))
    assert dmin > 1e-3 * tab.eps
    # eq:patcherrl2 per basis function: || S sigma_a - q_a ||_L2 / |Gamma|.  Measured with the tables' one-patch
    # discretisation (13 panels x 20, R18): 1.5e-12 (eps 0.1), 1.5e-10 (0.02), 1.8e-9 (0.009),
    # 1.2e-8 (0.005), 5.4e-8 (0.003) -- the regime of the paper's reported residuals (~1e-8)
    err = np.sqrt(np.sum(tab.res_w[:, None] * (tab.res_S - _q_at(tab)) ** 2, axis=0)) / area
    assert np.max(err) <= 1e-7


def test_oracle_residual_single_patch_exact_solution():
    tab = _phys("C1")
    c = np.array([[0.0, 0.0, 1.0]])
    x = (tab.P @ np.ones(tab.Kstar))[None, :]           # the N = 1 solution: (I + 0) x = P 1
    res, pw = O.residual(tab.kind, c, tab, x, [0])
    assert res[0] <= 1e-12
    res2, _ = O.residual(tab.kind, c, tab, x * (1 + 1e-6), [0])
    assert res2[0] > 1e3 * max(res[0], 1e-15)


def test_oracle_residual_after_solve_C1():
    cfg = CONFIGS["C1"]
    tab = _phys("C1")
    c = cfg.centers()
    r_loose = O.solve(cfg.kind, c, tab, tol=1e-4)
    r_tight = O.solve(cfg.kind, c, tab, tol=1e-11)
    res_l, _ = O.residual(cfg.kind, c, tab, r_loose["x"], range(cfg.N))
    res_t, _ = O.residual(cfg.kind, c, tab, r_tight["x"], range(cfg.N))
    assert np.max(res_t) < np.max(res_l)
    assert np.max(res_t) <= 1e-6


def test_synthetic_residual_attaches_grid():
    tab = synthetic_residual(synthetic_tables(0, 0.05, seed=3), seed=4)
    assert tab.res_S.shape == (24 * 33, tab.K)
    assert abs(tab.res_w.sum() - 4 * np.pi * np.sin(0.025) ** 2) < 1e-15


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


@pytest.mark.gpu
@pytest.mark.parametrize("kind,N,eps", [(0, 300, 0.02), (1, 1000, 0.02)])
def test_residual_gpu_parity(kind, N, eps):
    torch = pytest.importorskip("torch")
    c = make_centers("uniform", N, eps, seed=60 + kind)
    tab = synthetic_residual(synthetic_tables(kind, eps, seed=61), seed=62)
    x = random_coeffs(N, tab.K, 63)
    pats = np.random.default_rng(64).choice(N, 7, replace=False)
    h = _nc().Handle(kind, c, eps, tab)
    xi = torch.from_numpy(h.to_internal(x)).cuda()
    res, pw = h.residual(xi, pats, tab)
    ref, pref = O.residual(kind, c, tab, x, pats)
    assert np.linalg.norm(pw - pref) / np.linalg.norm(pref) <= 1e-12
    assert np.max(np.abs(res - ref) / ref) <= 1e-12
    with pytest.raises(_nc().NcError, match="NC_EINVAL"):
        h.residual(xi, [N], tab)
    assert h.residual(xi, [], tab)[0].shape == (0,)
    h.close()


@pytest.mark.gpu
def test_residual_gpu_after_solve_C1():
    """The paper's accuracy metric on a physical solve: GPU residual of the GPU solution equals the oracle's
    residual of that same solution (1e-9: a small number formed by cancellation of O(1) terms), and is small."""
    torch = pytest.importorskip("torch")
    cfg = CONFIGS["C1"]
    tab = _phys("C1")
    c = cfg.centers()
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    xs, _, _ = h.gmres(rtol=1e-12, max_iter=200)
    res, pw = h.residual(xs, np.arange(cfg.N), tab)
    ref, pref = O.residual(cfg.kind, c, tab, h.to_caller(xs.cpu().numpy()), np.arange(cfg.N))
    assert np.max(np.abs(pw - pref)) <= 1e-12
    # | ||a|| - ||b|| | <= ||a - b|| (weighted norms): the residuals agree as far as their pointwise values do
    bound = np.sqrt(np.sum(tab.res_w[None, :] * (pw - pref) ** 2, axis=1)) / np.sum(tab.res_w)
    assert np.all(np.abs(res - ref) <= 1.01 * bound + 1e-30)
    assert np.max(res) <= 1e-6
    h.close()


@pytest.mark.gpu
def test_residual_gpu_hier_handle_matches_direct_handle():
    """nc_residual needs only the base-rung records, which both modes keep: a hierarchical handle gives the same
    residuals as a direct one on the same solution (C3-sized layout, physical tables)."""
    torch = pytest.importorskip("torch")
    cfg = CONFIGS["C2"]
    tab = _phys("C2")
    c = cfg.centers()
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    hh = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    x = random_coeffs(cfg.N, tab.K, 71)
    pats = np.arange(0, cfg.N, 97)
    rd, pd = hd.residual(torch.from_numpy(hd.to_internal(x)).cuda(), pats, tab)
    rh, ph = hh.residual(torch.from_numpy(hh.to_internal(x)).cuda(), pats, tab)
    assert np.max(np.abs(pd - ph)) <= 1e-12 * max(1.0, np.max(np.abs(pd)))
    hd.close()
    hh.close()
