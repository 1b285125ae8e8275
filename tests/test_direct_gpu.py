"""Direct-mode parity of the CUDA path (libnc via its C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): direct matvec <= 1e-12 relative l2; solved J / mu <= 1e-7 relative."""
import numpy as np
import pytest

from nc_inputs import CONFIGS, make_centers, random_coeffs, synthetic_tables
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-12


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def gpu_matvec(h, x_caller):
    xi = torch.from_numpy(h.to_internal(x_caller)).cuda()
    y = h.matvec(xi)
    torch.cuda.synchronize()
    return h.to_caller(y.cpu().numpy())


@pytest.mark.parametrize("kind", [0, 1])
def test_matvec_parity_C1(kind):
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(kind, cfg.eps, seed=31)
    x = random_coeffs(cfg.N, tab.K, 2001)
    h = _nc().Handle(kind, c, cfg.eps, tab)
    y = gpu_matvec(h, x)
    assert rel(y, O.matvec(kind, c, tab, x)) <= MATVEC_TOL


@pytest.mark.parametrize("M,nr,nth,p,N", [(15, 16, 31, 97, 37), (3, 3, 5, 5, 9), (2, 2, 3, 1, 3), (6, 7, 13, 300, 23)])
def test_matvec_parity_ragged(M, nr, nth, p, N):
    # tiles straddling patches (Kstar not a multiple of 256), ragged GEMM tiles, p = 1 and p > 256
    eps = 0.05
    c = make_centers("uniform", N, eps, seed=77)
    for kind in (0, 1):
        tab = synthetic_tables(kind, eps, seed=5, M=M, p=p, n_r=nr, n_theta=nth)
        x = random_coeffs(N, tab.K, 3)
        h = _nc().Handle(kind, c, eps, tab)
        assert rel(gpu_matvec(h, x), O.matvec(kind, c, tab, x)) <= MATVEC_TOL


def test_single_patch_is_identity():
    # in the one-patch case the summation term vanishes
    tab = synthetic_tables(0, 0.1, seed=1)
    x = random_coeffs(1, tab.K, 4)
    h = _nc().Handle(0, np.array([[0.0, 0.6, 0.8]]), 0.1, tab)
    np.testing.assert_array_equal(gpu_matvec(h, x), x)


def test_matvec_parity_C2_full_size_sampled_rows():
    # C2 at its full size (N = 1000, Kstar = 512, p = 120): sampled target patches against the oracle rows
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=32)
    x = random_coeffs(cfg.N, tab.K, 2002)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    y = gpu_matvec(h, x)
    rows = np.random.default_rng(0).choice(cfg.N, 12, replace=False)
    assert rel(y[rows], O.matvec(cfg.kind, c, tab, x, rows=rows)) <= MATVEC_TOL
    # deterministic: a second application is bitwise identical
    np.testing.assert_array_equal(gpu_matvec(h, x), y)


def test_host_entry_point_matches_device():
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=33)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    x = random_coeffs(cfg.N, tab.K, 5)
    xi = h.to_internal(x)
    np.testing.assert_array_equal(h.matvec_host(xi), h.matvec(torch.from_numpy(xi).cuda()).cpu().numpy())


@pytest.mark.parametrize("kind", [0, 1])
def test_gmres_and_readout_C1(kind):
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(kind, cfg.eps, seed=34, coupling=30.0)
    ref = O.solve(kind, c, tab, tol=1e-12)
    h = _nc().Handle(kind, c, cfg.eps, tab)
    x, it, hist = h.gmres(rtol=1e-12, max_iter=100)
    xg = h.to_caller(x.cpu().numpy())
    assert abs(it - ref["iters"]) <= 1
    assert rel(xg, ref["x"]) < 1e-10
    Is, v = h.flux_or_mfpt(x) if (kind == 1 or ref["I_sigma"] > 0) else (None, None)
    if Is is not None:
        assert abs(Is - ref["I_sigma"]) <= 1e-7 * abs(ref["I_sigma"])
        assert abs(v - ref["value"]) <= 1e-7 * abs(ref["value"])
    assert np.all(np.diff(hist) <= 1e-15)


def test_gmres_explicit_rhs_matches_oracle_C2():
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=35, coupling=0.05)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    b = random_coeffs(cfg.N, tab.K, 9)
    x, it, _ = h.gmres(b=torch.from_numpy(h.to_internal(b)).cuda(), rtol=1e-10, max_iter=60)
    xg = h.to_caller(x.cpu().numpy())
    # residual of the GPU solution measured through the oracle on sampled rows
    rows = np.arange(0, cfg.N, 125)
    r = O.matvec(cfg.kind, c, tab, xg, rows=rows) - b[rows]
    assert np.linalg.norm(r) / np.linalg.norm(b[rows]) < 1e-9


def test_errors():
    nc = _nc()
    tab = synthetic_tables(0, 0.1, seed=1)
    with pytest.raises(nc.NcError, match="NC_ESEP"):
        nc.Handle(0, np.array([[0, 0, 1.0], [np.sin(0.2), 0, np.cos(0.2)]]), 0.1, tab)
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        nc.Handle(0, np.array([[0, 0, 2.0]]), 0.1, tab)
    bad = synthetic_tables(0, 0.1, seed=1, M=3)
    bad.M = 4
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        nc.Handle(0, np.array([[0, 0, 1.0]]), 0.1, bad)


def _phys(name):
    import os
    from nc_inputs.tables import load_tables
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tables", "data", f"{name}.npz")
    return load_tables(path)


def test_solve_physical_tables_C1_mu_matches_oracle():
    # BASELINE north_star: solved mu within 1e-7 relative of the oracle on the same seeded inputs
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = _phys("C1")
    ref = O.solve(cfg.kind, c, tab, tol=1e-10)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    x, it, hist = h.gmres(rtol=1e-10, max_iter=100)
    Is, mu = h.flux_or_mfpt(x)
    assert abs(it - ref["iters"]) <= 1
    assert abs(mu - ref["value"]) <= 1e-7 * abs(ref["value"])
    assert abs(Is - ref["I_sigma"]) <= 1e-7 * abs(ref["I_sigma"])
    assert rel(h.to_caller(x.cpu().numpy()), ref["x"]) < 1e-8


def test_solve_physical_tables_C2_residual_via_oracle_rows():
    # C2 (N = 1000, exterior): the GPU solution's residual measured by the oracle on sampled rows
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = _phys("C2")
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab)
    x, it, hist = h.gmres(rtol=1e-10, max_iter=200)
    Is, J = h.flux_or_mfpt(x)
    assert hist[-1] <= 1e-10 and -4 * np.pi < J < 0
    xg = h.to_caller(x.cpu().numpy())
    rows = np.random.default_rng(1).choice(cfg.N, 6, replace=False)
    b = O.rhs(tab, cfg.N)
    r = O.matvec(cfg.kind, c, tab, xg, rows=rows) - b[rows]
    assert np.linalg.norm(r) / np.linalg.norm(b[rows]) < 1e-9
    # matvec parity with physical tables at full size (sampled rows)
    xr = random_coeffs(cfg.N, tab.K, 77)
    y = gpu_matvec(h, xr)
    assert rel(y[rows], O.matvec(cfg.kind, c, tab, xr, rows=rows)) <= MATVEC_TOL
