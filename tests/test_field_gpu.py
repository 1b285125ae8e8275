"""Off-surface field (NEXT-3, nc_field) of the CUDA path against the CPU oracle (oracle.offsurface): the same
compressed densities, the paper's off-surface Green's functions (eq:Gintoffsurface / eq:Gextoffsurface,
PAPER.md:350-353, 391-394).  Tiles of 256 points with ragged tails, a single point, no point; the argument checks;
and the physical identity v(0) = 2 I_sigma after a solve with physical tables.

Bar: <= 1e-12 relative l2 (the direct-mode tolerance of BASELINE.json), also for random coefficients whose
mixed-sign charges make the field a ~1e-3 residual of its terms (sum |G rho| ~ 900 |u| at C2): per point the error
is additionally held to 1e-15 sum |G rho|.  The oracle projects each skeleton node onto the sphere in long double
before evaluating the literal formulas (they hold for |x'| = 1; R27)."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, make_centers, random_coeffs, synthetic_tables
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-12


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def _points(kind, n, seed, rmax=0.85):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = rng.uniform(0.0, rmax, n) if kind == 0 else rng.uniform(1.15, 3.0, n)
    return d * r[:, None]


@pytest.mark.parametrize("kind,N,eps,n_pts", [(0, 200, 0.02, 1), (0, 200, 0.02, 1000), (1, 1000, 0.02, 257),
                                              (1, 300, 0.01, 513)])
def test_field_parity(kind, N, eps, n_pts):
    c = make_centers("uniform", N, eps, seed=40 + N)
    tab = synthetic_tables(kind, eps, seed=41)
    x = random_coeffs(N, tab.K, 42)
    pts = _points(kind, n_pts, 43)
    h = _nc().Handle(kind, c, eps, tab)
    xi = torch.from_numpy(h.to_internal(x)).cuda()
    v, dmin = h.field(xi, pts)
    ref, dref, absum = O.offsurface(kind, c, tab, x, pts, with_absum=True)
    assert rel(v, ref) <= TOL
    assert np.max(np.abs(v - ref) / absum) <= 1e-15
    assert np.max(np.abs(dmin - dref)) <= 1e-14
    h.close()


def test_field_hier_handle_and_empty():
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=44)
    x = random_coeffs(cfg.N, tab.K, 45)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    xi = torch.from_numpy(h.to_internal(x)).cuda()
    v, _ = h.field(xi, np.zeros((0, 3)))
    assert v.shape == (0,)
    pts = _points(cfg.kind, 300, 46)
    v, _ = h.field(xi, pts)
    ref, _, absum = O.offsurface(cfg.kind, c, tab, x, pts, with_absum=True)
    assert rel(v, ref) <= TOL
    assert np.max(np.abs(v - ref) / absum) <= 1e-15
    h.close()


def test_field_argument_checks():
    nc = _nc()
    c = make_centers("uniform", 50, 0.02, seed=47)
    tab = synthetic_tables(0, 0.02, seed=48)
    h = nc.Handle(0, c, 0.02, tab)
    xi = torch.from_numpy(h.to_internal(random_coeffs(50, tab.K, 49))).cuda()
    with pytest.raises(nc.NcError, match="NC_EINVAL"):       # exterior point for an interior problem
        h.field(xi, np.array([[0.0, 0.0, 1.5]]))
    with pytest.raises(nc.NcError, match="NC_EINVAL"):       # too close to a patch (the compressed form is invalid)
        h.field(xi, c[:1] * (1.0 - 0.02))
    h.close()


def test_field_physical_origin_identity_C1():
    """After the GPU solve (physical tables, interior C1): v(0) = 2 sum_j sum_m rho_jm, and since the skeleton
    reproduces each patch's monopole to the ID tolerance, v(0) / 2 = I_sigma of the read-out to ~1e-9."""
    from nc_inputs.tables import load_tables
    cfg = CONFIGS["C1"]
    tab = load_tables(os.path.join(ROOT, "tables", "data", "C1.npz"))
    h = _nc().Handle(cfg.kind, cfg.centers(), cfg.eps, tab)
    xs, _, _ = h.gmres(rtol=1e-12, max_iter=200)
    Is, mu = h.flux_or_mfpt(xs)
    v, _ = h.field(xs, np.zeros((1, 3)))
    assert abs(v[0] / 2 - Is) <= 1e-9 * abs(Is)
    pts = _points(cfg.kind, 200, 50, rmax=0.6)     # >= 3 eps (0.3) from the patches; same-sign charges
    vp, _ = h.field(xs, pts)
    xc = h.to_caller(xs.cpu().numpy())
    assert rel(vp, O.offsurface(cfg.kind, cfg.centers(), tab, xc, pts)[0]) <= TOL
    vbar0 = O.mfpt_field(v, np.zeros((1, 3)), Is)[0]
    assert 0.0 < vbar0 and np.isfinite(vbar0)
    h.close()


def test_field_exterior_far_field_C2():
    """Exterior problem (physical C2 tables, GPU solve): |x| u(x) -> I_sigma as |x| -> infinity (|x| G_E -> 1,
    DESIGN.md R3; the capacitance-like identity behind J = -4 pi I_sigma, R2)."""
    from nc_inputs.tables import load_tables
    cfg = CONFIGS["C2"]
    tab = load_tables(os.path.join(ROOT, "tables", "data", "C2.npz"))
    h = _nc().Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    xs, _, _ = h.gmres(rtol=1e-10, max_iter=200)
    Is, J = h.flux_or_mfpt(xs)
    d = np.array([[0.3, -0.5, 0.81]])
    d /= np.linalg.norm(d)
    for R, tol in ((1e3, 2e-3), (1e5, 2e-5)):
        u, _ = h.field(xs, R * d)
        assert abs(R * u[0] - Is) <= tol * abs(Is)
    h.close()
