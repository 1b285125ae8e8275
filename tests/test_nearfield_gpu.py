"""NEXT-3 near the surface on the GPU (nc_field_near) against the oracle (oracle.nearfield, pinned by
tests/test_nearfield_oracle.py): the potential and the MFPT v-bar on spheres of radius 1 -+ eps/5 (PAPER.md:2069-2097,
Fig. sphereplots), where the patches near a point are evaluated from their density sigma = B fhat (eq:recoversig).
Both sides take the same coefficients x; tolerance 1e-10 relative to max(1, |value|) (VERDICT r1 NEXT-3 bar)."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def _phys(name):
    from nc_inputs.tables import load_tables
    return load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))


def _points(c, eps, radius, n_near_per, patches, n_far, seed):
    """Points at |p| = radius: n_near_per within ~2 eps (arc) of each listed patch centre, plus n_far Fibonacci points."""
    rng = np.random.default_rng(seed)
    out = []
    for j in patches:
        cj = c[j]
        a = np.cross(cj, [1.0, 0.0, 0.0] if abs(cj[0]) < 0.9 else [0.0, 1.0, 0.0])
        a /= np.linalg.norm(a)
        b = np.cross(cj, a)
        for _ in range(n_near_per):
            t, th = 2.0 * eps * np.sqrt(rng.random()), 2 * np.pi * rng.random()
            d = np.cos(t) * cj + np.sin(t) * (np.cos(th) * a + np.sin(th) * b)
            out.append(radius * d / np.linalg.norm(d))
    k = np.arange(n_far) + 0.5
    z = 1.0 - 2.0 * k / n_far
    ph = np.pi * (1.0 + 5 ** 0.5) * k
    out += list(radius * np.stack([np.sqrt(1 - z * z) * np.cos(ph), np.sqrt(1 - z * z) * np.sin(ph), z], 1))
    return np.array(out)


def _check(name, x, pts, mfpt):
    cfg = CONFIGS[name]
    tab = _phys(name)
    c = cfg.centers()
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    xi = torch.from_numpy(h.to_internal(x)).cuda()
    v, mf, nnear = h.field_near(xi, pts, tab, mfpt=mfpt)
    ref = O.nearfield(cfg.kind, c, tab, x, pts)
    scale = np.maximum(1.0, np.abs(ref))
    assert nnear >= len(pts) // 2
    assert np.max(np.abs(v - ref) / scale) <= TOL
    if mfpt:
        Is = O.readout(cfg.kind, tab.I, x)[0]
        mref = O.mfpt_field(ref, pts, Is)
        assert np.max(np.abs(mf - mref) / np.maximum(1.0, np.abs(mref))) <= TOL
    h.close()
    return v, mf


def test_near_field_C1_interior_radius_one_minus_eps_over_5():
    cfg = CONFIGS["C1"]
    tab = _phys("C1")
    x = O.solve(cfg.kind, cfg.centers(), tab, tol=1e-12)["x"]
    pts = _points(cfg.centers(), cfg.eps, 1.0 - cfg.eps / 5, 4, [0, 3, 6, 9], 24, 1)
    v, mf = _check("C1", x, pts, mfpt=True)
    assert np.all(mf > -1e-6)                      # an MFPT is non-negative (0 on the absorbing patches)


def test_near_field_C2_exterior_radius_one_plus_eps_over_5():
    cfg = CONFIGS["C2"]
    tab = _phys("C2")
    x = random_coeffs(cfg.N, tab.K, 77)
    pts = _points(cfg.centers(), cfg.eps, 1.0 + cfg.eps / 5, 4, [0, 250, 500, 750, 999], 8, 2)
    _check("C2", x, pts, mfpt=False)


def test_near_field_C5_sampled():
    """The bench's workload (N = 1e5, eps = 0.003): a few points next to patches, against the oracle."""
    cfg = CONFIGS["C5"]
    tab = _phys("C5")
    x = random_coeffs(cfg.N, tab.K, 2005)
    pts = _points(cfg.centers(), cfg.eps, 1.0 - cfg.eps / 5, 2, [12, 54321, 99000], 0, 3)
    _check("C5", x, pts, mfpt=True)


def test_near_field_rejects_points_too_close():
    nc = _nc()
    cfg = CONFIGS["C1"]
    tab = _phys("C1")
    c = cfg.centers()
    h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
    xi = torch.zeros((cfg.N, tab.K), dtype=torch.float64, device="cuda")
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        h.field_near(xi, (1.0 - cfg.eps / 1000) * c[:1], tab)
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        h.field_near(xi, 1.01 * c[:1], tab)        # interior problem: the point must be inside
    v, _, nn = h.field_near(xi, np.zeros((1, 3)), tab)   # the centre: no near patch, zero density -> 0
    assert nn == 0 and abs(v[0]) == 0.0
    h.close()
