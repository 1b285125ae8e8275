"""Full-size parity of the hierarchical matvec and the solve (BASELINE.json north_star
tolerances), in the configuration bench.py times (physical tables with the per-level ladder, precision 1e-9).

Expected values come only from the oracle:
  * tests/golden/oracle_rows_C{3,4,5}.npz -- oracle rows for target patches chosen from the geometry alone (cube
    corners and edges, face and level-1 box boundaries, the densest patches, uniform picks), written by
    tools/make_goldens.py, which calls only oracle/;
  * rows the product's own tree makes interesting (patches with non-empty near lists, patches next to the
    work-weighted rank cuts of world 2, 4 and 8) are computed by the oracle here, live;
  * tests/golden/oracle_solve_C2.json -- the oracle's full GMRES solve of C2 (J, I_sigma), tools/make_goldens.py.
Tolerances: hierarchical matvec <= 1e-8 relative l2 (contract) and <= the requested precision 1e-9 over each group of
rows; direct matvec <= 1e-12; solved J / mu <= 1e-7 relative."""
import json
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
HIER_TOL = 1e-8
PRECISION = 1e-9


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def _phys(name):
    from nc_inputs.tables import load_tables
    return load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def gpu_matvec(h, x_caller):
    y = h.matvec(torch.from_numpy(h.to_internal(x_caller)).cuda())
    torch.cuda.synchronize()
    return h.to_caller(y.cpu().numpy())


_cache = {}


def _hier(name):
    """(config, tables, centers, x, handle, y) for the bench's workload of a config, built once per session."""
    if name not in _cache:
        cfg = CONFIGS[name]
        tab = _phys(name)
        c = cfg.centers()
        x = random_coeffs(cfg.N, tab.K, 2000 + int(name[1:]))
        h = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
        _cache[name] = (cfg, tab, c, x, h, gpu_matvec(h, x))
    return _cache[name]


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_hier_rows_vs_oracle_golden(name):
    """Oracle rows chosen from the geometry (tools/make_goldens.py): every tag group (corners, edges, boundaries,
    densest, uniform) within the precision, so a fault confined to one region of the tree cannot hide."""
    cfg, tab, c, x, h, y = _hier(name)
    g = np.load(os.path.join(GOLD, f"oracle_rows_{name}.npz"))
    assert int(g["N"]) == cfg.N and int(g["x_seed"]) == 2000 + int(name[1:])
    rows, tags, ref = g["rows"], g["tags"], g["y"]
    assert rel(y[rows], ref) <= PRECISION
    for t in np.unique(tags):
        sel = tags == t
        assert rel(y[rows[sel]], ref[sel]) <= PRECISION, t
    # and the operator part alone (y - x) within the contract relative to its own size
    assert rel(y[rows] - x[rows], ref - x[rows]) <= HIER_TOL


def _special_rows(name, n_near, n_cut):
    """Rows picked from the product's tree: the largest near lists, and the patches on both sides of the
    work-weighted rank cuts of world 2, 4, 8 (rank-emulation handles: the same partition nc_setup uses)."""
    cfg, tab, c, x, h, y = _hier(name)
    nc = _nc()
    counts = h.near_counts()
    order = np.argsort(-counts, kind="stable")
    near = [int(h.perm[h.row_begin + i]) for i in order[:n_near] if counts[i] > 0]
    cut = []
    for world in (2, 4, 8):
        hr = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision, world=world, rank=1)
        for r in (hr.row_begin - 1, hr.row_begin):
            cut.append(int(hr.perm[r]))
        hr.close()
    return sorted(set(near)), sorted(set(cut[: 2 * n_cut]))


@pytest.mark.parametrize("name,n_near,n_cut", [("C3", 4, 3), ("C4", 4, 3), ("C5", 2, 1)])
def test_hier_rows_near_lists_and_rank_cuts_vs_oracle(name, n_near, n_cut):
    cfg, tab, c, x, h, y = _hier(name)
    near, cut = _special_rows(name, n_near, n_cut)
    assert len(near) >= 1, "no patch with a near list at this configuration"
    for rows in (near, cut):
        rows = np.asarray(rows, dtype=np.int64)
        assert rel(y[rows], O.matvec(cfg.kind, c, tab, x, rows=rows)) <= PRECISION


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_hier_full_vector_vs_gpu_direct(name):
    """The whole hierarchical matvec against the GPU direct sum (itself <= 1e-12 from the oracle,
    tests/test_direct_gpu.py), random x and the physical right-hand side: within the requested precision with the
    per-level ladder on and hence within the 1e-8 contract."""
    cfg, tab, c, x, h, y = _hier(name)
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    assert rel(y, gpu_matvec(hd, x)) <= PRECISION
    b = np.tile(tab.P @ np.ones(tab.Kstar), (cfg.N, 1))
    assert rel(gpu_matvec(h, b), gpu_matvec(hd, b)) <= PRECISION
    assert h.stats()["hier_grid_pairs"] > 0
    hd.close()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_hier_solve_matches_direct_solve(name):
    """GMRES to 1e-10 on the physical right-hand side: hierarchical mu / J equals the direct-mode solve's to 1e-7
    (north_star), iteration counts within 2."""
    cfg, tab, c, x, h, y = _hier(name)
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    xd, itd, _ = hd.gmres(rtol=cfg.gmres_tol, max_iter=200)
    xh, ith, _ = h.gmres(rtol=cfg.gmres_tol, max_iter=200)
    Id, vd = hd.flux_or_mfpt(xd)
    Ih, vh = h.flux_or_mfpt(xh)
    assert abs(vh - vd) <= 1e-7 * abs(vd)
    assert abs(Ih - Id) <= 1e-7 * abs(Id)
    assert abs(ith - itd) <= 2
    hd.close()


@pytest.mark.parametrize("mode", ["direct", "hier"])
def test_C2_solve_vs_oracle_golden(mode):
    """The oracle's full C2 solve (tools/make_goldens.py solve C2: MGS GMRES on the brute-force O(N^2) matvec, 1e-10):
    the GPU's J = -4 pi I_sigma (R2) in both modes within 1e-7 (north_star)."""
    path = os.path.join(GOLD, "oracle_solve_C2.json")
    if not os.path.exists(path):
        pytest.skip("golden oracle solve of C2 not generated yet (tools/make_goldens.py solve C2)")
    g = json.load(open(path))
    cfg = CONFIGS["C2"]
    tab = _phys("C2")
    nc = _nc()
    h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=nc.NC_DIRECT if mode == "direct" else nc.NC_HIER,
                  precision=cfg.precision)
    xs, it, _ = h.gmres(rtol=g["gmres_tol"], max_iter=200)
    Is, J = h.flux_or_mfpt(xs)
    assert abs(J - g["J"]) <= 1e-7 * abs(g["J"])
    assert abs(Is - g["I_sigma"]) <= 1e-7 * abs(g["I_sigma"])
    assert abs(it - g["iters"]) <= 2
    h.close()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_ladder_gate_boundary(name):
    """nc_setup admits the per-level ladder when the requested precision is >= the rungs' ID tolerance:
    at exactly that precision the hierarchical matvec (ladder on) must still meet it against the GPU direct sum."""
    cfg, tab, c, x, h, y = _hier(name)
    assert tab.ladder_tol > 0
    nc = _nc()
    hb = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=tab.ladder_tol)
    hd = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
    assert rel(gpu_matvec(hb, x), gpu_matvec(hd, x)) <= tab.ladder_tol
    hn = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=0.5 * tab.ladder_tol)   # ladder off
    assert hn.stats()["hier_grid_pairs"] > hb.stats()["hier_grid_pairs"]
    for hh in (hb, hd, hn):
        hh.close()


def test_C5_solution_residual_on_oracle_rows():
    """the oracle's residual of the GPU-hierarchical C5 solution on sampled rows,
    (I + A_off) x - P 1 by the brute-force direct sum, relative to b: the GMRES tolerance plus the hierarchical
    matvec error (<= the requested precision 1e-9)."""
    cfg, tab, c, x, h, y = _hier("C5")
    xs, it, _ = h.gmres(rtol=cfg.gmres_tol, max_iter=200)
    xg = h.to_caller(xs.cpu().numpy())
    rows = np.array([3, 4242, 50505, 99999], dtype=np.int64)
    b = np.tile(tab.P @ np.ones(tab.Kstar), (len(rows), 1))
    r = O.matvec(cfg.kind, c, tab, xg, rows=rows) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 2e-9
