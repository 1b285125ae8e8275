"""Hierarchical mode (NC_HIER): tree audit and parity against the direct sum / the oracle.

Tolerance (BASELINE.json north_star): hierarchical matvec <= 1e-8 relative l2 at the requested precision 1e-9;
solved J / mu <= 1e-7 relative."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, make_centers, random_coeffs, synthetic_tables
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HIER_TOL = 1e-8
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def _phys(name):
    from nc_inputs.tables import load_tables
    return load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def gpu_matvec(h, x_caller):
    xi = torch.from_numpy(h.to_internal(x_caller)).cuda()
    y = h.matvec(xi)
    torch.cuda.synchronize()
    return h.to_caller(y.cpu().numpy())


def _group_ranges(bop):
    L1, N = bop.shape
    G = int(bop.max()) + 1
    first = np.full(G, N, dtype=np.int64)
    last = np.zeros(G, dtype=np.int64)
    for lvl in range(L1):
        g = bop[lvl]
        np.minimum.at(first, g, np.arange(N))
        np.maximum.at(last, g, np.arange(N) + 1)
    return first, last


@pytest.mark.parametrize("layout,N,eps", [("uniform", 700, 0.02), ("vmf", 1500, 0.005), ("uniform", 1, 0.1),
                                          ("uniform", 7, 0.1)])
def test_pair_coverage_exactly_once(layout, N, eps):
    """PAPER.md:1366-1372 (note to step 3): every other patch is either a leaf neighbour or in exactly one
    interaction list of the groups containing the target patch.  Exhaustive over all ordered pairs."""
    c = make_centers(layout, N, eps, seed=5)
    tab = synthetic_tables(0, eps, seed=1, M=2, p=3, n_r=2, n_theta=3)
    h = _nc().Handle(0, c, eps, tab, mode=_nc().NC_HIER)
    il, nb, bop = h.tree_lists()
    first, last = _group_ranges(bop)
    cnt = np.zeros((N, N), dtype=np.int32)
    for _, g, b in np.concatenate([il, nb]) if len(il) + len(nb) else []:
        cnt[first[g]:last[g], first[b]:last[b]] += 1
    off = ~np.eye(N, dtype=bool)
    assert np.all(cnt[off] == 1)
    assert np.all(np.diag(cnt) == 0)
    # interaction lists hold at most 27 boxes; leaf neighbours at most 8
    if len(il):
        _, counts = np.unique(il[:, 1], return_counts=True)
        assert counts.max() <= 27
    if len(nb):
        _, counts = np.unique(nb[:, 1], return_counts=True)
        assert counts.max() <= 8


@pytest.mark.parametrize("kind", [0, 1])
def test_hier_matches_direct_C2(kind):
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = _phys("C2")
    x = random_coeffs(cfg.N, tab.K, 2002)
    hd = _nc().Handle(kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    hh = _nc().Handle(kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=1e-9)
    yd = gpu_matvec(hd, x)
    yh = gpu_matvec(hh, x)
    assert rel(yh, yd) <= HIER_TOL
    # the operator part alone (y - x) also within tolerance of its own norm x 10
    assert rel(yh - x, yd - x) <= 10 * HIER_TOL
    rows = np.random.default_rng(3).choice(cfg.N, 4, replace=False)
    assert rel(yh[rows], O.matvec(kind, c, tab, x, rows=rows)) <= HIER_TOL


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_hier_sampled_rows_vs_oracle(name):
    cfg = CONFIGS[name]
    c = cfg.centers()
    tab = _phys(name)
    x = random_coeffs(cfg.N, tab.K, 2003)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    y = gpu_matvec(h, x)
    rows = np.random.default_rng(4).choice(cfg.N, 3, replace=False)
    assert rel(y[rows], O.matvec(cfg.kind, c, tab, x, rows=rows)) <= HIER_TOL


def test_hier_solve_matches_direct_solve_C2():
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = _phys("C2")
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    hh = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=1e-9)
    xd, itd, _ = hd.gmres(rtol=1e-10, max_iter=200)
    xh, ith, _ = hh.gmres(rtol=1e-10, max_iter=200)
    Jd = hd.flux_or_mfpt(xd)[1]
    Jh = hh.flux_or_mfpt(xh)[1]
    assert abs(Jh - Jd) <= 1e-7 * abs(Jd)
    assert abs(ith - itd) <= 2


def test_per_level_outgoing_ladder_matches_direct_C2():
    """Per-level recompressed outgoing operators: hier with the ladder == hier without it ==
    direct, within the hierarchical tolerance; the ladder lowers the grid pair count."""
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = _phys("C2")
    assert tab.ladder_r is not None and len(tab.ladder_r) >= 2
    x = random_coeffs(cfg.N, tab.K, 2004)
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    h1 = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, use_ladder=True)
    h0 = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, use_ladder=False)
    yd = gpu_matvec(hd, x)
    assert rel(gpu_matvec(h1, x), yd) <= HIER_TOL
    assert rel(gpu_matvec(h0, x), yd) <= HIER_TOL
    assert h1.stats()["hier_grid_pairs"] < 0.8 * h0.stats()["hier_grid_pairs"]


def test_hier_C5_full_size_sampled_rows_bench_config():
    """C5 (N = 100,000, the bench.py workload) in exactly the configuration bench.py times (physical tables with
    the per-level ladder, precision 1e-9, seeded x of bench.py): sampled output blocks against the oracle, which
    computes those rows one by one by the brute-force direct sum."""
    cfg = CONFIGS["C5"]
    c = cfg.centers()
    tab = _phys("C5")
    x = random_coeffs(cfg.N, tab.K, 2000 + 5)
    h = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    y = gpu_matvec(h, x)
    assert np.all(np.isfinite(y))
    rows = np.random.default_rng(55).choice(cfg.N, 2, replace=False)
    assert rel(y[rows], O.matvec(cfg.kind, c, tab, x, rows=rows)) <= HIER_TOL


_FAR_CHILD = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_1906_04209_b200 as nc
from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
cfg = CONFIGS[os.environ.get("CFG", "C3")]
tab = load_tables(os.path.join(os.environ["ROOT"], "tables", "data", cfg.name + ".npz"))
h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
x = torch.from_numpy(h.to_internal(random_coeffs(cfg.N, tab.K, 2006))).cuda()
np.save(os.environ["OUT"], h.matvec(x).cpu().numpy())
"""


@pytest.mark.parametrize("cfg,far", [("C3", "8,2,4,64,9,3,2"), ("C3", "8,2,4,64,10,3,3"), ("C3", "8,2,4,64,5,3,3"),
                                     ("C3", "8,2,4,64,8,3,2"), ("C5", "8,2,4,64,9,3,2"), ("C4", "8,2,4,64,9,3,2")])
def test_far_field_pair_variant_error(tmp_path, cfg, far):
    """k_pairs_grid_w's far-field evaluations (R23: dot-product distance + one-Newton rsqrt; R25: the
    exponent-indexed log table with c from rcp.approx; R32: the unclamped table, FB = 9 quadratic or FB = 7 cubic;
    R35: the same with high-word SFU seeds, the defaults) against the EXACT difference-form pair kernel on the same grids and sources (the CTA-level kernel,
    far 0), at the C3 / C4 / C5 epsilons: the difference must stay far below the hierarchical precision."""
    import subprocess
    import sys
    outs = []
    for v in ("32,2,4,256,0", far):   # the exact form on the same 64-point units (one-warp CTAs)
        out = str(tmp_path / f"y{len(outs)}.npy")
        env = dict(os.environ, NC_TUNING="1", NC_GRID_VARIANT=v, ROOT=ROOT, OUT=out, CFG=cfg)
        subprocess.run([sys.executable, "-c", _FAR_CHILD], env=env, check=True, timeout=900)
        outs.append(np.load(out))
    assert rel(outs[1], outs[0]) <= 1e-11


@pytest.mark.parametrize("env", [{"NC_INTERP_SEP": "0"}, {"NC_TRANSFORM": "0"}, {"NC_INTERP_VARIANT": "128,4,1,4"},
                                 {"NC_INTERP_VARIANT": "128,4,2,4"}, {"NC_INTERP_VARIANT": "128,2,3,4"},
                                 {"NC_INTERP_VARIANT": "128,2,0,4"}])
def test_step4_evaluation_variants_agree(tmp_path, env):
    """Step 4 evaluated three ways: angular sums first with register accumulators (default),
    Chebyshev sums first (MB = 1) or blocked orders (MB = 2), and single-member groups separably on the Zernike node
    rings (k_interp_sep) or directly (NC_INTERP_SEP=0); step 4a's ring Fourier sums by Clenshaw's recurrence
    (default, R37) or by tabulated twiddles (NC_TRANSFORM=0).  The same expansion at the same nodes: rounding-level agreement."""
    import subprocess
    import sys
    outs = []
    for e in ({}, env):   # the per-node order truncation (R26c) and the proxies (R36) off in both: the same
        out = str(tmp_path / f"y{len(outs)}.npy")   # expansion at the same nodes, evaluated two ways
        subprocess.run([sys.executable, "-c", _FAR_CHILD], env=dict(os.environ, NC_TUNING="1", ROOT=ROOT, OUT=out, NC_INTERP_TRUNC="0",
                                                                    NC_PROXY="0", **e), check=True, timeout=600)
        outs.append(np.load(out))
    assert rel(outs[1], outs[0]) <= 1e-13


def test_step4_order_truncation_below_tolerance(tmp_path):
    """The per-node order truncation of step 4 (R26c) drops only orders below the grid tolerance: the
    matvec moves by far less than the requested precision (C3)."""
    import subprocess
    import sys
    outs = []
    for v in ("0", "1"):
        out = str(tmp_path / f"y{v}.npy")
        subprocess.run([sys.executable, "-c", _FAR_CHILD], env=dict(os.environ, NC_TUNING="1", ROOT=ROOT, OUT=out, NC_INTERP_TRUNC=v),
                       check=True, timeout=600)
        outs.append(np.load(out))
    assert rel(outs[1], outs[0]) <= 1e-10


_PROXY_CHILD = _FAR_CHILD + r"""
import json
st = h.stats()
json.dump({k: st[k] for k in ("proxy_n", "proxy_kappa", "proxy_far_frac")}, open(os.environ["OUT"] + ".json", "w"))
"""


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_step4_proxies_agree_with_nodes(tmp_path, cfg):
    """DESIGN.md R36: the far levels of step 4 evaluated at the patch's proxy points and carried to the Zernike nodes
    by the proxy rule's matrix, against every level evaluated at the nodes (NC_PROXY=0, the paper's literal step 4,
    PAPER.md:1381-1397): the two matvecs differ by far less than the requested precision (1e-9), and the proxies are
    in use on a large share of the (patch, level) pairs."""
    import json
    import subprocess
    import sys
    outs, stats = [], []
    for e in ({"NC_PROXY": "0"}, {}):
        out = str(tmp_path / f"y{len(outs)}.npy")
        subprocess.run([sys.executable, "-c", _PROXY_CHILD],
                       env=dict(os.environ, NC_TUNING="1", ROOT=ROOT, OUT=out, CFG=cfg, **e), check=True, timeout=900)
        outs.append(np.load(out))
        stats.append(json.load(open(out + ".json")))
    assert stats[0]["proxy_n"] == 0
    assert stats[1]["proxy_n"] > 0 and stats[1]["proxy_far_frac"] > 0.3, stats[1]
    assert rel(outs[1], outs[0]) <= 1e-10


@pytest.mark.parametrize("precision", [1e-7, 1e-11])
def test_hier_precision_knob_C2(precision):
    """The requested precision controls the incoming-grid tolerance (R21): the matvec error tracks it
    (<= precision, with the calibrated margin), and a tighter request costs more grid pairs."""
    cfg = CONFIGS["C2"]
    c = cfg.centers()
    tab = _phys("C2")
    x = random_coeffs(cfg.N, tab.K, 2007)
    hd = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_DIRECT)
    hh = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=precision)
    hr = _nc().Handle(cfg.kind, c, cfg.eps, tab, mode=_nc().NC_HIER, precision=1e-9)
    assert rel(gpu_matvec(hh, x), gpu_matvec(hd, x)) <= max(precision, 1e-11)
    if precision < 1e-9:
        assert hh.stats()["hier_grid_pairs"] > hr.stats()["hier_grid_pairs"]
    else:
        assert hh.stats()["hier_grid_pairs"] < hr.stats()["hier_grid_pairs"]


@pytest.mark.parametrize("layout,N,eps,kind", [("uniform", 37, 0.05, 0), ("vmf", 300, 0.01, 1), ("uniform", 2, 0.3, 0)])
def test_hier_small_layouts_vs_oracle(layout, N, eps, kind):
    """Small hierarchical cases (shallow trees, near lists, N = 2) against the oracle's full brute-force matvec,
    synthetic tables with real node geometry (SURVEY.md §7 phase 1)."""
    c = make_centers(layout, N, eps, seed=11)
    tab = synthetic_tables(kind, eps, seed=3)
    x = random_coeffs(N, tab.K, 12)
    h = _nc().Handle(kind, c, eps, tab, mode=_nc().NC_HIER, precision=1e-9)
    assert rel(gpu_matvec(h, x), O.matvec(kind, c, tab, x)) <= HIER_TOL


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_matvec_bitwise_reproducible(name):
    """Two matvecs of the same input are bitwise identical (fixed-order reductions everywhere, R16).  With
    compute-sanitizer closed on this GPU pool, this is also the run-time evidence against races in the warp-level
    grid kernel's cp.async double buffer and k_interp's: a race would make the sums order- or timing-dependent."""
    cfg = CONFIGS[name]
    tab = _phys(name)
    h = _nc().Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=_nc().NC_HIER, precision=cfg.precision)
    x = torch.from_numpy(h.to_internal(random_coeffs(cfg.N, tab.K, 31))).cuda()
    ys = [h.matvec(x).cpu().numpy() for _ in range(3)]
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])
    h.close()


def test_tuning_knobs_ignored_without_nc_tuning(tmp_path):
    """The numerics-changing knobs (here the grid kernel variant and the interpolation truncation) are read only with
    NC_TUNING=1: without it a stray environment variable leaves the default matvec bit for bit."""
    import subprocess
    import sys
    outs = []
    for extra in ({}, {"NC_GRID_VARIANT": "32,2,4,256,0", "NC_INTERP_TRUNC": "0"}):
        out = str(tmp_path / f"y{len(outs)}.npy")
        env = {k: v for k, v in os.environ.items() if k != "NC_TUNING"}
        subprocess.run([sys.executable, "-c", _FAR_CHILD], env=dict(env, ROOT=ROOT, OUT=out, **extra), check=True,
                       timeout=600)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
