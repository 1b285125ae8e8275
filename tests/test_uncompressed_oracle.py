"""the compressed outgoing representation against the uncompressed density it stands for.

eq:outgoingcompressed: for targets in Theta (arc > 2 eps from the source centre)
    sum_l G(x, f_l) w_l (B fhat)_l  ~=  sum_m G(x, s_m) (T fhat)_m,   T = Pi W B (eq:Tmap)
with the ID error of the skeleton.  Here the oracle recomputes both sides with its own brute-force
Green's-function sum (oracle_field.c) instead of trusting the error the table builder stored:
  * whole matvecs, oracle.matvec (skeleton, base T) vs oracle.matvec_uncompressed (fine grid, B), on C1 and on
    clusters of the C2 (exterior) and C5 (interior, eps = 0.003) layouts: the operator part agrees to ~10x the base ID
    tolerance 1e-11 (SURVEY.md §8(c) "Skeleton/T");
  * every per-level rung T_k on its own region {arc > r_k}: the compressed field's max error
    relative to the field's max over the rung's region and four random densities stays within 50x the rungs' ID
    tolerance (the ID bound carries a factor sqrt(p (n_f - p)) over the tolerance; measured <= 14x at 3e-10 for every
    rung of C2 and C5 -- the builder's own stored estimate, a sparser sample, is 2-5x lower).  This pointwise
    single-patch error is far more pessimistic than the matvec's: what the precision promises is checked on the
    matvec itself (tests/test_parity_golden_gpu.py, ladder on, including at precision = the ladder tolerance).
B, w and the fine grid f come from the Step-1 builder (nc_tables.onepatch), as T does; the arithmetic of both sides
is the oracle's."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_fine = {}


def _load(name):
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    if name not in _fine:
        from nc_tables import onepatch
        meta = eval(tab.meta["repr"], {"__builtins__": {}})
        op = onepatch.solve_onepatch(tab.kind, tab.eps, tab.M, meta["npan"], meta["k"], meta["n_theta"])
        _fine[name] = onepatch.fine_grid(op)
    return tab, _fine[name]


def _cluster(name, n):
    c = CONFIGS[name].centers()
    d = np.linalg.norm(c - c[0], axis=1)
    return np.ascontiguousarray(c[np.argsort(d)[:n]])


@pytest.mark.parametrize("name,n", [("C1", 10), ("C2", 16), ("C5", 8)])
def test_compressed_matvec_matches_uncompressed(name, n):
    tab, (fine, wf, B) = _load(name)
    c = CONFIGS[name].centers() if n == CONFIGS[name].N else _cluster(name, n)
    x = random_coeffs(len(c), tab.K, 81)
    yc = O.matvec(tab.kind, c, tab, x)
    yu = O.matvec_uncompressed(tab.kind, c, tab, fine, wf, B, x)
    err = np.linalg.norm(yc - yu) / np.linalg.norm(yu - x)
    assert err <= 1e-9, err


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_ladder_rungs_match_uncompressed(name):
    tab, (fine, wf, B) = _load(name)
    assert tab.ladder_r is not None
    rng = np.random.default_rng(5)
    F = rng.standard_normal((tab.K, 4))
    q_full = (wf[:, None] * (B @ F))                       # uncompressed charges of 4 densities
    off = np.concatenate([[0], np.cumsum(tab.ladder_p)])
    worst = 0.0
    for k, rk in enumerate(tab.ladder_r):
        # targets on the sphere in the rung's region {arc > r_k} about the source centre (the pole)
        arc = rk * (1.0 + 1e-9) * (np.pi / rk) ** (rng.random(300) ** 3)
        az = 2.0 * np.pi * rng.random(300)
        X = np.stack([np.sin(arc) * np.cos(az), np.sin(arc) * np.sin(az), np.cos(arc)], axis=-1)
        sk = tab.ladder_shat[off[k]:off[k + 1]]
        qc = tab.ladder_T[off[k]:off[k + 1]] @ F
        tp = np.full(len(X), -1, dtype=np.int64)
        full = np.stack([O.field(tab.kind, X, tp, fine, np.zeros(len(fine), dtype=np.int64), q_full[:, a])
                         for a in range(F.shape[1])], axis=1)
        comp = np.stack([O.field(tab.kind, X, tp, sk, np.zeros(len(sk), dtype=np.int64), qc[:, a])
                         for a in range(F.shape[1])], axis=1)
        worst = max(worst, float(np.max(np.abs(full - comp)) / np.max(np.abs(full))))
    assert tab.ladder_tol > 0
    assert worst <= 50.0 * tab.ladder_tol, (worst, tab.ladder_tol)
