"""Residual-grid table for the L2 residual diagnostic (NEXT-4, eq:l2res).

    res_i = || S sigma_i + sum_{j != i} S_ij sigma_j - 1 ||_{L2(Gamma_i)} / |Gamma_i|

"computed by quadrature on a Legendre-Fourier grid which does not overlap with the grid on which the integral
equation is solved".  Per patch radius this builder provides, in the canonical frame:
  res_rhat (n_res x 3)  the residual grid: n_r Gauss-Legendre radii in t on [0, eps] x n_theta equispaced angles
                        offset by half a step (2M + 3 of them: neither the solve's collocation radii nor the Zernike
                        sampling grid)
  res_w    (n_res)      quadrature weights of int_Gamma f dS (GL weight x sin t x 2 pi / n_theta)
  res_S    (n_res x K)  (S sigma_a)(x_k): the self-patch single-layer potential of the one-patch solution of each
                        Zernike datum q_a, evaluated at the residual grid by the one-patch solver's own singular
                        quadrature (onepatch._row_rules at the new radii), so S sigma_i = res_S fhat_i there.
If the one-patch solve were exact, res_S would equal q_a at the residual points: the difference is the one-patch
residual the paper reports as eq:patcherrl2, pinned by tests/test_tables.py.
"""
from __future__ import annotations

import numpy as np

from . import zernike
from .kernel import modal
from .onepatch import _row_rules, solve_onepatch


def residual_table(kind: int, eps: float, M: int = 15, npan: int = 13, k: int = 20, n_r: int = 24,
                   n_theta: int | None = None, op=None):
    op = op or solve_onepatch(kind, eps, M, npan, k)
    g = op.grid
    n_theta = n_theta or (2 * M + 3)
    x, w = np.polynomial.legendre.leggauss(n_r)
    tr = 0.5 * eps * (x + 1.0)
    wr = 0.5 * eps * w * np.sin(tr)
    th = 2.0 * np.pi * (np.arange(n_theta) + 0.5) / n_theta
    idx = op.basis
    # nodal unknowns of each basis solution (sigma on the regular panels, g = sigma sqrt(eps - t) on the last one)
    last = g.panel == g.npan - 1
    U = op.sigma_radial.copy()
    U[:, last] *= np.sqrt(eps - g.t[last])[None, :]
    # radial part: SR[r, a] = row_m(t_r) . U_a = (S sigma_a)'s m-th Fourier coefficient at radius t_r
    SR = np.zeros((n_r, len(idx)))
    for ri, t in enumerate(tr):
        rules = _row_rules(g, t)
        tq = np.concatenate([r[0] for r in rules])
        Gm = modal(kind, np.full(tq.size, t), tq, M)
        row = np.zeros((M + 1, g.t.size))
        off = 0
        for pi, (tqp, wt, L) in enumerate(rules):
            sl = slice(off, off + tqp.size)
            off += tqp.size
            cols = np.where(g.panel == pi)[0]
            row[:, cols] = (Gm[sl] * wt[:, None]).T @ L
        for a, (n, m, c) in enumerate(idx):
            SR[ri, a] = row[m] @ U[a]
    T, TH = np.meshgrid(tr, th, indexing="ij")               # radius-major
    S = np.empty((n_r * n_theta, len(idx)))
    for a, (n, m, c) in enumerate(idx):
        ang = np.cos(m * th) if c > 0 else np.sin(m * th)
        S[:, a] = (SR[:, a][:, None] * ang[None, :]).ravel()
    rhat = zernike.patch_xyz(eps, (T / eps).ravel(), TH.ravel())
    wts = (wr[:, None] * np.full(n_theta, 2.0 * np.pi / n_theta)[None, :]).ravel()
    return dict(res_rhat=rhat, res_w=wts, res_S=S, res_r=(T / eps).ravel(), res_theta=TH.ravel())


def add_to_tables(path: str, npan: int = 13, k: int = 20):
    """Append res_rhat / res_w / res_S to an existing table file (the other arrays are kept bit for bit)."""
    d = dict(np.load(path, allow_pickle=False))
    rt = residual_table(int(d["kind"]), float(d["eps"]), int(d["M"]), npan, k)
    d.update(res_rhat=rt["res_rhat"], res_w=rt["res_w"], res_S=rt["res_S"])
    np.savez(path, **d)


if __name__ == "__main__":
    import glob
    import os
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in sys.argv[1:] or sorted(glob.glob(os.path.join(root, "tables", "data", "C*.npz"))):
        t0 = time.time()
        add_to_tables(p)
        print(f"{p}: residual table added in {time.time() - t0:.1f} s", flush=True)
