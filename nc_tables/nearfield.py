"""Near-field table for the near-surface potential (NEXT-3; PAPER.md:797-807 eq:recoversig,
PAPER.md:2069-2097 Fig. sphereplots at radius 1 - eps/5).

The density of a patch is sigma(t, theta) = sum_a fhat_a sigma_a(t) ang_a(theta) (eq:recoversig with the one-patch
solver's basis solutions; ang_a = cos(m_a theta) or sin(m_a theta)), known at the solver's radial nodes: k Gauss-
Legendre nodes on each regular panel (sigma_a is a degree-(k-1) polynomial there) and k Gauss-Jacobi nodes on the last
panel (sigma_a = g_a(t) / sqrt(eps - t), g_a a polynomial).  Points closer than a few eps to a
patch see its density through this representation instead of the compressed skeleton.  The table stores, in the
canonical patch frame (centre +z, theta from +x):
  near_edges (npan + 1)  panel breakpoints in t (arc length from the centre)
  near_t     (n_r)       the radial nodes (panel-major, k per panel)
  near_w     (n_r)       weights of int_0^eps F(t) sigma(t) sin t dt = sum_j near_w[j] F(t_j) sigma(t_j)
                         (the last panel's Gauss-Jacobi weight times sqrt(eps - t_j) already folded in)
  near_sigma (K x n_r)   sigma_a(t_j) (the singular density on the last panel, not g)
  near_m, near_c (K)     angular order and cos (+1) / sin (-1) of each basis column
  near_k     ()          nodes per panel
Both the oracle and the CUDA path read these arrays (they are patch-operator tables, an input of the method, like T
and P); neither imports this module.
"""
from __future__ import annotations

import numpy as np

from .onepatch import solve_onepatch


def near_table(kind: int, eps: float, M: int = 15, npan: int = 13, k: int = 20, op=None):
    op = op or solve_onepatch(kind, eps, M, npan, k)
    g = op.grid
    return dict(near_edges=np.asarray(g.edges, dtype=np.float64), near_t=np.asarray(g.t, dtype=np.float64),
                near_w=np.asarray(g.w, dtype=np.float64), near_sigma=np.ascontiguousarray(op.sigma_radial),
                near_m=np.array([m for _, m, _ in op.basis], dtype=np.int32),
                near_c=np.array([c for _, _, c in op.basis], dtype=np.int32), near_k=np.int32(g.k))


def add_to_tables(path: str, npan: int = 13, k: int = 20):
    """Append the near-field arrays to an existing table file (the other arrays are kept bit for bit)."""
    d = dict(np.load(path, allow_pickle=False))
    d.update(near_table(int(d["kind"]), float(d["eps"]), int(d["M"]), npan, k))
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
        print(f"{p}: near-field table added in {time.time() - t0:.1f} s", flush=True)
