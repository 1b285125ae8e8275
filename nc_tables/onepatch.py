"""One-patch solver: B = S^{-1} Q on the fine grid (PAPER.md §"The one-patch integral equation", :1466-1687;
Step 1(a), :1287-1294).

Fourier reduction (eq:modalinteqn): for data f(t) cos(m theta) (or sin), sigma = sigma_m(t) cos(m theta) with
    2 pi int_0^eps G_m(t, t') sigma_m(t') sin t' dt' = f(t).
Radial discretisation: panels [a_{i-1}, a_i] dyadically refined toward eps,
a_0 = 0, a_i = eps (1 - 2^-i) (i < npan), a_npan = eps; sigma_m is a degree-(k-1) polynomial (Lagrange at
k Gauss-Legendre nodes) on every panel but the last, where sigma_m = g(t) / sqrt(eps - t) with g a polynomial at
k Gauss-Jacobi (alpha = -1/2, beta = 0) nodes.  Collocation at the same nodes; matrix entries by graded
Gauss-Legendre quadrature in t' (log singularity at t' = t_i; the last panel via t' = eps - s^2) of the
modal kernel (kernel.modal).  One LU per Fourier mode, reused for every Zernike right-hand side.

Fine grid: collocation radii x n_theta equispaced angles; weights = panel Gauss weight
x sin t (x sqrt(eps - t) on the last panel, which carries the Jacobi weight) x 2 pi / n_theta.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from . import zernike
from .kernel import modal
from .quad import barycentric_matrix, gauss_jacobi, gauss_legendre, singular_rule


@dataclass
class RadialGrid:
    eps: float
    npan: int
    k: int
    edges: np.ndarray        # npan + 1
    t: np.ndarray            # collocation / fine-grid radii (npan * k)
    w: np.ndarray            # radial quadrature weights for int h(t) sigma(t) sin t dt  (sigma samples)
    panel: np.ndarray        # panel index of each node


def radial_grid(eps: float, npan: int = 13, k: int = 20) -> RadialGrid:
    edges = np.array([0.0] + [eps * (1.0 - 2.0 ** (-i)) for i in range(1, npan)] + [eps])
    ts, ws, ps = [], [], []
    x, w = gauss_legendre(k)
    for i in range(npan - 1):
        a, b = edges[i], edges[i + 1]
        h = 0.5 * (b - a)
        t = a + h * (x + 1.0)
        ts.append(t)
        ws.append(h * w * np.sin(t))
        ps.append(np.full(k, i))
    a = edges[npan - 1]
    xj, wj = gauss_jacobi(k, -0.5, 0.0)      # weight (1 - x)^(-1/2); x = +1 <-> t = eps
    t = a + 0.5 * (eps - a) * (xj + 1.0)
    # int_a^eps F(t) (eps - t)^(-1/2) dt = sqrt((eps - a)/2) sum_j wj F(t_j);  sigma = g / sqrt(eps - t)
    ts.append(t)
    ws.append(np.sqrt(0.5 * (eps - a)) * wj * np.sqrt(eps - t) * np.sin(t))
    ps.append(np.full(k, npan - 1))
    return RadialGrid(eps, npan, k, edges, np.concatenate(ts), np.concatenate(ws), np.concatenate(ps))


def _row_rules(g: RadialGrid, ti: float):
    """For collocation radius ti: per panel (t' nodes, weights incl. sin t' and 2 pi, Lagrange matrix)."""
    out = []
    for pi in range(g.npan):
        a, b = g.edges[pi], g.edges[pi + 1]
        nodes = g.t[g.panel == pi]
        if pi < g.npan - 1:
            tq, wq = singular_rule(a, b, ti)
            L = barycentric_matrix(nodes, tq)
            wt = 2.0 * np.pi * wq * np.sin(tq)
        else:
            # t' = eps - s^2, s in [0, sqrt(eps - a)]: (eps - t')^(-1/2) dt' = 2 ds
            smax = np.sqrt(g.eps - a)
            si = np.sqrt(max(g.eps - ti, 0.0))
            sq, wq = singular_rule(0.0, smax, si)
            tq = g.eps - sq * sq
            L = barycentric_matrix(nodes, tq)
            wt = 2.0 * np.pi * 2.0 * wq * np.sin(tq)
        out.append((tq, wt, L))
    return out


def modal_matrices(kind: int, g: RadialGrid, M: int, modal_fn=None):
    """A_m (n x n) for m = 0..M: rows = collocation radii, columns = nodal unknowns (sigma or g values).
    ``modal_fn(kind, t, tp, M)``: the modal-kernel evaluator for all rows' quadrature pairs at once (default the
    numpy kernel.modal; the GPU one is paper_1906_04209_b200.modal_kernels with the same phi rule, NEXT-1)."""
    n = g.t.size
    A = np.zeros((M + 1, n, n))
    rules_all = [_row_rules(g, ti) for ti in g.t]
    tq_all = [np.concatenate([r[0] for r in rules]) for rules in rules_all]
    T = np.concatenate([np.full(tq.size, ti) for ti, tq in zip(g.t, tq_all)])
    TQ = np.concatenate(tq_all)
    G_all = (modal_fn or modal)(kind, T, TQ, M)                # (sum nq, M+1)
    row0 = np.concatenate([[0], np.cumsum([tq.size for tq in tq_all])])
    for i, ti in enumerate(g.t):
        rules = rules_all[i]
        Gm = G_all[row0[i]:row0[i + 1]]                         # (nq, M+1)
        off = 0
        for pi, (tqp, wt, L) in enumerate(rules):
            sl = slice(off, off + tqp.size)
            off += tqp.size
            cols = np.where(g.panel == pi)[0]
            # A[m, i, cols] = sum_q G_m(ti, t'_q) wt_q L[q, :]
            A[:, i, cols] = (Gm[sl] * wt[:, None]).T @ L
    return A


@dataclass
class OnePatch:
    kind: int
    eps: float
    M: int
    grid: RadialGrid
    n_theta: int
    sigma_radial: np.ndarray   # (K, n_r): sigma_a(t_j) (the singular density, not g)
    basis: list                # (n, m, c) per column


def solve_onepatch(kind: int, eps: float, M: int = 15, npan: int = 13, k: int = 20, n_theta: int | None = None,
                   A=None, modal_fn=None) -> OnePatch:
    g = radial_grid(eps, npan, k)
    if A is None:
        A = modal_matrices(kind, g, M, modal_fn)
    idx = zernike.basis_indices(M)
    sig = np.zeros((len(idx), g.t.size))
    last = g.panel == g.npan - 1
    for m in range(M + 1):
        cols = [a for a, (n, mm, c) in enumerate(idx) if mm == m]
        if not cols:
            continue
        lu = sla.lu_factor(A[m])
        F = np.stack([zernike.radial(idx[a][0], m, g.t / eps) / np.sqrt(zernike.norm2(idx[a][0], m))
                      for a in cols], axis=1)
        U = sla.lu_solve(lu, F)
        U[last] /= np.sqrt(eps - g.t[last])[:, None]              # g -> sigma on the last panel
        sig[cols] = U.T
    return OnePatch(kind, eps, M, g, n_theta or (4 * M + 4), sig, idx)


def fine_grid(op: OnePatch):
    """Fine-grid points (canonical frame), weights w^f and B (n_f x K)."""
    g = op.grid
    nth = op.n_theta
    th = 2.0 * np.pi * np.arange(nth) / nth
    T, TH = np.meshgrid(g.t, th, indexing="ij")              # radial-major
    xyz = np.stack([np.sin(T) * np.cos(TH), np.sin(T) * np.sin(TH), np.cos(T)], axis=-1).reshape(-1, 3)
    wf = (g.w[:, None] * np.full(nth, 2.0 * np.pi / nth)[None, :]).ravel()
    B = np.empty((xyz.shape[0], len(op.basis)))
    for a, (n, m, c) in enumerate(op.basis):
        ang = np.cos(m * th) if c > 0 else np.sin(m * th)
        B[:, a] = (op.sigma_radial[a][:, None] * ang[None, :]).ravel()
    return xyz, wf, B
