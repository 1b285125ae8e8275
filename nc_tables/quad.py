"""Quadrature rules for the Step-1 table builder (§one-patch, :1581-1687)."""
from __future__ import annotations

from functools import lru_cache

import numpy as np
from scipy.special import roots_jacobi


@lru_cache(maxsize=None)
def gauss_legendre(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return x, w


@lru_cache(maxsize=None)
def gauss_jacobi(n: int, alpha: float, beta: float):
    x, w = roots_jacobi(n, alpha, beta)
    return x, w


def map_rule(a, b, n):
    x, w = gauss_legendre(n)
    h = 0.5 * (b - a)
    return a + h * (x + 1.0), h * w


def composite(edges, n):
    xs, ws = [], []
    for a, b in zip(edges[:-1], edges[1:]):
        if b > a:
            x, w = map_rule(a, b, n)
            xs.append(x)
            ws.append(w)
    return np.concatenate(xs), np.concatenate(ws)


def graded_edges(a, b, toward_a: bool, hmin: float, ratio: float):
    """Breakpoints of [a, b] refined geometrically toward one endpoint down to width hmin."""
    L = b - a
    if L <= 0:
        return [a, b]
    offs = [L]
    h = L
    while h * ratio > hmin:
        h *= ratio
        offs.append(h)
    offs.append(0.0)
    offs = offs[::-1]                      # 0, hmin-ish, ..., L
    if toward_a:
        return [a + o for o in offs]
    return [b - o for o in offs[::-1]]


def singular_rule(a, b, c, n_sub=20, n_far=32, ratio=0.25, rel_floor=1e-15):
    """Nodes/weights on [a, b] for integrands smooth except for a log-type singularity at c.

    c inside (a, b): split at c, grade toward c on both sides.  c outside: grade toward the nearer
    endpoint down to the singularity's distance; far away: plain Gauss-Legendre with n_far nodes."""
    L = b - a
    floor = rel_floor * max(L, abs(c), 1e-300)
    if a < c < b:
        e1 = graded_edges(a, c, toward_a=False, hmin=floor, ratio=ratio)
        e2 = graded_edges(c, b, toward_a=True, hmin=floor, ratio=ratio)
        x1, w1 = composite(e1, n_sub)
        x2, w2 = composite(e2, n_sub)
        return np.concatenate([x1, x2]), np.concatenate([w1, w2])
    dist = (a - c) if c <= a else (c - b)
    if dist >= L:
        return map_rule(a, b, n_far)
    toward_a = c <= a
    e = graded_edges(a, b, toward_a=toward_a, hmin=max(0.5 * dist, floor), ratio=ratio)
    return composite(e, n_sub)


def barycentric_matrix(nodes, pts):
    """Lagrange basis values L[q, j] = l_j(pts[q]) for interpolation at `nodes` (barycentric form)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    pts = np.asarray(pts, dtype=np.float64)
    n = nodes.size
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    # weights scaled to avoid overflow
    lw = -np.sum(np.log(np.abs(diff)), axis=1)
    sgn = np.prod(np.sign(diff), axis=1)
    wb = sgn * np.exp(lw - lw.max())
    D = pts[:, None] - nodes[None, :]
    exact = D == 0.0
    D[exact] = 1.0
    T = wb[None, :] / D
    L = T / T.sum(axis=1, keepdims=True)
    rows = np.where(exact.any(axis=1))[0]
    for r in rows:
        L[r] = exact[r].astype(np.float64)
    return L
