"""Seeded synthetic patch layouts (BASELINE.json ``configs``).

This module is shared by the oracle and the CUDA path and therefore holds *no* arithmetic of
the method: it only draws unit-sphere points.  The layouts stand in for the paper's own random /
Fibonacci / clustered layouts, whose seeds are not published (§9.2).

Recipes
-------
* ``uniform``  : normalised Gaussian triples, sequential rejection (RSA) at centre arc
  distance >= ``sep * eps`` (the well-separatedness condition of PAPER.md:641-646, §3).
* ``fibonacci``: z_i = 1 - (2i-1)/N, phi_i = 2*pi*i/golden**2, i = 1..N (the paper cites
  "Fibonacci spiral points" without a formula; reading R19),
  optionally followed by a seeded Haar rotation (QR of a 3x3 Gaussian, sign-fixed, det +1).
* ``vmf``      : equal-weight mixture of ``ncaps`` von Mises-Fisher caps (kappa) about uniform
  axes, sampled with Wood's inverse CDF w = 1 + log(u + (1-u) e^{-2 kappa}) / kappa, with the
  same sequential rejection.  Stands in for the paper's 20 dodecahedral clusters.
"""
from __future__ import annotations

import numpy as np

try:  # scipy is only a speed-up for the rejection test
    from scipy.spatial import cKDTree
except Exception:  # pragma: no cover
    cKDTree = None


def _chord(arc: float) -> float:
    return 2.0 * np.sin(0.5 * arc)


class _Rejector:
    """Sequential random-sequential-adsorption acceptance with a minimum arc distance."""

    def __init__(self, min_arc: float, capacity: int):
        self.r = _chord(min_arc)
        self.pts = np.zeros((capacity, 3))
        self.n = 0
        self._tree = None
        self._tree_n = 0
        self._pending = []

    def _near(self, x):
        # rebuild a KD tree occasionally; check the recent tail by brute force
        if cKDTree is not None and self.n - self._tree_n > 256:
            self._tree = cKDTree(self.pts[: self.n])
            self._tree_n = self.n
        if self._tree is not None and self._tree_n > 0:
            if self._tree.query_ball_point(x, self.r * (1 - 1e-15), return_length=True) > 0:
                return True
            tail = self.pts[self._tree_n: self.n]
        else:
            tail = self.pts[: self.n]
        if len(tail) == 0:
            return False
        d = np.linalg.norm(tail - x, axis=1)
        return bool(np.any(d < self.r))

    def offer(self, x) -> bool:
        if self._near(x):
            return False
        self.pts[self.n] = x
        self.n += 1
        return True


def haar_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation: QR of a 3x3 Gaussian, columns sign-fixed, det +1."""
    a = rng.standard_normal((3, 3))
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))[None, :]
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def uniform_rsa(n: int, eps: float, seed: int, sep: float = 3.0, max_proposals: int | None = None):
    rng = np.random.default_rng(seed)
    rej = _Rejector(sep * eps, n)
    budget = max_proposals or 200 * n + 1000
    tries = 0
    while rej.n < n:
        if tries >= budget:
            raise RuntimeError(f"uniform RSA placed only {rej.n}/{n} patches")
        g = rng.standard_normal(3)
        x = g / np.linalg.norm(g)
        rej.offer(x)
        tries += 1
    return rej.pts.copy(), tries


def fibonacci(n: int, seed: int | None = None):
    i = np.arange(1, n + 1, dtype=np.float64)
    golden = 0.5 * (1.0 + np.sqrt(5.0))
    z = 1.0 - (2.0 * i - 1.0) / n
    phi = 2.0 * np.pi * i / golden**2
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    pts = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    if seed is not None:
        rot = haar_rotation(np.random.default_rng(seed))
        pts = pts @ rot.T
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    return pts


def _vmf_sample(rng, axis, kappa):
    u = rng.random()
    w = 1.0 + np.log(u + (1.0 - u) * np.exp(-2.0 * kappa)) / kappa
    # uniform direction orthogonal to the axis
    v = rng.standard_normal(3)
    v -= v.dot(axis) * axis
    v /= np.linalg.norm(v)
    x = w * axis + np.sqrt(max(0.0, 1.0 - w * w)) * v
    return x / np.linalg.norm(x)


def vmf_mixture(n: int, eps: float, seed: int, ncaps: int = 20, kappa: float = 20.0, sep: float = 3.0,
                max_proposals: int | None = None):
    rng = np.random.default_rng(seed)
    axes = rng.standard_normal((ncaps, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    rej = _Rejector(sep * eps, n)
    budget = max_proposals or 200 * n + 1000
    tries = 0
    while rej.n < n:
        if tries >= budget:
            raise RuntimeError(f"vMF RSA placed only {rej.n}/{n} patches")
        c = rng.integers(ncaps)
        rej.offer(_vmf_sample(rng, axes[c], kappa))
        tries += 1
    return rej.pts.copy(), tries


def min_arc_distance(pts: np.ndarray) -> float:
    """Smallest centre-to-centre arc distance (KD tree on chords)."""
    if len(pts) < 2:
        return np.pi
    if cKDTree is not None:
        d, _ = cKDTree(pts).query(pts, k=2)
        c = d[:, 1].min()
    else:
        g = pts @ pts.T
        np.fill_diagonal(g, -2)
        c = np.sqrt(max(0.0, 2 - 2 * g.max()))
    return 2.0 * np.arcsin(min(1.0, c / 2))
