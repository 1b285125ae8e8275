"""Zernike basis on a patch, sampling nodes and the discrete Zernike transform P (§4, :816-870).

  Z_n^m  = R_n^m(r) cos(m theta),   Z_n^{-m} = R_n^m(r) sin(m theta),   0 <= m <= n <= M, n - m even
  R_n^m(r) = (-1)^{(n-m)/2} r^m P^{(m,0)}_{(n-m)/2}(1 - 2 r^2)
  int_0^{2pi} int_0^1 Z Z' r dr dtheta = (1 + delta_{m0}) pi / (2n + 2) delta delta   (eq:zorthog)

q_a = Z / sqrt(norm): orthonormal on the unit disk with the flat measure r dr dtheta, r = t / eps (t = arc length
from the patch centre) -- DESIGN.md reading R6.  Ordering: n ascending; within n, m ascending; cos before sin.
K = (M+1)(M+2)/2 (reading R5).

Sampling nodes ("Gauss-Legendre rule in the radial variable and a trapezoidal rule in the angular
variable"): M+1 Gauss-Legendre radii on [0,1] x 2M+2 equispaced angles; exact for products of two degree-M
functions (radial degree <= 2M+1, angular frequency <= 2M < 2M+2), so P Q = I_K exactly.
"""
from __future__ import annotations

import numpy as np
from scipy.special import eval_jacobi


def basis_indices(M: int):
    """List of (n, m, c) with c = +1 (cos) / -1 (sin), in table order."""
    out = []
    for n in range(M + 1):
        for m in range(n % 2, n + 1, 2):
            out.append((n, m, 1))
            if m > 0:
                out.append((n, m, -1))
    assert len(out) == (M + 1) * (M + 2) // 2
    return out


def radial(n: int, m: int, r):
    r = np.asarray(r, dtype=np.float64)
    k = (n - m) // 2
    return (-1.0) ** k * r ** m * eval_jacobi(k, m, 0, 1.0 - 2.0 * r * r)


def norm2(n: int, m: int) -> float:
    return (2.0 if m == 0 else 1.0) * np.pi / (2.0 * n + 2.0)


def q_eval(M: int, r, theta):
    """Orthonormal basis values, shape (len(r), K) for points (r, theta) on the unit disk."""
    r = np.asarray(r, dtype=np.float64).ravel()
    theta = np.asarray(theta, dtype=np.float64).ravel()
    idx = basis_indices(M)
    Q = np.empty((r.size, len(idx)))
    for a, (n, m, c) in enumerate(idx):
        ang = np.cos(m * theta) if c > 0 else np.sin(m * theta)
        Q[:, a] = radial(n, m, r) * ang / np.sqrt(norm2(n, m))
    return Q


def sampling_grid(M: int, n_r: int | None = None, n_theta: int | None = None, radial: str = "r"):
    """radial = "r": n_r (default M+1) Gauss-Legendre radii in r with weight r (2M+2 angles by default: K* = 512 at
    M = 15); radial = "r2": n_r (default (M+1)/2 rounded up) Gauss-Legendre nodes in s = r^2 (r dr = ds/2) with
    2M+1 angles (K* = 8 x 31 = 248 at M = 15).  Both integrate every product of two basis functions
    exactly (radial: R R' r is a polynomial of degree <= 2M+1 in r, or R R' of degree <= M in r^2; angular:
    frequencies <= 2M), so P Q = I_K either way."""
    if radial == "r2":
        n_r = n_r or (M + 2) // 2
        n_theta = n_theta or (2 * M + 1)
        x, w = np.polynomial.legendre.leggauss(n_r)
        r = np.sqrt(0.5 * (x + 1.0))
        wr = 0.25 * w                     # int_0^1 f r dr = int_0^1 f ds / 2, ds = dx / 2
        th = 2.0 * np.pi * np.arange(n_theta) / n_theta
        R, TH = np.meshgrid(r, th, indexing="ij")
        WR = np.broadcast_to(wr[:, None], R.shape)
        return R.ravel(), TH.ravel(), WR.ravel() * (2.0 * np.pi / n_theta)
    n_r = n_r or (M + 1)
    n_theta = n_theta or (2 * M + 2)
    x, w = np.polynomial.legendre.leggauss(n_r)
    r = 0.5 * (x + 1.0)
    wr = 0.5 * w
    th = 2.0 * np.pi * np.arange(n_theta) / n_theta
    R, TH = np.meshgrid(r, th, indexing="ij")
    WR = np.broadcast_to(wr[:, None], R.shape)
    return R.ravel(), TH.ravel(), (WR * R).ravel() * (2.0 * np.pi / n_theta)


def transform(M: int, n_r: int | None = None, n_theta: int | None = None, radial: str = "r"):
    """Returns (r, theta, P) with P (K x Kstar): coefficients = P @ samples (the discrete Zernike transform)."""
    r, th, w = sampling_grid(M, n_r, n_theta, radial)
    Q = q_eval(M, r, th)
    P = (Q * w[:, None]).T
    return r, th, P


def patch_xyz(eps: float, r, theta):
    """Canonical-frame point (patch centre at +z) at arc distance t = eps r, azimuth theta."""
    t = eps * np.asarray(r, dtype=np.float64)
    th = np.asarray(theta, dtype=np.float64)
    return np.stack([np.sin(t) * np.cos(th), np.sin(t) * np.sin(th), np.cos(t)], axis=-1)
