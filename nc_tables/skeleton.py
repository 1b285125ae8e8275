"""Skeletonised outgoing representation T = Pi W B (§7.1, :1104-1173; Step 1(b), :1295-1299).

Training grid on the far-field region Theta = {arc distance from the patch centre > 2 eps}:
dyadic shells [2 eps 2^s, 2 eps 2^(s+1)] in arc distance (Gauss-Legendre radii per shell) x equispaced azimuths,
up to the antipode.  A_{jl} = G(x^t_j, x^f_l) (n_t x n_f).  The ID is computed from a
Gaussian sketch Y = Omega A (the randomised ID of the paper's reference [liberty07]) by column-pivoted QR:
Y[:, J] Pi ~= Y, p = #{|R_kk| > tol |R_11|}, skeleton x^f_{pi(m)} = x^f_{J_m}; then T = Pi W B (eq:Tmap).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .kernel import green_xyz
from .quad import gauss_legendre


def training_grid(eps: float, n_per_shell: int = 10, n_az: int = 96, inner: float = 2.0):
    r0 = inner * eps
    shells = []
    a = r0
    while a < np.pi - 1e-12:
        b = min(2.0 * a, np.pi)
        shells.append((a, b))
        a = b
    x, _ = gauss_legendre(n_per_shell)
    rs = np.concatenate([lo + 0.5 * (hi - lo) * (x + 1.0) for lo, hi in shells] + [[r0, np.pi]])
    az = 2.0 * np.pi * (np.arange(n_az) + 0.5) / n_az
    R, AZ = np.meshgrid(rs, az, indexing="ij")
    return np.stack([np.sin(R) * np.cos(AZ), np.sin(R) * np.sin(AZ), np.cos(R)], axis=-1).reshape(-1, 3)


def test_matrix(n_train: int, oversample: int = 400, seed: int = 0, chunk: int = 512) -> np.ndarray:
    """The Gaussian test matrix Omega (l x n_train), drawn in the column chunks interp_decomp consumes."""
    rng = np.random.default_rng(seed)
    l = min(oversample, n_train)
    return np.concatenate([rng.standard_normal((l, min(n_train, a + chunk) - a)) for a in range(0, n_train, chunk)],
                          axis=1)


def interp_decomp(kind: int, train: np.ndarray, fine: np.ndarray, tol: float, oversample: int = 400, seed: int = 0,
                  chunk: int = 512, sketch=None):
    """Column ID of A = G(train, fine) from a Gaussian sketch.  Returns (J, Pi) with A ~= A[:, J] Pi.
    ``sketch(kind, train, fine, omega)``: optional Y = omega A evaluator (the GPU one: paper_1906_04209_b200.id_sketch,
    NEXT-1); default the numpy chunk loop below."""
    l = min(oversample, train.shape[0])
    if sketch is not None:
        Y = sketch(kind, train, fine, test_matrix(train.shape[0], oversample, seed, chunk))
    else:
        rng = np.random.default_rng(seed)
        Y = np.zeros((l, fine.shape[0]))
        for a in range(0, train.shape[0], chunk):
            b = min(train.shape[0], a + chunk)
            A = green_xyz(kind, train[a:b, None, :], fine[None, :, :])
            Y += rng.standard_normal((l, b - a)) @ A
    Q, R, piv = sla.qr(Y, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    p = int(np.sum(d > tol * d[0]))
    R11, R12 = R[:p, :p], R[:p, p:]
    Pi = np.zeros((p, fine.shape[0]))
    Pi[:, piv[:p]] = np.eye(p)
    Pi[:, piv[p:]] = sla.solve_triangular(R11, R12)
    return piv[:p], Pi


def outgoing_error(kind: int, fine, wf, B, shat, T, eps: float, n_test: int = 400, seed: int = 1, inner: float = 2.0):
    """max relative error of the compressed field (eq:outgoingcompressed) over random far-field points and
    random coefficient vectors, relative to the field's max norm."""
    rng = np.random.default_rng(seed)
    r0 = inner * eps * (1.0 + 1e-9)
    rad = r0 * (np.pi / r0) ** rng.random(n_test) ** 3
    az = 2.0 * np.pi * rng.random(n_test)
    X = np.stack([np.sin(rad) * np.cos(az), np.sin(rad) * np.sin(az), np.cos(rad)], axis=-1)
    F = rng.standard_normal((B.shape[1], 8))
    full = green_xyz(kind, X[:, None, :], fine[None, :, :]) @ (wf[:, None] * (B @ F))
    comp = green_xyz(kind, X[:, None, :], shat[None, :, :]) @ (T @ F)
    return float(np.max(np.abs(full - comp)) / np.max(np.abs(full)))
