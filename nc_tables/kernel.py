"""Green's functions and their azimuthal Fourier (modal) coefficients for the table builder.

On-surface kernels (PAPER.md:355-358, eq:Gextonsurface; :396-399, eq:Gintonsurface), d = |x - x'|:
  G_E = 2/d - log(2/d) - log(1 + d/2),   G_I = 2/d + log(2/d) - log(1 + d/2).
Modal kernels: G_n(t, t') = (1/pi) int_0^pi G(d) cos(n phi) dphi, with
  d^2 = 4 sin^2((t - t')/2) + 4 sin t sin t' sin^2(phi/2)   (equivalent to PAPER.md:1545-1548, cancellation-free).
The phi integral is done by a Gauss-Legendre rule geometrically graded toward phi = 0, where the integrand is
nearly singular when t ~ t'.  (The paper evaluates G^(1) via half-integer Legendre functions and G^(2) in closed
form; the closed form pins this routine in tests/test_tables.py.)
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from .quad import composite

INTERIOR, EXTERIOR = 0, 1


def green_d(kind: int, d):
    d = np.asarray(d, dtype=np.float64)
    if kind == INTERIOR:
        return 2.0 / d + np.log(2.0 / d) - np.log1p(0.5 * d)
    return 2.0 / d - np.log(2.0 / d) - np.log1p(0.5 * d)


def green_xyz(kind: int, x, y):
    d = np.linalg.norm(np.asarray(x) - np.asarray(y), axis=-1)
    return green_d(kind, d)


@lru_cache(maxsize=None)
def phi_rule(n_per=14, ratio=1.0 / 3.0, levels=31, n_uniform=24):
    """Uniform panels of width pi/n_uniform (resolve cos(m phi), m <= ~40) plus geometric grading toward 0."""
    h = np.pi / n_uniform
    edges = [0.0] + [h * ratio ** k for k in range(levels, 0, -1)] + [h * k for k in range(1, n_uniform + 1)]
    x, w = composite(edges, n_per)
    return x, w


def modal(kind: int, t, tp, M: int, chunk: int = 4096):
    """G_m(t, t') for m = 0..M at paired points; returns array (npairs, M+1)."""
    t = np.asarray(t, dtype=np.float64).ravel()
    tp = np.asarray(tp, dtype=np.float64).ravel()
    phi, wphi = phi_rule()
    C = (wphi[:, None] * np.cos(np.outer(phi, np.arange(M + 1)))) / np.pi       # (nphi, M+1)
    s2 = np.sin(0.5 * phi) ** 2
    out = np.empty((t.size, M + 1))
    for a in range(0, t.size, chunk):
        b = min(t.size, a + chunk)
        A = 4.0 * np.sin(0.5 * (t[a:b] - tp[a:b])) ** 2
        B = 4.0 * np.sin(t[a:b]) * np.sin(tp[a:b])
        d = np.sqrt(A[:, None] + B[:, None] * s2[None, :])
        out[a:b] = green_d(kind, d) @ C
    return out


def modal_gpu(kind: int, t, tp, M: int):
    """kernel.modal on the GPU (nc_modal_kernels, NEXT-1) with the same phi rule."""
    import paper_1906_04209_b200 as nc
    phi, wphi = phi_rule()
    return nc.modal_kernels(kind, t, tp, M, phi, wphi)
