"""The five seeded workloads of BASELINE.json ``configs``.

Only sizes, seeds and layout recipes live here; no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import layouts

INTERIOR, EXTERIOR = 0, 1


@dataclass(frozen=True)
class Config:
    name: str
    kind: int
    N: int
    eps: float
    layout: str
    seed: int
    modes: tuple
    precision: float = 1e-9
    gmres_tol: float = 1e-10

    def centers(self) -> np.ndarray:
        return make_centers(self.layout, self.N, self.eps, self.seed)


CONFIGS = {
    "C1": Config("C1", INTERIOR, 10, 0.1, "uniform", 1001, ("direct",)),
    "C2": Config("C2", EXTERIOR, 1000, 0.02, "uniform", 1002, ("direct", "hier")),
    "C3": Config("C3", INTERIOR, 10000, 0.009, "fibonacci", 1003, ("hier",)),
    "C4": Config("C4", EXTERIOR, 10000, 0.005, "vmf", 1004, ("hier",)),
    "C5": Config("C5", INTERIOR, 100000, 0.003, "fibonacci", 1005, ("hier",)),
}


def make_centers(layout: str, N: int, eps: float, seed: int, sep: float = 3.0) -> np.ndarray:
    if layout == "uniform":
        pts, _ = layouts.uniform_rsa(N, eps, seed, sep=sep)
    elif layout == "fibonacci":
        pts = layouts.fibonacci(N, seed)
    elif layout == "fibonacci_unrotated":
        pts = layouts.fibonacci(N, None)
    elif layout == "vmf":
        pts, _ = layouts.vmf_mixture(N, eps, seed, sep=sep)
    else:
        raise ValueError(layout)
    return np.ascontiguousarray(pts, dtype=np.float64)


def random_coeffs(N: int, K: int, seed: int) -> np.ndarray:
    """x ~ N(0,1)^{N K}, patch-major (K contiguous per patch); SURVEY.md §8(d) 'Matvec inputs'."""
    return np.random.default_rng(seed).standard_normal((N, K))
