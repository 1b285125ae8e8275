"""Patch-operator table container, file IO and *synthetic* tables.

The tables are the Step-1 outputs the paper stores per patch radius (§8
"Step 1": "only the p x K matrix T and the 1 x K vector I") plus the Zernike sampling nodes and
the discrete Zernike transform P (§6) and the skeleton nodes x^f_{pi(m)}
(eq:outgoingcompressed).  They are an *input* of ``nc_setup`` (SURVEY.md
§8(b)); both the oracle and the CUDA path read the same arrays.

Synthetic tables (``synthetic_tables``) keep the real node geometry (a tensor polar grid on the
patch: Gauss-Legendre radii x equispaced angles) but draw T, P and I at random:
matvec parity only needs *identical* tables on both sides.  Physical tables
come from ``nc_tables`` (the CPU Step-1 builder) and are stored with the same keys.

Layout conventions (all float64, C order):
  zhat  (Kstar, 3)  Zernike sampling nodes, canonical frame (patch centre = +z, theta=0 along +x)
  P     (K, Kstar)  discrete Zernike transform
  shat  (p, 3)      skeleton (outgoing) nodes, canonical frame
  T     (p, K)      outgoing map rho = T fhat (eq:Tmap)
  I     (K,)        integration row, I_sigma = I . sum_i fhat_i (eq:getI)
Optional per-level outgoing operators, rung k valid for targets at arc > ladder_r[k]:
  ladder_r (nk,), ladder_p (nk,) int32, ladder_shat (sum p_k, 3), ladder_T (sum p_k, K)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TABLE_VERSION = 1


@dataclass
class PatchTables:
    kind: int            # 0 = interior / narrow escape (G_I), 1 = exterior / narrow capture (G_E)
    eps: float           # patch radius in arc length
    M: int               # Zernike truncation, K = (M+1)(M+2)/2
    zhat: np.ndarray
    P: np.ndarray
    shat: np.ndarray
    T: np.ndarray
    I: np.ndarray
    meta: dict = field(default_factory=dict)
    ladder_r: np.ndarray | None = None
    ladder_p: np.ndarray | None = None
    ladder_shat: np.ndarray | None = None
    ladder_T: np.ndarray | None = None
    # optional residual-grid table for the L2 residual diagnostic (NEXT-4; nc_tables/residual.py):
    #   res_rhat (n_res, 3) residual grid (canonical frame), res_w (n_res,) weights of int_Gamma f dS,
    #   res_S (n_res, K) self-patch potential of each basis solution at the grid
    res_rhat: np.ndarray | None = None
    res_w: np.ndarray | None = None
    res_S: np.ndarray | None = None
    # optional near-field table for the near-surface potential (NEXT-3; nc_tables/nearfield.py): the one-patch
    # solver's radial panels and basis densities sigma_a(t) (canonical frame):
    #   near_edges (npan+1), near_t (n_r), near_w (n_r), near_sigma (K, n_r), near_m (K,), near_c (K,), near_k ()
    near_edges: np.ndarray | None = None
    near_t: np.ndarray | None = None
    near_w: np.ndarray | None = None
    near_sigma: np.ndarray | None = None
    near_m: np.ndarray | None = None
    near_c: np.ndarray | None = None
    near_k: int | None = None

    @property
    def K(self) -> int:
        return self.T.shape[1]

    @property
    def Kstar(self) -> int:
        return self.zhat.shape[0]

    @property
    def p(self) -> int:
        return self.shat.shape[0]

    def validate(self):
        K = (self.M + 1) * (self.M + 2) // 2
        assert self.T.shape == (self.p, K), (self.T.shape, self.p, K)
        assert self.P.shape == (K, self.Kstar)
        assert self.I.shape == (K,)
        assert self.zhat.shape == (self.Kstar, 3) and self.shat.shape == (self.p, 3)
        for a in (self.zhat, self.shat):
            assert np.allclose(np.linalg.norm(a, axis=1), 1.0, atol=1e-13)
        if self.res_S is not None:
            assert self.res_rhat.shape == (self.res_S.shape[0], 3) and self.res_w.shape == (self.res_S.shape[0],)
            assert self.res_S.shape[1] == K
        if self.near_sigma is not None:
            assert self.near_sigma.shape == (K, self.near_t.size) and self.near_w.shape == self.near_t.shape
            assert self.near_m.shape == (K,) and self.near_c.shape == (K,)
            assert self.near_edges.size * self.near_k == self.near_t.size + self.near_k
        if self.ladder_r is not None:
            n = int(np.sum(self.ladder_p))
            assert self.ladder_shat.shape == (n, 3) and self.ladder_T.shape == (n, K)
            assert np.all(np.diff(self.ladder_r) > 0) and self.ladder_r[0] > 2 * self.eps
        return self

    @property
    def ladder_tol(self) -> float:
        """ID tolerance of the ladder rungs (table meta; 0 when unknown)."""
        import re
        m = re.search(r"'ladder_id_tol': ([0-9.eE+-]+)", str(self.meta.get("repr", "")) if self.meta else "")
        return float(m.group(1)) if m else 0.0

    @property
    def ladder_err(self) -> float:
        """The rungs' largest measured relative field error (table meta ``ladder_err``: max over random far-field points
        and random densities relative to the field's max norm, nc_tables.skeleton.outgoing_error); 0 when unknown."""
        import re
        m = re.search(r"'ladder_err': \[([^\]]*)\]", str(self.meta.get("repr", "")) if self.meta else "")
        return max(float(v) for v in m.group(1).split(",")) if m and m.group(1).strip() else 0.0

    def without_ladder(self):
        return PatchTables(self.kind, self.eps, self.M, self.zhat, self.P, self.shat, self.T, self.I, self.meta,
                           res_rhat=self.res_rhat, res_w=self.res_w, res_S=self.res_S, near_edges=self.near_edges,
                           near_t=self.near_t, near_w=self.near_w, near_sigma=self.near_sigma, near_m=self.near_m,
                           near_c=self.near_c, near_k=self.near_k)


_OPTIONAL = ("ladder_r", "ladder_p", "ladder_shat", "ladder_T", "res_rhat", "res_w", "res_S", "near_edges", "near_t",
             "near_w", "near_sigma", "near_m", "near_c", "near_k")


def save_tables(path, t: PatchTables):
    extra = {k: getattr(t, k) for k in _OPTIONAL if getattr(t, k) is not None}
    np.savez(path, version=TABLE_VERSION, kind=t.kind, eps=t.eps, M=t.M, zhat=t.zhat, P=t.P,
             shat=t.shat, T=t.T, I=t.I, meta=np.array(repr(t.meta)), **extra)


def load_tables(path) -> PatchTables:
    z = np.load(path, allow_pickle=False)
    assert int(z["version"]) == TABLE_VERSION, "table file version mismatch"
    lad = {k: np.ascontiguousarray(z[k]) for k in _OPTIONAL if k in z.files}
    if "near_k" in lad:
        lad["near_k"] = int(np.asarray(lad["near_k"]).reshape(-1)[0])
    return PatchTables(kind=int(z["kind"]), eps=float(z["eps"]), M=int(z["M"]),
                       zhat=np.ascontiguousarray(z["zhat"]), P=np.ascontiguousarray(z["P"]),
                       shat=np.ascontiguousarray(z["shat"]), T=np.ascontiguousarray(z["T"]),
                       I=np.ascontiguousarray(z["I"]), meta={"repr": str(z["meta"])}, **lad).validate()


def patch_point(t, theta):
    """Canonical-frame point at arc distance t from the pole in azimuth theta."""
    t = np.asarray(t, dtype=np.float64)
    theta = np.asarray(theta, dtype=np.float64)
    return np.stack([np.sin(t) * np.cos(theta), np.sin(t) * np.sin(theta), np.cos(t)], axis=-1)


def polar_node_grid(eps: float, n_r: int, n_theta: int):
    """Tensor Gauss-Legendre (radius r in [0,1], t = eps*r) x trapezoid (theta) node set.

    Returns (r, theta, xyz) with node index k = i_r * n_theta + i_theta.
    """
    x, _ = np.polynomial.legendre.leggauss(n_r)
    r = 0.5 * (x + 1.0)
    th = 2.0 * np.pi * np.arange(n_theta) / n_theta
    R, TH = np.meshgrid(r, th, indexing="ij")
    xyz = patch_point(eps * R.ravel(), TH.ravel())
    return R.ravel(), TH.ravel(), xyz


def synthetic_tables(kind: int, eps: float, seed: int, M: int = 15, p: int = 120, n_r: int = 16,
                     n_theta: int = 32, coupling: float = 1.0) -> PatchTables:
    """Real node geometry, random operators (parity-only tables)."""
    rng = np.random.default_rng(seed)
    K = (M + 1) * (M + 2) // 2
    _, _, zhat = polar_node_grid(eps, n_r, n_theta)
    # skeleton nodes: random points strictly inside the patch
    t = eps * np.sqrt(rng.random(p)) * 0.999
    th = 2.0 * np.pi * rng.random(p)
    shat = patch_point(t, th)
    Kstar = zhat.shape[0]
    T = rng.standard_normal((p, K)) * (coupling * eps / np.sqrt(K * p))
    P = rng.standard_normal((K, Kstar)) / Kstar
    I = rng.standard_normal(K) * eps
    return PatchTables(kind=kind, eps=eps, M=M, zhat=zhat, P=P, shat=shat, T=T, I=I,
                       meta={"synthetic": True, "seed": seed, "coupling": coupling}).validate()


def synthetic_residual(tab: PatchTables, seed: int, n_r: int = 24, n_theta: int = 33) -> PatchTables:
    """Attach a parity-only residual table to ``tab``: the residual grid geometry (Gauss-Legendre radii x offset
    equispaced angles), its quadrature weights, and a random self-potential matrix."""
    rng = np.random.default_rng(seed)
    x, w = np.polynomial.legendre.leggauss(n_r)
    t = 0.5 * tab.eps * (x + 1.0)
    th = 2.0 * np.pi * (np.arange(n_theta) + 0.5) / n_theta
    T, TH = np.meshgrid(t, th, indexing="ij")
    tab.res_rhat = patch_point(T.ravel(), TH.ravel())
    tab.res_w = ((0.5 * tab.eps * w * np.sin(t))[:, None] * np.full(n_theta, 2.0 * np.pi / n_theta)[None, :]).ravel()
    tab.res_S = rng.standard_normal((n_r * n_theta, tab.K)) / np.sqrt(tab.K)
    return tab.validate()
