"""CPU oracle for the multiple-scattering matvec, GMRES and read-out -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product path (``paper_1906_04209_b200``) never
does, and this module never imports the product.  It is deliberately plain and slow: numpy for the
library primitives (matmul, dense solve), ``oracle_field.c`` (plain C + OpenMP) for the O(N^2)
Green's-function sum.  Floating point is fp64 throughout.

Steps, in the paper's order and notation (SURVEY.md §8(c) "What it computes"):

1. frames R_i = [e1 e2 c_i] -- "a coordinate system fixed about the centre" (§3);
   the rule is DESIGN.md reading R8 (part of the ABI).
2. global nodes z_{ik} = R_i zhat_k (Zernike sampling nodes, §4) and
   s_{jm} = R_j shat_m (skeleton nodes x^f_{j,pi(m)}, §7).
3. outgoing charges rho_j = T fhat_j  (eq:Tmap; matvec step 1).
4. field u_{ik} = sum_{j != i} sum_m G(z_{ik}, s_{jm}) rho_{jm}  (eq:mssums with eq:outgoingcompressed;
   oracle_field.c).
5. y_i = fhat_i + P u_i  (eq:opinteqnsdisc / eq:sysmatapply; step 5,
   PAPER.md:1404-1408).
6. GMRES on (I + A_off) fhat = P 1, x0 = 0, modified Gram-Schmidt with one
   re-orthogonalisation pass, Givens rotations, no restart (R9).
7. read-out I_sigma = I . sum_i fhat_i (eq:getI); interior
   mu = 1/(3 I_sigma) - 3/5 (eq:mufromsigma2); exterior J = -4 pi I_sigma (R2,
   correcting the 4 pi dropped at PAPER.md:475).

Pins (tests/test_oracle.py): the Green's-function sphere means, the N = 1 identity
(PAPER.md:883), rotation/permutation invariance, the dense-LU solve (a textbook routine), and the
physical single-patch limit once real tables exist.  mfpt_field: Delta v-bar = -1 and its ball averages
(tests/test_mfpt_oracle.py).  matvec vs matvec_uncompressed (tests/test_uncompressed_oracle.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle_field.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", "-o", _LIB_PATH,
                               src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.oracle_field.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ip, ctypes.c_int64, dp, ip, dp, dp]
        L.oracle_field.restype = None
        L.oracle_green_batch.argtypes = [ctypes.c_int, ctypes.c_int64, dp, dp, dp]
        L.oracle_green_batch.restype = None
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_offsurface.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ctypes.c_int64, dp, dp, dp, dp, dp]
        L.oracle_offsurface.restype = None
        L.oracle_green_off_batch.argtypes = [ctypes.c_int, ctypes.c_int64, dp, dp, dp]
        L.oracle_green_off_batch.restype = None
        L.oracle_rings.argtypes = [ctypes.c_int, dp, ctypes.c_int64, dp, ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.oracle_rings.restype = None
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------------------------------------
# Green's function (on-surface), for pins
# ---------------------------------------------------------------------------------------------
def green(kind: int, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(np.broadcast_to(x, np.broadcast(x, y).shape), dtype=np.float64).reshape(-1, 3)
    y = np.ascontiguousarray(np.broadcast_to(y, np.broadcast(x, y).shape), dtype=np.float64).reshape(-1, 3)
    g = np.empty(len(x))
    lib().oracle_green_batch(int(kind), len(x), _dp(x), _dp(y), _dp(g))
    return g


def green_off(kind: int, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Off-surface G(x, x') for |x'| = 1 (eq:Gintoffsurface / eq:Gextoffsurface)."""
    x = np.ascontiguousarray(np.broadcast_to(x, np.broadcast(x, y).shape), dtype=np.float64).reshape(-1, 3)
    y = np.ascontiguousarray(np.broadcast_to(y, np.broadcast(x, y).shape), dtype=np.float64).reshape(-1, 3)
    g = np.empty(len(x))
    lib().oracle_green_off_batch(int(kind), len(x), _dp(x), _dp(y), _dp(g))
    return g


# ---------------------------------------------------------------------------------------------
# Step 1-2: frames and global nodes
# ---------------------------------------------------------------------------------------------
def frames(centers: np.ndarray) -> np.ndarray:
    """R_i = [e1 e2 c_i] (3x3 per patch; columns).  e1 = normalize(xhat - (xhat.c) c), with yhat used
    instead of xhat when |c . xhat| > 0.9; e2 = c x e1 (R8)."""
    c = np.asarray(centers, dtype=np.float64)
    R = np.empty((len(c), 3, 3))
    for i, ci in enumerate(c):
        a = np.array([1.0, 0.0, 0.0]) if abs(ci[0]) <= 0.9 else np.array([0.0, 1.0, 0.0])
        e1 = a - a.dot(ci) * ci
        e1 /= np.linalg.norm(e1)
        e2 = np.cross(ci, e1)
        R[i, :, 0], R[i, :, 1], R[i, :, 2] = e1, e2, ci
    return R


def global_nodes(R: np.ndarray, local: np.ndarray) -> np.ndarray:
    """x_{i,k} = R_i xhat_k  -> array (N, n, 3)."""
    return np.einsum("iab,kb->ika", R, local)


# ---------------------------------------------------------------------------------------------
# Step 3-5: the matvec
# ---------------------------------------------------------------------------------------------
def outgoing(T: np.ndarray, x: np.ndarray) -> np.ndarray:
    """rho_j = T fhat_j for every patch (eq:Tmap)."""
    return x @ T.T


def field(kind, tgt, tpatch, src, spatch, rho):
    tgt = np.ascontiguousarray(tgt, dtype=np.float64).reshape(-1, 3)
    src = np.ascontiguousarray(src, dtype=np.float64).reshape(-1, 3)
    tpatch = np.ascontiguousarray(tpatch, dtype=np.int64)
    spatch = np.ascontiguousarray(spatch, dtype=np.int64)
    rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
    u = np.empty(len(tgt))
    lib().oracle_field(int(kind), len(tgt), _dp(tgt), _ip(tpatch), len(src), _dp(src), _ip(spatch), _dp(rho),
                       _dp(u))
    return u


def offsurface(kind, centers, tab, x, pts, with_absum=False):
    """NEXT-3: the single-layer potential of the solution at off-surface points,
    v(p) = int G_I(p, x') sigma dS (interior, eq:intBVPansatz) or u(p) = int G_E(p, x') sigma dS (exterior,
    eq:urep), each patch's density in its compressed outgoing representation (eq:outgoingcompressed:
    skeleton nodes s_jm = R_j shat_m, charges rho_j = T fhat_j).  Returns (values, min distance to a skeleton node)
    per point.  ``with_absum``: also return sum |G rho| per point (the conditioning scale of the sum)."""
    N = len(centers)
    x = np.asarray(x, dtype=np.float64).reshape(N, -1)
    s = global_nodes(frames(centers), tab.shat).reshape(-1, 3)
    rho = outgoing(tab.T, x).reshape(-1)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out, dmin, absum = np.empty(len(pts)), np.empty(len(pts)), np.empty(len(pts))
    lib().oracle_offsurface(int(kind), len(pts), _dp(pts), len(s), _dp(np.ascontiguousarray(s)),
                            _dp(np.ascontiguousarray(rho)), _dp(out), _dp(dmin), _dp(absum))
    return (out, dmin, absum) if with_absum else (out, dmin)


def residual(kind, centers, tab, x, patches):
    """NEXT-4: the relative L2 residual of the multiple-scattering system on patch i,
    eq:l2res:  (1/|Gamma_i|) || S sigma_i + sum_{j != i} S_ij sigma_j - 1 ||_{L2(Gamma_i)},
    on the residual grid of the tables (independent of the solve's grids):
      S sigma_i at the grid = res_S fhat_i  (the self-patch potential of the basis solutions, nc_tables/residual.py)
      sum_{j != i} S_ij sigma_j = the compressed field of every other patch (steps 2-4 of ``matvec``)
      the norm and |Gamma_i| by the grid's quadrature weights.
    Returns (res per listed patch, pointwise residual (n, n_res))."""
    N = len(centers)
    x = np.asarray(x, dtype=np.float64).reshape(N, -1)
    R = frames(centers)
    s = global_nodes(R, tab.shat).reshape(-1, 3)
    spatch = np.repeat(np.arange(N, dtype=np.int64), tab.shat.shape[0])
    rho = outgoing(tab.T, x).reshape(-1)
    res, pw = [], []
    for i in np.asarray(patches, dtype=np.int64):
        xr = global_nodes(R[[i]], tab.res_rhat)[0]
        u = field(kind, xr, np.full(len(xr), i, dtype=np.int64), s, spatch, rho)
        r = tab.res_S @ x[i] + u - 1.0
        pw.append(r)
        res.append(np.sqrt(np.sum(tab.res_w * r * r)) / np.sum(tab.res_w))
    return np.array(res), np.array(pw)


def density(x, patches, B):
    """sigma_i = B fhat_i (eq:recoversig) for the listed patches: the definition, a matmul."""
    return np.asarray(x, dtype=np.float64)[np.asarray(patches, dtype=np.int64)] @ np.asarray(B, dtype=np.float64).T


# ---------------------------------------------------------------------------------------------
# NEXT-3 near the surface: the density itself, by adaptive quadrature
# ---------------------------------------------------------------------------------------------
def _panel_profiles(tab, xj):
    """Per angular order m: the radial profiles A_m(t), B_m(t) at the table's radial nodes, sigma(t, theta) =
    sum_m A_m(t) cos(m theta) + B_m(t) sin(m theta) = sum_a fhat_a sigma_a(t) ang_a(theta) (eq:recoversig)."""
    M1 = int(np.max(tab.near_m)) + 1
    AB = np.zeros((tab.near_t.size, 2 * M1))
    for a, (m, c) in enumerate(zip(tab.near_m, tab.near_c)):
        AB[:, 2 * m + (0 if c > 0 else 1)] += xj[a] * tab.near_sigma[a]
    return AB, M1


def _interp_profiles(tab, AB, panel, tq, g_only=False):
    """The profiles at radii tq inside one panel: degree-(k-1) polynomial interpolation of the panel's k nodal
    values (numpy Legendre fit through k points = the interpolant); on the last panel the polynomial is
    g = sigma sqrt(eps - t) (sigma has the 1/sqrt(eps - t) edge singularity there), returned as
    g itself when g_only."""
    k, eps = tab.near_k, tab.eps
    sl = slice(panel * k, (panel + 1) * k)
    tn, vals = tab.near_t[sl], AB[sl]
    a, b = tab.near_edges[panel], tab.near_edges[panel + 1]
    last = panel == len(tab.near_edges) - 2
    if last:
        vals = vals * np.sqrt(eps - tn)[:, None]
    out = np.empty((len(tq), AB.shape[1]))
    for c in range(AB.shape[1]):
        out[:, c] = np.polynomial.Legendre.fit(tn, vals[:, c], k - 1, domain=[a, b])(tq)
    if last and not g_only:
        out /= np.sqrt(eps - tq)[:, None]
    return out


def _rings(kind, p, t, AB, M1):
    """int_0^2pi G_off(p, x'(t, theta)) sigma(t, theta) dtheta for each t: trapezoid rule, doubled until converged."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    AB = np.ascontiguousarray(AB, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    prev = None
    n = 64
    while True:
        out, ab = np.empty(len(t)), np.empty(len(t))
        lib().oracle_rings(int(kind), _dp(p), len(t), _dp(t), n, M1, _dp(AB), _dp(out), _dp(ab))
        # converged: the doubled rule changes each ring integral by less than rounding of its terms' sum
        if prev is not None and np.all(np.abs(out - prev) <= 1e-15 * np.maximum(np.abs(out), 1e-300) + 1e-15 * ab):
            return out
        if n >= 524288:
            raise RuntimeError("oracle ring integral did not converge")
        prev, n = out, 2 * n


def near_patch(kind, tab, xj, p_local, rtol=1e-14):
    """The potential of ONE patch's density at p_local (the patch's canonical frame), by adaptive quadrature of
    int_Gamma G_off(p, x') sigma(x') dS = int_0^eps sin t int_0^2pi G_off sigma dtheta dt (eq:intBVPansatz /
    eq:urep restricted to one patch, sigma = B fhat by eq:recoversig).  Radial: on every panel of the one-patch
    grid, 20-point Gauss-Legendre on the panel compared with the sum over its halves, bisected until they agree
    (the last panel in s = sqrt(eps - t), where sigma ds is smooth); angular: the converged trapezoid rule."""
    AB, M1 = _panel_profiles(tab, np.asarray(xj, dtype=np.float64))
    eps = tab.eps
    xg, wg = np.polynomial.legendre.leggauss(20)
    npan = len(tab.near_edges) - 1

    def F(panel, tq, g_only=False):                    # sin t x ring integral at radii tq of a panel
        return np.sin(tq) * _rings(kind, p_local, tq, _interp_profiles(tab, AB, panel, tq, g_only), M1)

    def gl(panel, a, b, last):
        if last:   # t = eps - s^2, dt = 2 s ds, sigma = g / s: the integrand in s is 2 sin t ring(g), smooth
            s = 0.5 * (a + b) + 0.5 * (b - a) * xg
            return 0.5 * (b - a) * np.sum(wg * 2.0 * F(panel, eps - s * s, g_only=True))
        tq = 0.5 * (a + b) + 0.5 * (b - a) * xg
        return 0.5 * (b - a) * np.sum(wg * F(panel, tq))

    # scale of the patch's potential (native nodes): the adaptive criterion is absolute relative to it
    scale = np.sum(np.abs(tab.near_w * _rings(kind, p_local, tab.near_t, AB, M1)))
    total = 0.0
    for panel in range(npan):
        a, b = tab.near_edges[panel], tab.near_edges[panel + 1]
        last = panel == npan - 1
        if last:
            a, b = 0.0, np.sqrt(eps - a)
        stack = [(a, b, gl(panel, a, b, last), 0)]
        while stack:
            lo, hi, whole, depth = stack.pop()
            mid = 0.5 * (lo + hi)
            left, right = gl(panel, lo, mid, last), gl(panel, mid, hi, last)
            if abs(left + right - whole) <= rtol * scale or depth >= 40:
                total += left + right
            else:
                stack += [(lo, mid, left, depth + 1), (mid, hi, right, depth + 1)]
    return total


def nearfield(kind, centers, tab, x, pts, near_r=4.0):
    """NEXT-3 at any off-surface point (PAPER.md:2069-2097 plot the MFPT at radius 1 - eps/5): v(p) (interior) or
    u(p) (exterior) = sum over patches j of the patch's single-layer potential, by near_patch (the density itself,
    eq:recoversig) for patches whose centre is closer than near_r eps to p, and by the compressed skeleton
    (eq:outgoingcompressed, valid >= 3 eps from every skeleton node, R27) for the others."""
    N = len(centers)
    x = np.asarray(x, dtype=np.float64).reshape(N, -1)
    c = np.asarray(centers, dtype=np.float64)
    R = frames(c)
    s = global_nodes(R, tab.shat)                                     # (N, p, 3)
    rho = outgoing(tab.T, x)                                          # (N, p)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(pts))
    for i, p in enumerate(pts):
        near = np.where(np.linalg.norm(c - p, axis=1) < near_r * tab.eps)[0]
        far = np.setdiff1d(np.arange(N), near)
        v = 0.0
        if len(far):
            sf = np.ascontiguousarray(s[far].reshape(-1, 3))
            rf = np.ascontiguousarray(rho[far].reshape(-1))
            o, dm, ab = np.empty(1), np.empty(1), np.empty(1)
            lib().oracle_offsurface(int(kind), 1, _dp(np.ascontiguousarray(p[None])), len(sf), _dp(sf), _dp(rf),
                                    _dp(o), _dp(dm), _dp(ab))
            v += o[0]
        for j in near:
            v += near_patch(kind, tab, x[j], R[j].T @ p)
        out[i] = v
    return out


def mfpt_field(v, pts, I_sigma):
    """Interior MFPT at a point from the potential v (eq:vtilde, with D = -I_sigma from the lemma
    at PAPER.md:556-566): vbar = (v - 1) / (3 D) + (1 - |x|^2) / 6."""
    r2 = np.sum(np.asarray(pts, dtype=np.float64).reshape(-1, 3) ** 2, axis=1)
    return (np.asarray(v) - 1.0) / (3.0 * (-I_sigma)) + (1.0 - r2) / 6.0


def matvec(kind, centers, tab, x, rows=None, R=None):
    """y = (I + A_off) x  (eq:sysmatapply).  ``rows``: optional subset of target patches (sampled rows);
    returns y for those rows only.  ``R``: optional explicit frames (default: the ABI rule)."""
    N = len(centers)
    x = np.asarray(x, dtype=np.float64).reshape(N, -1)
    R = frames(centers) if R is None else R
    rows = np.arange(N) if rows is None else np.asarray(rows, dtype=np.int64)
    z = global_nodes(R[rows], tab.zhat)                      # (nr, K*, 3)
    s = global_nodes(R, tab.shat)                            # (N, p, 3)
    rho = outgoing(tab.T, x)                                 # (N, p)
    tpatch = np.repeat(rows, tab.Kstar)
    spatch = np.repeat(np.arange(N), tab.p)
    u = field(kind, z, tpatch, s, spatch, rho).reshape(len(rows), tab.Kstar)
    return x[rows] + u @ tab.P.T


def matvec_uncompressed(kind, centers, tab, fine, wf, B, x, rows=None):
    """the same matvec with every source patch's density in its UNcompressed form,
    u_{ik} = sum_{j != i} sum_l G(z_{ik}, f_{jl}) w_l (B fhat_j)_l  (the left side of eq:outgoingcompressed,
    PAPER.md:1082-1093, with sigma_j = B fhat_j, eq:recoversig PAPER.md:797-807, on the one-patch solver's fine grid
    f_l, w_l).  fine (n_f x 3, canonical frame), wf (n_f), B (n_f x K) come from the Step-1 builder; y = x + P u."""
    N = len(centers)
    x = np.asarray(x, dtype=np.float64).reshape(N, -1)
    R = frames(centers)
    rows = np.arange(N) if rows is None else np.asarray(rows, dtype=np.int64)
    z = global_nodes(R[rows], tab.zhat)
    f = global_nodes(R, np.asarray(fine, dtype=np.float64))       # (N, n_f, 3)
    q = (x @ np.asarray(B, dtype=np.float64).T) * np.asarray(wf)[None, :]   # charges w_l sigma_jl
    tpatch = np.repeat(rows, tab.Kstar)
    spatch = np.repeat(np.arange(N), f.shape[1])
    u = field(kind, z, tpatch, f, spatch, q).reshape(len(rows), tab.Kstar)
    return x[rows] + u @ tab.P.T


def rhs(tab, N):
    """b_i = P 1 (eq:opinteqnsdisc right-hand side)."""
    return np.tile(tab.P @ np.ones(tab.Kstar), (N, 1))


# ---------------------------------------------------------------------------------------------
# Step 6: GMRES
# ---------------------------------------------------------------------------------------------
def gmres(apply, b, tol=1e-10, max_iter=300):
    """Unrestarted GMRES, x0 = 0, MGS + one re-orthogonalisation pass, Givens rotations.

    Returns (x, iterations, history) where history[j] = implicit relative residual after j steps."""
    b = np.asarray(b, dtype=np.float64).ravel()
    n = b.size
    beta = np.linalg.norm(b)
    hist = [1.0]
    if beta == 0.0:
        return np.zeros(n), 0, hist
    V = np.zeros((max_iter + 1, n))
    H = np.zeros((max_iter + 1, max_iter))
    cs = np.zeros(max_iter)
    sn = np.zeros(max_iter)
    g = np.zeros(max_iter + 1)
    g[0] = beta
    V[0] = b / beta
    k = 0
    for j in range(max_iter):
        w = np.asarray(apply(V[j]), dtype=np.float64).ravel()
        for _ in range(2):                                   # MGS + one re-orthogonalisation pass
            for i in range(j + 1):
                h = V[i] @ w
                H[i, j] += h
                w = w - h * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        if H[j + 1, j] > 0:
            V[j + 1] = w / H[j + 1, j]
        for i in range(j):                                   # apply previous rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        r = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / r, H[j + 1, j] / r
        H[j, j] = r
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        hist.append(abs(g[j + 1]) / beta)
        if hist[-1] <= tol:
            break
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):                            # back substitution
        y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    x = V[:k].T @ y
    return x, k, hist


# ---------------------------------------------------------------------------------------------
# Step 7: read-out
# ---------------------------------------------------------------------------------------------
def readout(kind, I_row, x):
    """Returns (I_sigma, value): value = mu (interior) or J (exterior)."""
    xs = np.asarray(x, dtype=np.float64).reshape(-1, len(I_row))
    I_sigma = float(I_row @ xs.sum(axis=0))
    if kind == 0:
        return I_sigma, 1.0 / (3.0 * I_sigma) - 3.0 / 5.0
    return I_sigma, -4.0 * np.pi * I_sigma


def solve(kind, centers, tab, tol=1e-10, max_iter=300):
    N = len(centers)
    b = rhs(tab, N)
    x, it, hist = gmres(lambda v: matvec(kind, centers, tab, v.reshape(N, -1)).ravel(), b.ravel(), tol, max_iter)
    I_sigma, value = readout(kind, tab.I, x)
    xr = x.reshape(N, -1)
    res = np.linalg.norm(b - matvec(kind, centers, tab, xr)) / np.linalg.norm(b)
    return dict(x=xr, iters=it, hist=hist, I_sigma=I_sigma, value=value, explicit_residual=res)


def dense_operator(kind, centers, tab):
    """Assemble (I + A_off) column by column (tiny N only)."""
    N = len(centers)
    n = N * tab.K
    A = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        A[:, c] = matvec(kind, centers, tab, e.reshape(N, -1)).ravel()
    return A
