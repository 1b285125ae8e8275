"""Thin ctypes binding of libnc (include/nc.h).  Argument marshalling only: every arithmetic step of
the matvec, GMRES and read-out runs in libnc's CUDA kernels.  PyTorch supplies device memory and
streams.  There is no CPU fallback: if libnc.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnc.so")

NC_OK, NC_EINVAL, NC_ESEP, NC_ENOMEM, NC_ECUDA, NC_ENCCL, NC_ESTATE, NC_ENOCONV, NC_EUNSUP = 0, -1, -2, -3, -4, -5, -6, -7, -8
NC_INTERIOR, NC_EXTERIOR = 0, 1
NC_DIRECT, NC_HIER = 0, 1
_ERRNAMES = {-1: "NC_EINVAL", -2: "NC_ESEP", -3: "NC_ENOMEM", -4: "NC_ECUDA", -5: "NC_ENCCL", -6: "NC_ESTATE",
             -7: "NC_ENOCONV", -8: "NC_EUNSUP"}

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class NcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class NcTables(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("K", ctypes.c_int32), ("Kstar", ctypes.c_int32), ("p", ctypes.c_int32),
                ("zhat", _dp), ("P", _dp), ("shat", _dp), ("T", _dp), ("I", _dp),
                ("n_ladder", ctypes.c_int32), ("ladder_r", _dp), ("ladder_p", ctypes.POINTER(ctypes.c_int32)),
                ("ladder_shat", _dp), ("ladder_T", _dp), ("ladder_tol", ctypes.c_double)]


class NcOpts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("precision", ctypes.c_double), ("device", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("check_separation", ctypes.c_int32)]


class NcNearTables(ctypes.Structure):
    _fields_ = [("npan", ctypes.c_int32), ("k", ctypes.c_int32), ("edges", _dp), ("t", _dp), ("w", _dp),
                ("sigma", _dp), ("m", ctypes.POINTER(ctypes.c_int32)), ("c", ctypes.POINTER(ctypes.c_int32))]


class NcStats(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_count", ctypes.c_int64),
                ("K", ctypes.c_int32), ("Kstar", ctypes.c_int32), ("p", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("matvecs", ctypes.c_int64),
                ("pairs_per_matvec", ctypes.c_double), ("gemm_flops_per_matvec", ctypes.c_double),
                ("ms_last", ctypes.c_double * 8), ("tree_levels", ctypes.c_int32), ("tree_groups", ctypes.c_int64),
                ("hier_grid_pairs", ctypes.c_double), ("hier_near_pairs", ctypes.c_double),
                ("hier_interp_terms", ctypes.c_double), ("hier_grid_points", ctypes.c_int64),
                ("hier_grid_units", ctypes.c_int64), ("device_bytes", ctypes.c_double),
                ("launches_per_matvec", ctypes.c_int32), ("gmres_ortho_ms", ctypes.c_double),
                ("gmres_ortho_bytes", ctypes.c_double), ("gmres_ortho_iters", ctypes.c_int64),
                ("pair_fp64_flops_direct", ctypes.c_double), ("pair_fp64_inst_direct", ctypes.c_double),
                ("pair_fp64_flops_grid", ctypes.c_double), ("pair_fp64_inst_grid", ctypes.c_double),
                ("hier_grid_fill", ctypes.c_double), ("hier_grid_warp_fill", ctypes.c_double),
                ("grid_variant", ctypes.c_int32 * 8), ("hier_unit_points", ctypes.c_double),
                ("proxy_n", ctypes.c_int32), ("proxy_kappa", ctypes.c_double), ("proxy_far_frac", ctypes.c_double)]


EXPORTS = ["nc_setup", "nc_partition", "nc_matvec", "nc_matvec_emulated", "nc_matvec_host", "nc_gmres", "nc_flux_or_mfpt",
           "nc_field", "nc_field_near", "nc_residual", "nc_density", "nc_id_sketch", "nc_modal_kernels", "nc_stats",
           "nc_time_stages", "nc_tree_lists", "nc_near_counts", "nc_pair_mix", "nc_split_rows", "nc_proxy_rule", "nc_nccl_unique_id", "nc_destroy", "nc_last_error", "nc_version"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libnc.so (raises if it is missing: the product has no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libnc.so not built at {path}; run `python -m paper_1906_04209_b200.build`")
    L = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    L.nc_setup.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int64, _dp, ctypes.c_double,
                           ctypes.POINTER(NcTables), ctypes.POINTER(NcOpts)]
    L.nc_partition.argtypes = [vp, _i64p, _i64p, _i64p]
    L.nc_matvec.argtypes = [vp, vp, vp, vp]
    L.nc_matvec_emulated.argtypes = [vp, vp, vp, vp]
    L.nc_matvec_host.argtypes = [vp, _dp, _dp]
    L.nc_gmres.argtypes = [vp, vp, ctypes.c_double, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int), _dp, vp]
    L.nc_flux_or_mfpt.argtypes = [vp, vp, _dp, _dp]
    L.nc_field.argtypes = [vp, vp, ctypes.c_int64, _dp, _dp, _dp]
    L.nc_field_near.argtypes = [vp, vp, ctypes.c_int64, _dp, vp, _dp, _dp, _i64p]
    L.nc_residual.argtypes = [vp, vp, ctypes.c_int, _i64p, ctypes.c_int, _dp, _dp, _dp, _dp, _dp]
    L.nc_density.argtypes = [vp, vp, ctypes.c_int, _i64p, ctypes.c_int, _dp, _dp]
    L.nc_modal_kernels.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                   _dp, _dp, _dp]
    L.nc_id_sketch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, _dp, ctypes.c_int64, _dp, ctypes.c_int, _dp,
                               _dp]
    L.nc_stats.argtypes = [vp, ctypes.POINTER(NcStats)]
    L.nc_time_stages.argtypes = [vp, ctypes.c_int]
    L.nc_tree_lists.argtypes = [vp, _i64p, _i64p, _i64p, _i64p, _i64p]
    L.nc_near_counts.argtypes = [vp, _i64p]
    L.nc_pair_mix.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
    L.nc_split_rows.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _i64p, _i64p]
    L.nc_proxy_rule.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                ctypes.c_int, _dp, _dp, _dp, _dp]
    L.nc_nccl_unique_id.argtypes = [vp]
    L.nc_destroy.argtypes = [vp]
    L.nc_destroy.restype = None
    L.nc_last_error.restype = ctypes.c_char_p
    L.nc_version.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("nc_destroy", "nc_last_error", "nc_version"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc):
    if rc != NC_OK:
        raise NcError(rc, load_library().nc_last_error().decode())


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().nc_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def split_rows(N: int, world: int, weights=None):
    """Host-only: the contiguous row partition nc_setup uses -> (begin, count) arrays of length world."""
    L = load_library()
    b = np.zeros(world, dtype=np.int64)
    c = np.zeros(world, dtype=np.int64)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    _check(L.nc_split_rows(w.ctypes.data_as(_dp) if w is not None else None, int(N), int(world),
                           b.ctypes.data_as(_i64p), c.ctypes.data_as(_i64p)))
    return b, c


def proxy_rule(zhat, deg: int = 8, nring: int = 4, cphi: float = 24.0, tol: float = 1e-7):
    """Host-only: the step-4 proxy rule for the nodes zhat (nc_proxy_rule, R36) -> (pts n x 3,
    Int Kstar x n, kappa, h)."""
    L = load_library()
    z = np.ascontiguousarray(zhat, dtype=np.float64)
    ks = z.shape[0]
    nmax = 4096
    pts = np.zeros((nmax, 3))
    Int = np.zeros(ks * nmax)
    kap = ctypes.c_double()
    h = ctypes.c_double()
    n = L.nc_proxy_rule(z.ctypes.data_as(_dp), ks, int(deg), int(nring), float(cphi), float(tol), nmax,
                        pts.ctypes.data_as(_dp), Int.ctypes.data_as(_dp), ctypes.byref(kap), ctypes.byref(h))
    if n < 0:
        _check(n)
    return pts[:n].copy(), Int[:ks * n].reshape(ks, n).copy(), kap.value, h.value


def id_sketch(kind: int, train, fine, omega, device: int = 0) -> np.ndarray:
    """Y = omega @ G(train, fine) on the GPU (nc_id_sketch): the sketch of the Step-1 interpolative decomposition."""
    L = load_library()
    tr = np.ascontiguousarray(train, dtype=np.float64).reshape(-1, 3)
    fi = np.ascontiguousarray(fine, dtype=np.float64).reshape(-1, 3)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    Y = np.empty((om.shape[0], len(fi)))
    _check(L.nc_id_sketch(int(kind), int(device), len(tr), tr.ctypes.data_as(_dp), len(fi), fi.ctypes.data_as(_dp),
                          om.shape[0], om.ctypes.data_as(_dp), Y.ctypes.data_as(_dp)))
    return Y


def modal_kernels(kind: int, t, tp, M: int, phi, wphi, device: int = 0) -> np.ndarray:
    """G_m(t, t') for m = 0..M at paired radii on the GPU (nc_modal_kernels): the one-patch solver's modal kernels."""
    L = load_library()
    t = np.ascontiguousarray(t, dtype=np.float64).ravel()
    tp = np.ascontiguousarray(tp, dtype=np.float64).ravel()
    ph = np.ascontiguousarray(phi, dtype=np.float64)
    wp = np.ascontiguousarray(wphi, dtype=np.float64)
    out = np.empty((t.size, M + 1))
    _check(L.nc_modal_kernels(int(kind), int(device), t.size, t.ctypes.data_as(_dp), tp.ctypes.data_as(_dp), int(M),
                              ph.size, ph.ctypes.data_as(_dp), wp.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
    return out


def pair_mix(kind: int, far: int, ctas_per_sm: int = 2):
    """nc_pair_mix: (best ms, warp-pairs per launch) of the grid kernel's pair evaluation run in isolation."""
    L = load_library()
    ms, wp = ctypes.c_double(), ctypes.c_double()
    _check(L.nc_pair_mix(int(kind), int(far), int(ctas_per_sm), ctypes.byref(ms), ctypes.byref(wp)))
    return ms.value, wp.value


def _ptr(t, shape=None):
    """Device pointer of a contiguous float64 CUDA tensor (of the given shape: libnc trusts the sizes it is passed,
    so an undersized buffer would be read or written out of bounds on the device)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected a tensor of shape {tuple(shape)}, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class Handle:
    """One nc_setup'd layout.  ``tables`` is any object with M, zhat, P, shat, T, I numpy attributes."""

    def __init__(self, kind, centers, eps, tables, mode=NC_DIRECT, precision=1e-9, device=0, world=1, rank=0,
                 nccl_id: bytes | None = None, check_separation=True, use_ladder=True):
        L = load_library()
        self._L = L
        c = np.ascontiguousarray(centers, dtype=np.float64)
        self._keep = [np.ascontiguousarray(getattr(tables, k), dtype=np.float64) for k in ("zhat", "P", "shat", "T", "I")]
        zhat, P, shat, T, I = self._keep
        tab = NcTables(int(tables.M), T.shape[1], zhat.shape[0], shat.shape[0],
                       zhat.ctypes.data_as(_dp), P.ctypes.data_as(_dp), shat.ctypes.data_as(_dp),
                       T.ctypes.data_as(_dp), I.ctypes.data_as(_dp), 0, None, None, None, None, 0.0)
        if use_ladder and getattr(tables, "ladder_r", None) is not None and len(tables.ladder_r) > 0:
            lr = np.ascontiguousarray(tables.ladder_r, dtype=np.float64)
            lp = np.ascontiguousarray(tables.ladder_p, dtype=np.int32)
            ls = np.ascontiguousarray(tables.ladder_shat, dtype=np.float64)
            lt = np.ascontiguousarray(tables.ladder_T, dtype=np.float64)
            self._keep += [lr, lp, ls, lt]
            tab.n_ladder = len(lr)
            tab.ladder_r = lr.ctypes.data_as(_dp)
            tab.ladder_p = lp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            tab.ladder_shat = ls.ctypes.data_as(_dp)
            tab.ladder_T = lt.ctypes.data_as(_dp)
            # the gate of nc_setup: the rungs' ID tolerance (tests/test_parity_golden_gpu.py checks the matvec error
            # with the ladder on at a requested precision equal to it)
            tab.ladder_tol = float(getattr(tables, "ladder_tol", 0.0) or 0.0)
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        opts = NcOpts(int(mode), float(precision), int(device), int(world), int(rank),
                      ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None, int(bool(check_separation)))
        h = ctypes.c_void_p()
        _check(L.nc_setup(ctypes.byref(h), int(kind), len(c), c.ctypes.data_as(_dp), float(eps), ctypes.byref(tab),
                          ctypes.byref(opts)))
        self._h = h
        self.kind, self.N, self.eps, self.mode = int(kind), len(c), float(eps), int(mode)
        self.K, self.Kstar, self.p = T.shape[1], zhat.shape[0], shat.shape[0]
        rb, rc = ctypes.c_int64(), ctypes.c_int64()
        perm = np.empty(self.N, dtype=np.int64)
        _check(L.nc_partition(h, ctypes.byref(rb), ctypes.byref(rc), perm.ctypes.data_as(_i64p)))
        self.row_begin, self.row_count, self.perm = rb.value, rc.value, perm

    # ----------------------------------------------------------------------------------------------
    def to_internal(self, x_caller: np.ndarray) -> np.ndarray:
        """Caller-order (N, K) -> this rank's internal rows."""
        x = np.asarray(x_caller).reshape(self.N, -1)[self.perm]
        return np.ascontiguousarray(x[self.row_begin:self.row_begin + self.row_count])

    def to_caller(self, y_rows_all: np.ndarray) -> np.ndarray:
        """All ranks' internal rows (N, K) -> caller order."""
        out = np.empty_like(y_rows_all)
        out[self.perm] = y_rows_all
        return out

    def matvec(self, x, y=None, stream=None):
        import torch
        if y is None:
            y = torch.empty_like(x)
        rows = (self.row_count, self.K)
        _check(self._L.nc_matvec(self._h, _ptr(x, rows), _ptr(y, rows), _stream_ptr(stream)))
        return y

    def matvec_emulated(self, x_all, y=None, stream=None):
        """Rank emulation (world > 1, no nccl_id): this rank's rows from the full internal-order input."""
        import torch
        if y is None:
            y = torch.empty((self.row_count, x_all.shape[1]), dtype=x_all.dtype, device=x_all.device)
        _check(self._L.nc_matvec_emulated(self._h, _ptr(x_all, (self.N, self.K)), _ptr(y, (self.row_count, self.K)),
                                          _stream_ptr(stream)))
        return y

    def matvec_host(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.row_count, self.K):
            raise ValueError(f"expected shape {(self.row_count, self.K)}, got {x.shape}")
        y = np.empty_like(x)
        _check(self._L.nc_matvec_host(self._h, x.ctypes.data_as(_dp), y.ctypes.data_as(_dp)))
        return y

    def gmres(self, b=None, rtol=1e-10, max_iter=300, x=None, stream=None, allow_noconv=False):
        import torch
        if x is None:
            x = torch.empty((self.row_count, self.K), dtype=torch.float64, device="cuda")
        it = ctypes.c_int()
        hist = np.zeros(max_iter + 1)
        rows = (self.row_count, self.K)
        rc = self._L.nc_gmres(self._h, _ptr(b, rows) if b is not None else None, float(rtol), int(max_iter), _ptr(x, rows),
                              ctypes.byref(it), hist.ctypes.data_as(_dp), _stream_ptr(stream))
        if rc != NC_OK and not (allow_noconv and rc == NC_ENOCONV):
            _check(rc)
        return x, it.value, hist[: it.value + 1]

    def flux_or_mfpt(self, x):
        Is, v = ctypes.c_double(), ctypes.c_double()
        _check(self._L.nc_flux_or_mfpt(self._h, _ptr(x, (self.row_count, self.K)), ctypes.byref(Is), ctypes.byref(v)))
        return Is.value, v.value

    def field(self, x_all, pts):
        """Off-surface potential of the solution at host points ``pts`` (n x 3): v (interior) or u (exterior), and
        each point's distance to the nearest skeleton node (nc_field; ``x_all`` = all patches' coefficients on
        the device, internal order)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out, dmin = np.empty(len(pts)), np.empty(len(pts))
        _check(self._L.nc_field(self._h, _ptr(x_all, (self.N, self.K)), len(pts), pts.ctypes.data_as(_dp), out.ctypes.data_as(_dp),
                                dmin.ctypes.data_as(_dp)))
        return out, dmin

    def field_near(self, x_all, pts, tables, mfpt=False):
        """NEXT-3 at any off-surface point, near the patches included (nc_field_near): the potential v (interior)
        or u (exterior) at host points ``pts`` (n x 3), the patches within 4 eps of a point from their density
        (the tables' near-field arrays, nc_tables/nearfield.py).  Returns (values, mfpt or None, near pairs)."""
        if getattr(tables, "near_sigma", None) is None:
            raise ValueError("the tables carry no near-field table (nc_tables/nearfield.py)")
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        keep = [np.ascontiguousarray(tables.near_edges, dtype=np.float64),
                np.ascontiguousarray(tables.near_t, dtype=np.float64),
                np.ascontiguousarray(tables.near_w, dtype=np.float64),
                np.ascontiguousarray(tables.near_sigma, dtype=np.float64),
                np.ascontiguousarray(tables.near_m, dtype=np.int32), np.ascontiguousarray(tables.near_c, dtype=np.int32)]
        i32 = ctypes.POINTER(ctypes.c_int32)
        nt = NcNearTables(len(keep[0]) - 1, int(tables.near_k), keep[0].ctypes.data_as(_dp), keep[1].ctypes.data_as(_dp),
                          keep[2].ctypes.data_as(_dp), keep[3].ctypes.data_as(_dp), keep[4].ctypes.data_as(i32),
                          keep[5].ctypes.data_as(i32))
        out = np.empty(len(pts))
        mf = np.empty(len(pts)) if mfpt else None
        nn = ctypes.c_int64()
        _check(self._L.nc_field_near(self._h, _ptr(x_all, (self.N, self.K)), len(pts), pts.ctypes.data_as(_dp),
                                     ctypes.byref(nt), out.ctypes.data_as(_dp),
                                     mf.ctypes.data_as(_dp) if mf is not None else None, ctypes.byref(nn)))
        return out, mf, nn.value

    def residual(self, x_all, patches, tables):
        """L2 residual (eq:l2res) on the listed caller patches with the tables' residual grid (nc_residual);
        returns (res per patch, pointwise residual (n, n_res))."""
        if tables.res_S is None:
            raise ValueError("the tables carry no residual grid (nc_tables/residual.py)")
        pat = np.ascontiguousarray(patches, dtype=np.int64).reshape(-1)
        rh = np.ascontiguousarray(tables.res_rhat, dtype=np.float64)
        rw = np.ascontiguousarray(tables.res_w, dtype=np.float64)
        rs = np.ascontiguousarray(tables.res_S, dtype=np.float64)
        res, pw = np.empty(len(pat)), np.empty((len(pat), len(rw)))
        _check(self._L.nc_residual(self._h, _ptr(x_all, (self.N, self.K)), len(pat), pat.ctypes.data_as(_i64p), len(rw),
                                   rh.ctypes.data_as(_dp), rw.ctypes.data_as(_dp), rs.ctypes.data_as(_dp),
                                   res.ctypes.data_as(_dp), pw.ctypes.data_as(_dp)))
        return res, pw

    def density(self, x_all, patches, B):
        """sigma_i = B fhat_i at the fine grid for the listed caller patches (nc_density, eq:recoversig)."""
        pat = np.ascontiguousarray(patches, dtype=np.int64).reshape(-1)
        Bc = np.ascontiguousarray(B, dtype=np.float64)
        sig = np.empty((len(pat), Bc.shape[0]))
        _check(self._L.nc_density(self._h, _ptr(x_all, (self.N, self.K)), len(pat), pat.ctypes.data_as(_i64p), Bc.shape[0],
                                  Bc.ctypes.data_as(_dp), sig.ctypes.data_as(_dp)))
        return sig

    def time_stages(self, enable=True):
        _check(self._L.nc_time_stages(self._h, int(enable)))

    def stats(self) -> dict:
        s = NcStats()
        _check(self._L.nc_stats(self._h, ctypes.byref(s)))
        d = {k: getattr(s, k) for k, _ in NcStats._fields_}
        d["ms_last"] = list(s.ms_last)
        d["grid_variant"] = list(s.grid_variant)
        return d

    def tree_lists(self):
        L = self._L
        ni, nn = ctypes.c_int64(), ctypes.c_int64()
        _check(L.nc_tree_lists(self._h, ctypes.byref(ni), None, ctypes.byref(nn), None, None))
        il = np.empty((ni.value, 3), dtype=np.int64)
        nb = np.empty((nn.value, 3), dtype=np.int64)
        st = self.stats()
        bop = np.empty((st["tree_levels"] + 1, self.N), dtype=np.int64)
        _check(L.nc_tree_lists(self._h, ctypes.byref(ni), il.ctypes.data_as(_i64p), ctypes.byref(nn),
                               nb.ctypes.data_as(_i64p), bop.ctypes.data_as(_i64p)))
        return il, nb, bop

    def near_counts(self) -> np.ndarray:
        """Near-list source patches of each of this rank's rows (internal order; nc_near_counts, NC_HIER)."""
        out = np.empty(self.row_count, dtype=np.int64)
        _check(self._L.nc_near_counts(self._h, out.ctypes.data_as(_i64p)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._L.nc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
