"""Step-1 precomputation: build the patch-operator tables for one (kind, eps).

    python -m nc_tables.build --kind 0 --eps 0.003 --out tables/data/C5.npz
    python -m nc_tables.build --configs [--gpu-sketch]   # the five BASELINE.json configs (K* = 248, residual grids)

CPU, untimed, N-independent; its output file is the `nc_tables` input of nc_setup (include/nc.h) and of the
oracle.  Neither the oracle nor the CUDA path imports this package.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import zernike
from .onepatch import fine_grid, solve_onepatch
from .skeleton import interp_decomp, outgoing_error, training_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_tables(kind: int, eps: float, M: int = 15, npan: int = 13, k: int = 20, n_theta: int = 64,
                 id_tol: float = 1e-11, zn_r: int | None = None, zn_theta: int | None = None, verbose=False,
                 ladder: bool = True, ladder_max: float = 1.2, ladder_ratio: float = 2.0 ** (1.0 / 3.0),
                 ladder_id_tol: float | None = 3e-10, gpu_sketch: bool = False, zn_radial: str = "r2"):
    """gpu_sketch: form the ID sketches on the GPU (nc_id_sketch, NEXT-1) instead of numpy.  zn_radial: the Zernike
    sampling rule, "r2" (default: 8 Gauss nodes in r^2 x 31 angles, K* = 248, R7) or "r" (16 x 32 = 512)."""
    sk, mf = None, None
    if gpu_sketch:   # the GPU parts of Step 1 (NEXT-1): ID sketches and the one-patch solver's modal kernels
        import paper_1906_04209_b200 as ncgpu
        from .kernel import modal_gpu
        sk, mf = ncgpu.id_sketch, modal_gpu
    t0 = time.time()
    op = solve_onepatch(kind, eps, M, npan, k, n_theta, modal_fn=mf)
    t1 = time.time()
    fine, wf, B = fine_grid(op)
    train = training_grid(eps)
    J, Pi = interp_decomp(kind, train, fine, id_tol, sketch=sk)
    T = Pi @ (wf[:, None] * B)
    shat = fine[J]
    t2 = time.time()
    r, th, P = zernike.transform(M, zn_r, zn_theta, zn_radial)
    zhat = zernike.patch_xyz(eps, r, th)
    I = wf @ B
    err = outgoing_error(kind, fine, wf, B, shat, T, eps)
    # per-level recompression ("one matrix T per level"): a ladder of far-field regions
    # {arc > r_k}, r_k = 2 eps ladder_ratio^k (default 2^(1/3)), each with its own ID against a training grid on that
    # region at the ladder tolerance (default 3e-10: SURVEY.md A10 suggests 1e-10; 3e-10 measured to leave the matvec error
    # unchanged, R22; the base T keeps id_tol)
    lad_r, lad_p, lad_s, lad_T, lad_err = [], [], [], [], []
    if ladder:
        rung = 1
        inners = []
        while 2.0 * eps * ladder_ratio ** rung < ladder_max:
            inners.append(2.0 * ladder_ratio ** rung)
            rung += 1

        def one_rung(inner):
            Jk, Pik = interp_decomp(kind, training_grid(eps, inner=inner), fine, ladder_id_tol or id_tol, sketch=sk)
            Tk = Pik @ (wf[:, None] * B)
            return Jk, Tk, outgoing_error(kind, fine, wf, B, fine[Jk], Tk, eps, inner=inner)

        if sk is not None:   # GPU sketches: the host QRs of the rungs run concurrently (LAPACK releases the GIL)
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
                results = list(ex.map(one_rung, inners))
        else:
            results = [one_rung(inner) for inner in inners]
        for inner, (Jk, Tk, ek) in zip(inners, results):
            lad_r.append(inner * eps)
            lad_p.append(len(Jk))
            lad_s.append(fine[Jk])
            lad_T.append(Tk)
            lad_err.append(ek)
    t3 = time.time()
    meta = dict(kind=kind, eps=eps, M=M, npan=npan, k=k, n_theta=n_theta, id_tol=id_tol, p=len(J), n_f=len(wf),
                zn_radial=zn_radial, Kstar=len(r),
                ladder_ratio=ladder_ratio, ladder_id_tol=ladder_id_tol or id_tol,
                n_train=len(train), outgoing_rel_err=err, t_onepatch_s=t1 - t0, t_id_s=t2 - t1,
                ladder_r=lad_r, ladder_p=lad_p, ladder_err=lad_err, t_ladder_s=t3 - t2)
    if verbose:
        print(meta, file=sys.stderr)
    out = dict(kind=kind, eps=eps, M=M, zhat=zhat, P=P, shat=shat, T=T, I=I, meta=meta)
    if lad_r:
        out.update(ladder_r=np.array(lad_r), ladder_p=np.array(lad_p, dtype=np.int32),
                   ladder_shat=np.concatenate(lad_s), ladder_T=np.concatenate(lad_T))
    return out


def save(d, path):
    extra = {k: d[k] for k in ("ladder_r", "ladder_p", "ladder_shat", "ladder_T") if k in d}
    np.savez(path, version=1, kind=d["kind"], eps=d["eps"], M=d["M"], zhat=d["zhat"], P=d["P"], shat=d["shat"],
             T=d["T"], I=d["I"], meta=np.array(repr(d["meta"])), **extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--eps", type=float, default=0.1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", action="store_true")
    ap.add_argument("--id-tol", type=float, default=1e-11)
    ap.add_argument("--ladder-ratio", type=float, default=2.0 ** (1.0 / 3.0))
    ap.add_argument("--ladder-id-tol", type=float, default=3e-10)
    ap.add_argument("--radial", default="r2", choices=["r2", "r"])
    ap.add_argument("--gpu-sketch", action="store_true")
    a = ap.parse_args()
    from .residual import add_to_tables
    outdir = os.path.join(ROOT, "tables", "data")
    os.makedirs(outdir, exist_ok=True)
    if a.configs:
        sys.path.insert(0, ROOT)
        from nc_inputs import CONFIGS
        for name, cfg in CONFIGS.items():
            d = build_tables(cfg.kind, cfg.eps, id_tol=a.id_tol, verbose=True, ladder_ratio=a.ladder_ratio,
                             ladder_id_tol=a.ladder_id_tol, gpu_sketch=a.gpu_sketch, zn_radial=a.radial)
            save(d, os.path.join(outdir, f"{name}.npz"))
            add_to_tables(os.path.join(outdir, f"{name}.npz"))
        return
    d = build_tables(a.kind, a.eps, id_tol=a.id_tol, verbose=True, ladder_ratio=a.ladder_ratio,
                     ladder_id_tol=a.ladder_id_tol, gpu_sketch=a.gpu_sketch, zn_radial=a.radial)
    path = a.out or os.path.join(outdir, f"k{a.kind}_eps{a.eps:g}.npz")
    save(d, path)
    add_to_tables(path)


if __name__ == "__main__":
    main()
