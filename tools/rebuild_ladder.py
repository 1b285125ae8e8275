"""Rebuild only the per-level outgoing ladder (R22) of committed table files, keeping
every other array bit for bit (base T, P, zhat, I, residual grid).  Each rung takes the loosest ID tolerance of TOLS
whose MEASURED field error is <= the target (default use: 8e-10, below the default precision 1e-9 the ladder must
serve); one sketch and one pivoted QR per rung serve every candidate tolerance.

    python tools/rebuild_ladder.py 8e-10 [--gpu-sketch] [tables/data/C*.npz ...]

The rungs' measured field errors (nc_tables.skeleton.outgoing_error, max over random far-field points and random
densities relative to the field's max norm) are written to the table meta as ``ladder_err``; a hierarchical handle
uses the ladder only when the requested precision is >= max(ladder_err) (nc.py -> nc_tables.ladder_tol).
"""
from __future__ import annotations

import glob
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from nc_tables.onepatch import fine_grid, solve_onepatch  # noqa: E402
import scipy.linalg as sla  # noqa: E402

from nc_tables.skeleton import outgoing_error, test_matrix, training_grid  # noqa: E402


def qr_of_sketch(kind, train, fine, sketch=None, oversample=400, seed=0, chunk=512):
    """Column-pivoted QR of the Gaussian sketch Y = Omega G(train, fine), exactly as interp_decomp forms it."""
    l = min(oversample, train.shape[0])
    if sketch is not None:
        Y = sketch(kind, train, fine, test_matrix(train.shape[0], oversample, seed, chunk))
    else:
        from nc_tables.kernel import green_xyz
        rng = np.random.default_rng(seed)
        Y = np.zeros((l, fine.shape[0]))
        for a in range(0, train.shape[0], chunk):
            b = min(train.shape[0], a + chunk)
            Y += rng.standard_normal((l, b - a)) @ green_xyz(kind, train[a:b, None, :], fine[None, :, :])
    return sla.qr(Y, mode="economic", pivoting=True)


def rebuild(path, tols, target, gpu_sketch=False):
    d = dict(np.load(path, allow_pickle=False))
    meta = eval(str(d["meta"]), {"__builtins__": {}})
    kind, eps = int(d["kind"]), float(d["eps"])
    sk, mf = None, None
    if gpu_sketch:
        import paper_1906_04209_b200 as ncgpu
        from nc_tables.kernel import modal_gpu
        sk, mf = ncgpu.id_sketch, modal_gpu
    t0 = time.time()
    op = solve_onepatch(kind, eps, int(d["M"]), meta["npan"], meta["k"], meta["n_theta"], modal_fn=mf)
    fine, wf, B = fine_grid(op)
    ratio = meta["ladder_ratio"]
    inners = [r / eps for r in meta["ladder_r"]]
    assert np.allclose(inners, 2.0 * ratio ** np.arange(1, len(inners) + 1))

    def one_rung(inner):
        """The loosest ID tolerance in `tols` whose measured field error is <= target (one sketch, one QR)."""
        train = training_grid(eps, inner=inner)
        Q, R, piv = qr_of_sketch(kind, train, fine, sk)
        d = np.abs(np.diag(R))
        best = None
        for t in tols:
            p = int(np.sum(d > t * d[0]))
            Pi = np.zeros((p, fine.shape[0]))
            Pi[:, piv[:p]] = np.eye(p)
            Pi[:, piv[p:]] = sla.solve_triangular(R[:p, :p], R[:p, p:])
            Tk = Pi @ (wf[:, None] * B)
            err = outgoing_error(kind, fine, wf, B, fine[piv[:p]], Tk, eps, inner=inner)
            best = (piv[:p], Tk, err, t)
            if err <= target:
                break
        return best

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(one_rung, inners))
    d["ladder_p"] = np.array([len(J) for J, _, _, _ in res], dtype=np.int32)
    d["ladder_shat"] = np.concatenate([fine[J] for J, _, _, _ in res])
    d["ladder_T"] = np.concatenate([T for _, T, _, _ in res])
    meta["ladder_id_tol"] = max(t for _, _, _, t in res)
    meta["ladder_id_tols"] = [float(t) for _, _, _, t in res]
    meta["ladder_err_target"] = target
    meta["ladder_p"] = [int(v) for v in d["ladder_p"]]
    meta["ladder_err"] = [float(e) for _, _, e, _ in res]
    meta["t_ladder_s"] = time.time() - t0
    d["meta"] = np.array(repr(meta))
    np.savez(path, **d)
    print(f"{path}: tols {meta['ladder_id_tols']}, sum p_k {int(d['ladder_p'].sum())}, "
          f"max err {max(meta['ladder_err']):.3g}, {time.time() - t0:.1f} s", flush=True)


TOLS = (3e-10, 2.5e-10, 2e-10, 1.5e-10, 1.2e-10, 1e-10, 8e-11, 6e-11, 4e-11)


def main():
    target = float(sys.argv[1])
    gpu = "--gpu-sketch" in sys.argv
    paths = [a for a in sys.argv[2:] if a.endswith(".npz")] or sorted(glob.glob(os.path.join(ROOT, "tables", "data",
                                                                                             "C*.npz")))
    for p in paths:
        rebuild(p, TOLS, target, gpu)


if __name__ == "__main__":
    main()
