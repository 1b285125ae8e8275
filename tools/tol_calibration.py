"""Calibrate the incoming-grid tolerance factor (R21) against the matvec error (GPU box).

    python tools/tol_calibration.py C3 300 1000 3000
    NC_GRID_VARIANT=2,4,0,256,1 python tools/tol_calibration.py C5 300 1000

Reference: the direct sum on the GPU (already oracle-verified to 1e-12) for N <= 10^4; for C5 (direct too slow) the
hierarchical matvec at tolerance factor 0.3 (measured 1e-14 level at C3).  Two inputs: a random x and the physical
right-hand side P.1.  One JSON line per factor: relative l2 errors, grid pairs, k_pairs_grid and matvec ms.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS, random_coeffs  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402


def run(h, xs):
    out, g, t = [], [], []
    for x in xs:
        xi = torch.from_numpy(h.to_internal(x)).cuda()
        h.matvec(xi)
        h.time_stages(True)
        y = h.matvec(xi)
        st = h.stats()
        h.time_stages(False)
        g.append(st["ms_last"][4] if h.mode == nc.NC_HIER else st["ms_last"][2])
        t.append(st["ms_last"][6])
        out.append(h.to_caller(y.cpu().numpy()))
    return out, st, float(np.mean(g)), float(np.mean(t))


def main():
    name = sys.argv[1]
    facs = [float(v) for v in sys.argv[2:]] or [300.0]
    cfg = CONFIGS[name]
    tab = load_tables(os.environ.get("NC_TABLES_FILE") or
                      os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tables", "data",
                                   f"{name}.npz"))
    c = cfg.centers()
    xs = [random_coeffs(cfg.N, tab.K, 7), np.tile(tab.P @ np.ones(tab.Kstar), (cfg.N, 1))]
    if cfg.N <= 10000:
        href = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
        ref_kind = "direct"
    else:
        os.environ["NC_TUNING"] = "1"
        os.environ["NC_GRID_TOL_FACTOR"] = "0.3"
        href = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
        ref_kind = "hier tol factor 0.3"
    refs, _, _, _ = run(href, xs)
    href.close()
    for f in facs:
        os.environ["NC_GRID_TOL_FACTOR"] = repr(f)
        h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
        ys, st, gms, tms = run(h, xs)
        errs = [float(np.linalg.norm(y - r) / np.linalg.norm(r)) for y, r in zip(ys, refs)]
        print(json.dumps({"config": name, "precision": cfg.precision, "tol_factor": f, "reference": ref_kind,
                          "variant": os.environ.get("NC_GRID_VARIANT", "default"), "rel_err_random": errs[0],
                          "rel_err_P1": errs[1], "grid_pairs": st["hier_grid_pairs"],
                          "near_pairs": st["hier_near_pairs"], "interp_terms": st["hier_interp_terms"],
                          "grid_ms": gms, "matvec_ms": tms}), flush=True)
        h.close()


if __name__ == "__main__":
    main()
