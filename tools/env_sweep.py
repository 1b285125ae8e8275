"""Tuning sweep: hierarchical-vs-direct matvec error (C3, C4: full vectors, GPU direct), the difference from the first
setting, and the matvec / step-4 time, for a list of environment settings; one JSON line per (config, setting).
Default settings: the step-4 proxy rules (R36).

    NC_TUNING=1 python tools/env_sweep.py [--settings '[["label", {"NC_X": "v"}], ...]'] [configs...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS, random_coeffs  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402

assert os.environ.get("NC_TUNING") == "1"
SETTINGS = [("off", {"NC_PROXY": "0"}), ("11,6,24/0.01", {}), ("11,6,24/0.1", {"NC_PROXY_TOL": "0.1"}),
            ("10,5,29/0.01", {"NC_PROXY_RULE": "10,5,29"}), ("9,6,24/0.01", {"NC_PROXY_RULE": "9,6,24"}),
            ("8,4,24/0.01", {"NC_PROXY_RULE": "8,4,24"}), ("8,4,24/0.1", {"NC_PROXY_RULE": "8,4,24", "NC_PROXY_TOL": "0.1"})]
args = sys.argv[1:]
if args and args[0] == "--settings":
    SETTINGS = [tuple(e) for e in json.loads(args[1])]
    args = args[2:]
KEYS = sorted({k for _, env in SETTINGS for k in env})


def timed(h, xi, reps=5):
    h.time_stages(True)
    h.matvec(xi)
    torch.cuda.synchronize()
    rest, tot = [], []
    for _ in range(reps):
        h.matvec(xi)
        torch.cuda.synchronize()
        st = h.stats()
        rest.append(st["ms_last"][5])
        tot.append(st["ms_last"][6])
    h.time_stages(False)
    return float(np.median(rest)), float(np.median(tot))


for name in args or ["C3", "C4", "C5"]:
    cfg = CONFIGS[name]
    tab = load_tables(f"tables/data/{name}.npz")
    c = cfg.centers()
    x = random_coeffs(cfg.N, tab.K, 7)
    yd = None
    if cfg.N <= 20000:
        hd = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
        yd = hd.to_caller(hd.matvec(torch.from_numpy(hd.to_internal(x)).cuda()).cpu().numpy())
        hd.close()
    yoff = None
    for label, env in SETTINGS:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        hh = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=1e-9)
        xi = torch.from_numpy(hh.to_internal(x)).cuda()
        y = hh.to_caller(hh.matvec(xi).cpu().numpy())
        rest, tot = timed(hh, xi)
        st = hh.stats()
        if yoff is None:
            yoff = y
        rec = {"config": name, "setting": label, "proxy_n": st["proxy_n"], "kappa": st["proxy_kappa"],
               "far_frac": st["proxy_far_frac"], "hier_rest_ms": rest, "total_ms": tot,
               "grid_pairs": st["hier_grid_pairs"], "near_pairs": st["hier_near_pairs"], "grid_ms": st["ms_last"][4],
               "rel_vs_first": float(np.linalg.norm(y - yoff) / np.linalg.norm(yoff))}
        if yd is not None:
            rec["rel_err_vs_direct"] = float(np.linalg.norm(y - yd) / np.linalg.norm(yd))
        print(json.dumps(rec), flush=True)
        hh.close()
