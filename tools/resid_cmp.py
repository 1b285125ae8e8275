import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_1906_04209_b200 as nc
from nc_inputs import CONFIGS
from nc_inputs.tables import load_tables
name = sys.argv[1]
cfg = CONFIGS[name]
tab = load_tables(os.path.join(os.environ["ROOT"], "tables", "data", f"{name}.npz"))
modes = [("hier", nc.NC_HIER)] + ([("direct", nc.NC_DIRECT)] if cfg.N <= 10000 else [])
for label, mode in modes:
    h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=mode, precision=cfg.precision)
    xs, its, hist = h.gmres(rtol=cfg.gmres_tol, max_iter=300)
    Is, val = h.flux_or_mfpt(xs)
    pats = np.random.default_rng(123).choice(cfg.N, min(64, cfg.N), replace=False)
    res, _ = h.residual(xs, pats, tab)
    print(json.dumps({"config": name, "mode": label, "nr_margin": os.environ.get("NC_NR_MARGIN", "default"), "its": its,
                      "I_sigma": Is, "res_max": float(np.max(res)), "res_median": float(np.median(res)),
                      "res_mean": float(np.mean(res))}), flush=True)
    h.close()
