"""Every BASELINE.json config on one GPU: matvec time (CUDA events, 3 warm-up + 5 timed), GMRES time to solution,
iterations, J / mu, and the L2 residual (eq:l2res) on up to 16 patches.   python tools/all_configs.py > out.jsonl"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS, random_coeffs  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402

runs = [("C1", nc.NC_DIRECT), ("C2", nc.NC_DIRECT), ("C2", nc.NC_HIER), ("C3", nc.NC_HIER), ("C4", nc.NC_HIER),
        ("C5", nc.NC_HIER)]
for name, mode in runs:
    cfg = CONFIGS[name]
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    t0 = time.perf_counter()
    h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=mode, precision=cfg.precision)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = torch.from_numpy(h.to_internal(random_coeffs(cfg.N, tab.K, 2000 + int(name[1:])))).cuda()
    y = torch.empty_like(x)
    for _ in range(3):
        h.matvec(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        h.matvec(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    t0 = time.perf_counter()
    xs, its, hist = h.gmres(rtol=cfg.gmres_tol, max_iter=300)
    Is, val = h.flux_or_mfpt(xs)
    tts = time.perf_counter() - t0
    pats = np.random.default_rng(9).choice(cfg.N, min(16, cfg.N), replace=False)
    res, _ = h.residual(xs, pats, tab)
    st = h.stats()
    print(json.dumps({"config": name, "mode": "direct" if mode == nc.NC_DIRECT else "hier", "N": cfg.N, "eps": cfg.eps,
                      "kind": cfg.kind, "matvec_ms": ms, "matvec_per_s": 1e3 / ms, "pairs_per_matvec": st["pairs_per_matvec"],
                      "gmres_iters": its, "time_to_solution_s": tts, "setup_s": setup, "I_sigma": Is,
                      ("mu" if cfg.kind == 0 else "J"): val, "residual_max": float(np.max(res)),
                      "residual_median": float(np.median(res))}), flush=True)
    h.close()
