"""K* = 248 (8 Gauss nodes in r^2 x 31 angles) vs the tables' K* = 512 (16 x 32): tables built with
GPU sketches into a scratch dir, then per config the solved J / mu, GMRES iterations, the L2 residual diagnostic
(eq:l2res, NEXT-4) on random patches and the matvec time.   python tools/kstar_probe.py C1 C2 C3 C5"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402
from nc_tables.build import build_tables, save  # noqa: E402
from nc_tables.residual import add_to_tables  # noqa: E402

out_dir = "/tmp/kstar248"
os.makedirs(out_dir, exist_ok=True)
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    path = os.path.join(out_dir, f"{name}.npz")
    t0 = time.time()
    save(build_tables(cfg.kind, cfg.eps, gpu_sketch=True, zn_radial="r2"), path)
    add_to_tables(path)
    tb = time.time() - t0
    mode = nc.NC_DIRECT if name in ("C1", "C2") else nc.NC_HIER
    for label, tpath in (("512", os.path.join(ROOT, "tables", "data", f"{name}.npz")), ("248", path)):
        tab = load_tables(tpath)
        h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=mode, precision=cfg.precision)
        x = torch.randn(h.to_internal(np.zeros((cfg.N, tab.K))).shape, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(2):
            h.matvec(x, y)
        torch.cuda.synchronize()
        t1 = time.time()
        for _ in range(3):
            h.matvec(x, y)
        torch.cuda.synchronize()
        mv = (time.time() - t1) / 3
        t1 = time.time()
        xs, its, hist = h.gmres(rtol=cfg.gmres_tol, max_iter=300)
        Is, val = h.flux_or_mfpt(xs)
        tts = time.time() - t1
        pats = np.random.default_rng(5).choice(cfg.N, min(32, cfg.N), replace=False)
        res, _ = h.residual(xs, pats, tab)
        print(json.dumps({"config": name, "Kstar": tab.Kstar, "mode": "direct" if mode == nc.NC_DIRECT else "hier",
                          "matvec_ms": mv * 1e3, "gmres_iters": its, "tts_s": tts, "I_sigma": Is,
                          ("mu" if cfg.kind == 0 else "J"): val, "res_max": float(np.max(res)),
                          "res_median": float(np.median(res)), "table_build_s": tb if label == "248" else None}),
              flush=True)
        h.close()
