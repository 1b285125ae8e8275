"""Sweep the k_pairs_grid variants (NC_GRID_VARIANT="TPT,UNROLL,LOG8,STAGE") on one config (GPU box).

    python tools/sweep_grid.py C5 "128,2,4,256,1" "NC_INTERP_VARIANT=256,2,4" "NC_COST_NEAR=1.3;NC_COST_INTERP=0.15" ...

Each variant runs in its own process (the variant is read once per process); prints one JSON line per variant with
the per-matvec k_pairs_grid time (library CUDA events), the whole matvec time, and the relative difference of the
output against the first variant (all variants compute the same sums in a different order: expect ~1e-15).
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_1906_04209_b200 as nc
from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
cfg = CONFIGS[os.environ["CFG"]]
tab = load_tables(os.environ.get("NC_TABLES_FILE") or os.path.join(os.environ["ROOT"], "tables", "data", cfg.name + ".npz"))
h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
x = torch.from_numpy(h.to_internal(random_coeffs(cfg.N, tab.K, 2000 + int(cfg.name[1:])))).cuda()
y = torch.empty_like(x)
for _ in range(2):
    h.matvec(x, y)
torch.cuda.synchronize()
h.time_stages(True)
g, t, r = [], [], []
for _ in range(3):
    h.matvec(x, y)
    st = h.stats()
    g.append(st["ms_last"][4]); t.append(st["ms_last"][6]); r.append(st["ms_last"][5])
np.save(os.environ["OUT"], y.cpu().numpy())
print(json.dumps({"variant": os.environ.get("VARIANT"), "grid_ms": float(np.median(g)), "rest_ms": float(np.median(r)),
                  "matvec_ms": float(np.median(t)), "pairs": st["hier_grid_pairs"],
                  "units": st["hier_grid_units"], "fill": st["hier_grid_fill"], "warp_fill": st["hier_grid_warp_fill"]}))
"""


def main():
    cfg = sys.argv[1]
    ref = None
    for k, v in enumerate(sys.argv[2:]):
        out = f"/tmp/sweep_{k}.npy"
        env = dict(os.environ, NC_TUNING="1", ROOT=ROOT, CFG=cfg, OUT=out, VARIANT=v)
        for spec in v.split(";"):                 # "NAME=value;..." sets env vars, a bare value NC_GRID_VARIANT
            if "=" in spec:
                k_, v_ = spec.split("=", 1)
                env[k_] = v_
            elif spec:
                env["NC_GRID_VARIANT"] = spec
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=240)
        if r.returncode != 0:
            print(json.dumps({"variant": v, "error": r.stderr[-400:]}), flush=True)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        y = np.load(out)
        if ref is None:
            ref = y
        d["rel_diff_vs_first"] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
        d["pairs_per_s"] = d["pairs"] / (d["grid_ms"] * 1e-3)
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
