"""One setting of the grid-size knobs per process (the margins are read once per process): hierarchical matvec error
(C3, C4 against the GPU direct sum; C5 against the hierarchical matvec at tolerance factor 100 with the default
margins), grid pairs and matvec time.  References are cached under /tmp by the first call of a sweep.

    NC_TUNING=1 [NC_GRID_TOL_FACTOR=.. NC_NA_MARGIN=.. NC_NR_MARGIN=.. NC_RING_MARGIN=.. NC_RING_FLOOR=..] \
        python tools/margin_sweep.py <label> [configs...]
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
label = sys.argv[1]
KNOBS = ["NC_GRID_TOL_FACTOR", "NC_NA_MARGIN", "NC_NR_MARGIN", "NC_RING_MARGIN", "NC_RING_FLOOR"]
for name in sys.argv[2:] or ["C3", "C4", "C5"]:
    cfg = CONFIGS[name]
    tab = load_tables(f"tables/data/{name}.npz")
    c = cfg.centers()
    x = random_coeffs(cfg.N, tab.K, 7)
    ref_path = f"/tmp/margin_sweep_ref_{name}.npy"
    if label == "ref":
        if cfg.N <= 20000:
            hd = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
            y = hd.to_caller(hd.matvec(torch.from_numpy(hd.to_internal(x)).cuda()).cpu().numpy())
        else:
            assert os.environ.get("NC_GRID_TOL_FACTOR") == "100"
            hd = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=1e-9)
            y = hd.to_caller(hd.matvec(torch.from_numpy(hd.to_internal(x)).cuda()).cpu().numpy())
        hd.close()
        np.save(ref_path, y)
        continue
    yr = np.load(ref_path)
    hh = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=1e-9)
    xi = torch.from_numpy(hh.to_internal(x)).cuda()
    y = hh.to_caller(hh.matvec(xi).cpu().numpy())
    hh.time_stages(True)
    hh.matvec(xi)
    torch.cuda.synchronize()
    tot, grid, rest = [], [], []
    for _ in range(5):
        hh.matvec(xi)
        torch.cuda.synchronize()
        ms = hh.stats()["ms_last"]
        grid.append(ms[4]); rest.append(ms[5]); tot.append(ms[6])
    st = hh.stats()
    print(json.dumps({"config": name, "setting": label, "knobs": {k: os.environ[k] for k in KNOBS if k in os.environ},
                      "rel_err": float(np.linalg.norm(y - yr) / np.linalg.norm(yr)),
                      "reference": "GPU direct" if cfg.N <= 20000 else "hier, factor 100, default margins",
                      "grid_pairs": st["hier_grid_pairs"], "total_ms": float(np.median(tot)),
                      "grid_ms": float(np.median(grid)), "hier_rest_ms": float(np.median(rest))}), flush=True)
    hh.close()
