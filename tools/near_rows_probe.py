"""One setting of the grid-size knobs per process: the errors tests/test_parity_golden_gpu.py::
test_hier_rows_near_lists_and_rank_cuts_vs_oracle asserts on (rows with the largest near lists, rows at the rank cuts,
each against live oracle rows), so that a default can be chosen with a margin on the 2-row groups, not only on the
whole-vector error (R21).

    NC_TUNING=1 [knobs] python tools/near_rows_probe.py <label> [configs...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS, random_coeffs  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402
from oracle import oracle as O  # noqa: E402  (a probe is test infrastructure, not the product path)

assert os.environ.get("NC_TUNING") == "1"
label = sys.argv[1]
PICK = {"C3": (4, 3), "C4": (4, 3), "C5": (2, 1)}
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for name in sys.argv[2:] or ["C3", "C4", "C5"]:
    cfg = CONFIGS[name]
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    c = cfg.centers()
    x = random_coeffs(cfg.N, tab.K, 2000 + int(name[1:]))
    h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
    y = h.to_caller(h.matvec(torch.from_numpy(h.to_internal(x)).cuda()).cpu().numpy())
    n_near, n_cut = PICK[name]
    counts = h.near_counts()
    order = np.argsort(-counts, kind="stable")
    near = sorted({int(h.perm[h.row_begin + i]) for i in order[:8] if counts[i] > 0})
    near_t = sorted({int(h.perm[h.row_begin + i]) for i in order[:n_near] if counts[i] > 0})
    cut = []
    for world in (2, 4, 8):
        hr = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision, world=world, rank=1)
        cut += [int(hr.perm[hr.row_begin - 1]), int(hr.perm[hr.row_begin])]
        hr.close()
    cut_t = sorted(set(cut[: 2 * n_cut]))
    rows = np.asarray(sorted(set(near) | set(cut)), dtype=np.int64)
    ref = O.matvec(cfg.kind, c, tab, x, rows=rows)
    idx = {int(r): i for i, r in enumerate(rows)}
    per_row = {int(r): rel(y[r], ref[idx[int(r)]]) for r in rows}
    grp = lambda rs: rel(y[np.asarray(rs)], ref[[idx[r] for r in rs]])
    print(json.dumps({"config": name, "setting": label, "test_near_rows": grp(near_t), "test_cut_rows": grp(cut_t),
                      "near8": grp(near), "cuts_all": grp(sorted(set(cut))), "worst_row": max(per_row.values()),
                      "grid_pairs": h.stats()["hier_grid_pairs"]}), flush=True)
    h.close()
