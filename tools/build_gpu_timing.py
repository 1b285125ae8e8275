"""NEXT-1 measurement: Step-1 table build for a config with the ID sketches on the GPU (nc_id_sketch) vs the stored
CPU-built table: phase times, skeleton sizes per rung and the difference of the outgoing operators.
    python tools/build_gpu_timing.py C5"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from nc_inputs import CONFIGS  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402
from nc_tables.build import build_tables  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = CONFIGS[name]
ref = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
t0 = time.time()
d = build_tables(cfg.kind, cfg.eps, gpu_sketch=True)
wall = time.time() - t0
m = d["meta"]
same_p = bool(d["T"].shape == ref.T.shape and list(d["ladder_p"]) == list(ref.ladder_p))
out = {"config": name, "wall_s": wall, "t_onepatch_s": m["t_onepatch_s"], "t_id_s": m["t_id_s"],
       "t_ladder_s": m["t_ladder_s"], "p": int(d["T"].shape[0]), "ladder_p": [int(v) for v in d["ladder_p"]],
       "same_skeleton_sizes_as_cpu_table": same_p,
       "T_rel_diff_vs_cpu": (float(np.linalg.norm(d["T"] - ref.T) / np.linalg.norm(ref.T)) if d["T"].shape == ref.T.shape
                             else None),
       "outgoing_rel_err": m["outgoing_rel_err"], "cpu_table_meta_times": {k: v for k, v in
                                                                            (("t_id_s", None), ("t_ladder_s", None))}}
import re  # noqa: E402
for k in ("t_onepatch_s", "t_id_s", "t_ladder_s"):
    r = re.search(f"'{k}': ([0-9.e+-]+)", str(ref.meta.get("repr", "")))
    out["cpu_table_meta_times"][k] = float(r.group(1)) if r else None
# the base-rung ID on this machine's CPU (numpy sketch) vs the GPU sketch: same box, same inputs
from nc_tables import onepatch, skeleton  # noqa: E402
import paper_1906_04209_b200 as nc  # noqa: E402
op = onepatch.solve_onepatch(cfg.kind, cfg.eps)
fine, wf, B = onepatch.fine_grid(op)
train = skeleton.training_grid(cfg.eps)
t1 = time.time()
Jc, _ = skeleton.interp_decomp(cfg.kind, train, fine, 1e-11)
tc = time.time() - t1
t1 = time.time()
Jg, _ = skeleton.interp_decomp(cfg.kind, train, fine, 1e-11, sketch=nc.id_sketch)
tg = time.time() - t1
out["base_id_same_machine"] = {"cpu_s": tc, "gpu_s": tg, "cores": os.cpu_count(),
                               "same_skeleton": bool(np.array_equal(np.sort(Jc), np.sort(Jg)))}
print(json.dumps(out), flush=True)
