"""Build a config's tables with another ladder ratio (GPU sketches) into a scratch file, for sweep_grid / accuracy
runs with NC_TABLES_FILE.   python tools/ladder_ratio_probe.py C5 0.25 /tmp/C5_r4.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from nc_inputs import CONFIGS  # noqa: E402
from nc_tables.build import build_tables, save  # noqa: E402

name, expo, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
cfg = CONFIGS[name]
d = build_tables(cfg.kind, cfg.eps, ladder_ratio=2.0 ** expo, gpu_sketch=True)
save(d, out)
print(name, "ratio 2^", expo, "rungs", len(d["ladder_p"]), "sum p", int(sum(d["ladder_p"])), flush=True)
