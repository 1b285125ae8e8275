"""Build a config's tables with another ladder ID tolerance (GPU Step 1) into a scratch file, for NC_TABLES_FILE runs.
    python tools/ladder_tol_probe.py C5 3e-10 /tmp/C5_lt.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from nc_inputs import CONFIGS  # noqa: E402
from nc_tables.build import build_tables, save  # noqa: E402
from nc_tables.residual import add_to_tables  # noqa: E402

name, tol, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
cfg = CONFIGS[name]
d = build_tables(cfg.kind, cfg.eps, ladder_id_tol=tol, gpu_sketch=True)
save(d, out)
add_to_tables(out)
print(name, "ladder tol", tol, "sum p", int(sum(d["ladder_p"])), list(d["ladder_p"]), flush=True)
