"""Rebuild the physical tables (Step 1) with the ID sketches on the GPU (NEXT-1) into a directory:
    python tools/build_tables_gpu.py <out_dir> [radial=r2|r] C1 C2 ...
(one-patch solve, base ID, per-level ladder, residual grid; the same parameters as nc_tables.build --configs)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from nc_inputs import CONFIGS  # noqa: E402
from nc_tables.build import build_tables, save  # noqa: E402
from nc_tables.residual import add_to_tables  # noqa: E402

out, radial = sys.argv[1], sys.argv[2]
os.makedirs(out, exist_ok=True)
for name in sys.argv[3:]:
    cfg = CONFIGS[name]
    t0 = time.time()
    path = os.path.join(out, f"{name}.npz")
    save(build_tables(cfg.kind, cfg.eps, gpu_sketch=True, zn_radial=radial), path)
    add_to_tables(path)
    print(f"{name}: {time.time() - t0:.1f} s", flush=True)
