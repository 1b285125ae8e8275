"""Setup-phase wall-clock timings of nc_setup (NC_SETUP_TIMING=1 prints them to stderr), with the CUDA context and
libnc's module already initialised (so the first phase does not include process-level CUDA start-up).

    NC_SETUP_TIMING=1 python tools/setup_timing.py C5
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04209_b200 as nc  # noqa: E402
from nc_inputs import CONFIGS  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = CONFIGS[name]
tab = load_tables(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tables", "data",
                               f"{name}.npz"))
c = cfg.centers()
torch.zeros(1, device="cuda")
warm = nc.Handle(cfg.kind, c[:64], cfg.eps, tab, mode=nc.NC_HIER)   # loads libnc's kernels
warm.close()
torch.cuda.synchronize()
out = []
for rep in range(2):
    t0 = time.perf_counter()
    h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
    torch.cuda.synchronize()
    out.append(time.perf_counter() - t0)
    h.close()
print(json.dumps({"config": name, "setup_s": out, "threads": os.cpu_count()}))
