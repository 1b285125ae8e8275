"""Quick hierarchical-mode probe: setup time, stats, matvec time for a config (not a test)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1906_04209_b200 as nc
from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = CONFIGS[name]
tab = load_tables(os.environ.get("NC_TABLES_FILE") or f"tables/data/{name}.npz")
c = cfg.centers()
t0 = time.time()
h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
torch.cuda.synchronize(); ts = time.time() - t0
x = torch.from_numpy(h.to_internal(random_coeffs(cfg.N, tab.K, 1))).cuda()
y = h.matvec(x); torch.cuda.synchronize()
h.time_stages(True)
t0 = time.time(); y = h.matvec(x); torch.cuda.synchronize(); tm = time.time() - t0
st = h.stats()
print(json.dumps({"config": name, "setup_s": ts, "matvec_s": tm, "stats": st}))
