"""Hierarchical-vs-direct matvec error (full vectors, both on the GPU) for a config and a list of precisions."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1906_04209_b200 as nc
from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
name = sys.argv[1]
precs = [float(v) for v in sys.argv[2:]] or [1e-9]
cfg = CONFIGS[name]
tab = load_tables(os.environ.get("NC_TABLES_FILE") or f"tables/data/{name}.npz")
c = cfg.centers()
xr = random_coeffs(cfg.N, tab.K, 7)
xb = np.tile(tab.P @ np.ones(tab.Kstar), (cfg.N, 1))        # the physical right-hand side P.1 (coherent charges)
hd = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_DIRECT)
yds = [hd.to_caller(hd.matvec(torch.from_numpy(hd.to_internal(x)).cuda()).cpu().numpy()) for x in (xr, xb)]
hd.close()
fac = os.environ.get("NC_GRID_TOL_FACTOR", "default")
for pr in precs:
    hh = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=nc.NC_HIER, precision=pr)
    errs = []
    for x, yd in zip((xr, xb), yds):
        xi = torch.from_numpy(hh.to_internal(x)).cuda()
        hh.matvec(xi); torch.cuda.synchronize()
        t0 = time.time(); y = hh.matvec(xi); torch.cuda.synchronize(); dt = time.time() - t0
        yh = hh.to_caller(y.cpu().numpy())
        errs.append((np.linalg.norm(yh - yd) / np.linalg.norm(yd), np.linalg.norm(yh - yd) / np.linalg.norm(yd - x)))
    st = hh.stats()
    print(json.dumps({"config": name, "precision": pr, "tol_factor": fac, "rel_err_random": errs[0][0],
                      "rel_err_P1": errs[1][0], "rel_err_P1_vs_operator": errs[1][1], "matvec_s": dt,
                      "grid_pairs": st["hier_grid_pairs"], "near_pairs": st["hier_near_pairs"],
                      "grid_points": st["hier_grid_points"]}), flush=True)
    hh.close()
