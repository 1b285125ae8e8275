"""Write the oracle-computed golden values under tests/golden/ (TEST INFRASTRUCTURE; calls only oracle/ and the
seeded inputs of nc_inputs/ -- nothing here touches the CUDA path).

    python tools/make_goldens.py rows C3 C4 C5      # sampled matvec rows
    python tools/make_goldens.py solve C2           # the full oracle GMRES solve

rows: y_i = x_i + P u_i (eq:sysmatapply; eq:mssums with eq:outgoingcompressed) for target patches
chosen on purpose from the layout's geometry, so that a fault confined to one region of the tree cannot hide:
  * the patches nearest the 8 corners and the 12 edge midpoints of the cube the tree projects the sphere onto
    (R11: cube-face quadtree; corners have 7 neighbours);
  * patches on the face boundaries (the two largest |coordinates| within 1%: boxes that straddle two faces);
  * patches on the level-1 box boundaries (a face coordinate u/|x_max| near 0);
  * the patches with the most neighbours within 8 eps (the densest vMF cap of C4, the tightest spacing elsewhere);
  * seeded uniform picks for the rest.
x is the bench's seeded x ~ N(0,1) (seed 2000 + config number); tables are the committed physical tables.
solve: GMRES to 1e-10 from x0 = 0 on b = P 1, MGS + reorthogonalisation; the read-out
I_sigma = I . sum_i fhat_i (eq:getI) and J = -4 pi I_sigma (R2) or mu = 1/(3 I_sigma) - 3/5 (eq:mufromsigma2).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from nc_inputs import CONFIGS, random_coeffs  # noqa: E402
from nc_inputs.tables import load_tables  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
N_ROWS = {"C3": 64, "C4": 64, "C5": 40}


def _nearest(c, dirs, taken):
    out = []
    for d in dirs:
        d = np.asarray(d, dtype=np.float64)
        d = d / np.linalg.norm(d)
        order = np.argsort(-(c @ d))
        for i in order:
            if int(i) not in taken:
                out.append(int(i))
                taken.add(int(i))
                break
    return out


def select_rows(c, eps, n, seed):
    """Target patches chosen from the geometry alone (see the module docstring).  Returns (rows, tags)."""
    taken, rows, tags = set(), [], []

    def add(lst, tag):
        for i in lst:
            rows.append(i)
            tags.append(tag)

    corners = [(sx, sy, sz) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
    edges = []
    for a in range(3):
        for s1 in (-1, 1):
            for s2 in (-1, 1):
                v = [0.0, 0.0, 0.0]
                v[(a + 1) % 3], v[(a + 2) % 3] = s1, s2
                edges.append(v)
    n_corner = 8 if n >= 32 else 4
    n_edge = 12 if n >= 32 else 4
    add(_nearest(c, corners[:n_corner], taken), "cube_corner")
    add(_nearest(c, edges[:n_edge], taken), "cube_edge")
    rng = np.random.default_rng(seed)
    ab = np.sort(np.abs(c), axis=1)
    face_bd = np.where(ab[:, 2] - ab[:, 1] < 0.01 * ab[:, 2])[0]
    cand = [int(i) for i in rng.permutation(face_bd) if int(i) not in taken][: max(4, n // 8)]
    taken.update(cand)
    add(cand, "face_boundary")
    # level-1 box boundaries: the smaller face coordinate of the dominant axis' face near 0
    amax = np.argmax(np.abs(c), axis=1)
    u = np.abs(c[np.arange(len(c)), (amax + 1) % 3] / np.abs(c[np.arange(len(c)), amax]))
    lvl1 = np.where(u < 2.0 * eps)[0]
    cand = [int(i) for i in rng.permutation(lvl1) if int(i) not in taken][: max(4, n // 8)]
    taken.update(cand)
    add(cand, "level1_boundary")
    # densest: most neighbours within 8 eps (chord)
    from scipy.spatial import cKDTree
    cnt = cKDTree(c).query_ball_point(c, 2 * np.sin(4 * eps), return_length=True)
    dense = [int(i) for i in np.argsort(-cnt, kind="stable") if int(i) not in taken][: max(4, n // 8)]
    taken.update(dense)
    add(dense, "densest")
    rest = [int(i) for i in rng.permutation(len(c)) if int(i) not in taken][: n - len(rows)]
    add(rest, "uniform")
    return np.array(rows[:n], dtype=np.int64), tags[:n]


def rows_golden(name):
    cfg = CONFIGS[name]
    c = cfg.centers()
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    seed = 2000 + int(name[1:])
    x = random_coeffs(cfg.N, tab.K, seed)
    rows, tags = select_rows(c, cfg.eps, N_ROWS[name], seed=17)
    t0 = time.time()
    y = O.matvec(cfg.kind, c, tab, x, rows=rows)
    dt = time.time() - t0
    path = os.path.join(GOLD, f"oracle_rows_{name}.npz")
    np.savez_compressed(path, rows=rows, tags=np.array(tags), y=y, x_seed=seed, kind=cfg.kind, N=cfg.N, eps=cfg.eps,
                        tables=f"tables/data/{name}.npz", oracle_seconds=dt, oracle_threads=O.num_threads())
    print(f"{name}: {len(rows)} rows in {dt:.1f} s on {O.num_threads()} threads -> {path}", flush=True)


def solve_golden(name):
    cfg = CONFIGS[name]
    c = cfg.centers()
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    t0 = time.time()
    r = O.solve(cfg.kind, c, tab, tol=cfg.gmres_tol, max_iter=300)
    dt = time.time() - t0
    out = {"config": name, "kind": cfg.kind, "N": cfg.N, "eps": cfg.eps, "tables": f"tables/data/{name}.npz",
           "gmres_tol": cfg.gmres_tol, "iters": int(r["iters"]), "I_sigma": r["I_sigma"],
           ("mu" if cfg.kind == 0 else "J"): r["value"], "explicit_residual": r["explicit_residual"],
           "hist": [float(v) for v in r["hist"]], "oracle_seconds": dt, "oracle_threads": O.num_threads(),
           "source": "tools/make_goldens.py solve (oracle.solve: MGS+reorth GMRES, x0 = 0, b = P 1; read-out "
                     "eq:getI PAPER.md:1025-1033, J = -4 pi I_sigma DESIGN.md R2, mu eq:mufromsigma2 PAPER.md:618)"}
    path = os.path.join(GOLD, f"oracle_solve_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: solve in {dt:.1f} s, {r['iters']} iterations, I_sigma {r['I_sigma']:.15g} -> {path}", flush=True)


def main():
    os.makedirs(GOLD, exist_ok=True)
    what, names = sys.argv[1], sys.argv[2:]
    for n in names:
        (rows_golden if what == "rows" else solve_golden)(n)


if __name__ == "__main__":
    main()
