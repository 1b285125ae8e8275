"""The N > 1 path through the product in separate processes: two ranks, each its
own process with its own libnc handle (world 2, rank emulation: no communicator), exchange through torch.distributed
over gloo on the host -- the all-gather of x before every matvec and the all-reduce of the Arnoldi dot products and
norms, the two collectives nc_matvec / nc_gmres issue over NCCL at world > 1.  Each rank's matvec is libnc's
(nc_matvec_emulated on the gathered x: its work-weighted rows, redundant straddling groups, near lists); the GMRES
driver here mirrors nc_gmres's CGS2 on the rank shards with gloo reductions.  The two ranks' kernels never wait on
each other (the exchange is on the host), so one GPU serves both.  Checked against world 1 (nc_gmres): the sharded
matvec to 1e-14, the solved J to 1e-10."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, port, name, out):
    import torch.distributed as dist
    import paper_1906_04209_b200 as nc
    from nc_inputs.tables import load_tables
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS[name]
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision, world=world,
                  rank=rank)
    counts = [None] * world
    dist.all_gather_object(counts, (h.row_begin, h.row_count))
    mx = max(c for _, c in counts)

    def gather(v_rows):                                 # the all-gather of x (padded, as nc_matvec's ncclAllGather)
        pad = torch.zeros((mx, h.K), dtype=torch.float64)
        pad[:h.row_count] = v_rows.cpu()
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        return torch.cat([parts[r][:counts[r][1]] for r in range(world)]).cuda()

    def matvec(v_rows):
        return h.matvec_emulated(gather(v_rows))

    def allsum(t):                                      # the all-reduce of dot products / norms
        c = t.cpu()
        dist.all_reduce(c)
        return c.cuda()

    x_all = random_coeffs(cfg.N, tab.K, 123)
    x_rows = torch.from_numpy(h.to_internal(x_all)).cuda()
    y_rows = matvec(x_rows).cpu().numpy()
    # unrestarted GMRES, x0 = 0, b = P 1 (nc_gmres's problem), CGS2 with gloo-reduced dot products
    b = torch.from_numpy(np.tile(tab.P @ np.ones(tab.Kstar), (h.row_count, 1))).cuda()
    V = [b / torch.sqrt(allsum((b * b).sum().reshape(1)))[0]]
    beta = float(torch.sqrt(allsum((b * b).sum().reshape(1)))[0])
    H = np.zeros((61, 60))
    g = np.zeros(61)
    g[0] = beta
    cs, sn = np.zeros(60), np.zeros(60)
    k = 0
    for j in range(60):
        w = matvec(V[j])
        for _ in range(2):
            hv = allsum(torch.stack([(v * w).sum() for v in V]))
            for i, v in enumerate(V):
                w = w - hv[i] * v
            H[:j + 1, j] += hv.cpu().numpy()
        hn = float(torch.sqrt(allsum((w * w).sum().reshape(1)))[0])
        H[j + 1, j] = hn
        V.append(w / hn)
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        r = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / r, H[j + 1, j] / r
        H[j, j], H[j + 1, j] = r, 0.0
        g[j + 1], g[j] = -sn[j] * g[j], cs[j] * g[j]
        k = j + 1
        if abs(g[k]) / beta <= cfg.gmres_tol:
            break
    yk = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
    xs = sum(float(yk[i]) * V[i] for i in range(k))
    Is = float(allsum((xs.sum(dim=0) * torch.from_numpy(tab.I).cuda()).sum().reshape(1))[0])
    np.save(out + f".{rank}.npy", np.concatenate([y_rows.ravel(), [Is, k, h.row_begin, h.row_count]]))
    h.close()
    dist.destroy_process_group()


def test_two_process_ranks_match_world1(tmp_path):
    import socket
    import torch.multiprocessing as mp
    import paper_1906_04209_b200 as nc
    from nc_inputs.tables import load_tables
    name = "C2"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r")
    mp.start_processes(_rank, args=(2, port, name, out), nprocs=2, start_method="spawn", join=True)
    cfg = CONFIGS[name]
    tab = load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))
    h1 = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab, mode=nc.NC_HIER, precision=cfg.precision)
    x = torch.from_numpy(h1.to_internal(random_coeffs(cfg.N, tab.K, 123))).cuda()
    y1 = h1.matvec(x).cpu().numpy()
    xs, it1, _ = h1.gmres(rtol=cfg.gmres_tol, max_iter=100)
    Is1, J1 = h1.flux_or_mfpt(xs)
    parts = [np.load(out + f".{r}.npy") for r in range(2)]
    ys, Iss = [], []
    for p in parts:
        rb, rc = int(p[-2]), int(p[-1])
        ys.append(p[:rc * tab.K].reshape(rc, tab.K))
        Iss.append(p[-4])
        assert abs(int(p[-3]) - it1) <= 1
    y = np.concatenate(ys)
    assert np.linalg.norm(y - y1) / np.linalg.norm(y1) <= 1e-14
    assert Iss[0] == Iss[1]                           # the all-reduced read-out is the same on both ranks
    assert abs(Iss[0] - Is1) <= 1e-10 * abs(Is1)
    h1.close()
