"""N > 1 host logic on CPU (gloo, world size 2): libnc's row partition (nc_split_rows, host-only) and the sharded
matvec / GMRES algebra libnc runs over NCCL (rank-local T-apply, all-gather-v of the source charges, rank-local
pair sums and P-apply, all-reduced CGS2 dot products), emulated with the oracle's arithmetic on each rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from nc_inputs import CONFIGS, random_coeffs, synthetic_tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_split_rows_properties():
    from paper_1906_04209_b200 import nc
    rng = np.random.default_rng(0)
    for N, world in [(10, 3), (1000, 8), (7, 8), (1, 1), (100000, 4)]:
        w = rng.exponential(size=N) * 50
        for weights in (None, w):
            b, c = nc.split_rows(N, world, weights)
            assert b[0] == 0 and np.all(c >= 0) and b[-1] + c[-1] == N
            assert np.all(b[1:] == b[:-1] + c[:-1])                      # contiguous, ordered, complete
            ww = np.ones(N) if weights is None else weights + 1.0
            loads = np.array([ww[bb:bb + cc].sum() for bb, cc in zip(b, c)])
            assert loads.max() <= ww.sum() / world + ww.max() + 1e-9       # balanced up to one row


def _allgather_rows(local, counts):
    """all-gather-v of row blocks (pad to the max count, gather, trim) -- the NCCL broadcast-per-rank analogue."""
    mx = int(max(counts))
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=torch.float64)
    pad[: local.shape[0]] = torch.from_numpy(local)
    parts = [torch.zeros_like(pad) for _ in counts]
    dist.all_gather(parts, pad)
    return np.concatenate([p[:c].numpy() for p, c in zip(parts, counts)])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1906_04209_b200 import nc
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=21, coupling=30.0)
    N, K = cfg.N, tab.K
    b, cnt = nc.split_rows(N, world)
    rows = np.arange(b[rank], b[rank] + cnt[rank])
    R = O.frames(c)
    s = O.global_nodes(R, tab.shat).reshape(-1, 3)
    spatch = np.repeat(np.arange(N), tab.p)

    def dist_matvec(x_loc):
        rho_loc = O.outgoing(tab.T, x_loc)                     # K1 on this rank's rows
        rho = _allgather_rows(rho_loc, cnt)                    # all-gather-v of the charges
        z = O.global_nodes(R[rows], tab.zhat)
        u = O.field(cfg.kind, z, np.repeat(rows, tab.Kstar), s, spatch, rho).reshape(len(rows), tab.Kstar)
        return x_loc + u @ tab.P.T                              # K3 on this rank's rows

    x = random_coeffs(N, K, 2001)
    y = _allgather_rows(dist_matvec(x[rows]), cnt)

    # CGS2 GMRES with all-reduced projections (the structure of nc_gmres)
    def allreduce(v):
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    bvec = O.rhs(tab, N)[rows].ravel()
    beta = np.sqrt(allreduce(np.array([bvec @ bvec]))[0])
    m = 60
    V = [bvec / beta]
    H = np.zeros((m + 1, m))
    g = np.zeros(m + 1)
    g[0] = beta
    cs, sn = np.zeros(m), np.zeros(m)
    k = 0
    for j in range(m):
        w = dist_matvec(V[j].reshape(len(rows), K)).ravel()
        for _ in range(2):
            h = allreduce(np.array([v @ w for v in V]))
            w = w - sum(hh * v for hh, v in zip(h, V))
            H[: j + 1, j] += h
        H[j + 1, j] = np.sqrt(allreduce(np.array([w @ w]))[0])
        V.append(w / H[j + 1, j])
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        r = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / r, H[j + 1, j] / r
        H[j, j], H[j + 1, j] = r, 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        if abs(g[k]) / beta <= 1e-12:
            break
    yk = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
    xs = sum(yy * v for yy, v in zip(yk, V[:k])).reshape(len(rows), K)
    xs_all = _allgather_rows(xs, cnt)
    I_loc = tab.I @ xs.sum(axis=0)
    I_sigma = allreduce(np.array([I_loc]))[0]
    if rank == 0:
        out.put((y, xs_all, k, I_sigma))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_matvec_and_gmres_gloo_world2():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y, xs, k, I_sigma = q.get(timeout=280)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=21, coupling=30.0)
    x = random_coeffs(cfg.N, tab.K, 2001)
    np.testing.assert_allclose(y, O.matvec(cfg.kind, c, tab, x), rtol=1e-13, atol=1e-14)   # sharding changes nothing
    ref = O.solve(cfg.kind, c, tab, tol=1e-12)
    assert abs(k - ref["iters"]) <= 1
    assert np.linalg.norm(xs - ref["x"]) / np.linalg.norm(ref["x"]) < 1e-10
    assert abs(I_sigma - ref["I_sigma"]) <= 1e-9 * abs(ref["I_sigma"])
