"""Multi-rank partition on ONE GPU by rank emulation (include/nc.h nc_matvec_emulated): every rank of a world-W
partition computes its rows with the all-gather replaced by computing all outgoing records from the full input.
The concatenated rank outputs must equal the world-1 matvec (same kernels, same per-row summation order): this
checks the row cuts, the work-weighted hierarchical partition, the redundant groups straddling a cut and the
per-rank near lists — everything of the N > 1 path except NCCL itself."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _nc():
    import paper_1906_04209_b200 as nc
    return nc


def _phys(name):
    from nc_inputs.tables import load_tables
    return load_tables(os.path.join(ROOT, "tables", "data", f"{name}.npz"))


@pytest.mark.parametrize("name,mode,worlds", [("C2", 0, (2, 3)), ("C2", 1, (2, 3)), ("C4", 1, (4,)),
                                              ("C1", 0, (3,))])
def test_emulated_ranks_match_world1(name, mode, worlds):
    nc = _nc()
    cfg = CONFIGS[name]
    c = cfg.centers()
    tab = _phys(name)
    x = random_coeffs(cfg.N, tab.K, 99)
    h1 = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=mode, precision=cfg.precision)
    xi = torch.from_numpy(h1.to_internal(x)).cuda()
    y1 = h1.matvec(xi).cpu().numpy()
    perm1 = h1.perm.copy()
    h1.close()
    for W in worlds:
        parts, begins = [], []
        for r in range(W):
            h = nc.Handle(cfg.kind, c, cfg.eps, tab, mode=mode, precision=cfg.precision, world=W, rank=r)
            assert np.array_equal(h.perm, perm1)           # the internal order does not depend on the partition
            begins.append((h.row_begin, h.row_count))
            parts.append(h.matvec_emulated(xi).cpu().numpy())
            with pytest.raises(nc.NcError):                 # no communicator: the collective entry points refuse
                h.matvec(xi[h.row_begin:h.row_begin + h.row_count].contiguous())
            h.close()
        assert begins[0][0] == 0 and sum(b[1] for b in begins) == cfg.N
        assert all(begins[k][0] + begins[k][1] == begins[k + 1][0] for k in range(W - 1))
        y = np.concatenate(parts)
        err = np.linalg.norm(y - y1) / np.linalg.norm(y1)
        assert err <= 1e-14, (W, err)
