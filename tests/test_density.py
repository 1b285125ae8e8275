"""Density recovery (NEXT-3; eq:recoversig PAPER.md:797-807): sigma_i = B fhat_i.

CPU pin: the fine-grid quadrature of the recovered density is the read-out row, w . (B fhat) = I . fhat for every
fhat (the table's I is w^T B, eq:getI PAPER.md:1025-1033), rebuilt here from the one-patch solver and compared with
the stored physical table; and a single patch solved exactly (x = P 1) has a density whose integral is that
patch's I_sigma.  GPU parity: nc_density against the oracle's matmul."""
import os

import numpy as np
import pytest

from nc_inputs import CONFIGS, random_coeffs
from nc_inputs.tables import load_tables
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c1_fine():
    from nc_tables import onepatch
    tab = load_tables(os.path.join(ROOT, "tables", "data", "C1.npz"))
    op = onepatch.solve_onepatch(tab.kind, tab.eps, tab.M, 13, 20, 64)
    fine, wf, B = onepatch.fine_grid(op)
    return tab, fine, wf, B


def test_density_integral_is_readout_row(c1_fine):
    tab, fine, wf, B = c1_fine
    assert np.linalg.norm(wf @ B - tab.I) <= 1e-12 * np.linalg.norm(tab.I)
    x = random_coeffs(3, tab.K, 5)
    sig = O.density(x, [0, 1, 2], B)
    assert np.allclose(sig @ wf, x @ tab.I, rtol=1e-12, atol=1e-15)
    # one patch, exact solution of the N = 1 system (x = P 1): I_sigma = int sigma dS
    x1 = (tab.P @ np.ones(tab.Kstar))[None, :]
    Is, _ = O.readout(tab.kind, tab.I, x1)
    assert abs(O.density(x1, [0], B)[0] @ wf - Is) <= 1e-12 * abs(Is)


@pytest.mark.gpu
def test_density_gpu_parity(c1_fine):
    torch = pytest.importorskip("torch")
    import paper_1906_04209_b200 as nc
    tab, fine, wf, B = c1_fine
    cfg = CONFIGS["C1"]
    h = nc.Handle(cfg.kind, cfg.centers(), cfg.eps, tab)
    x = random_coeffs(cfg.N, tab.K, 6)
    xi = torch.from_numpy(h.to_internal(x)).cuda()
    pats = [3, 0, 9]
    sig = h.density(xi, pats, B)
    ref = O.density(x, pats, B)
    assert np.linalg.norm(sig - ref) / np.linalg.norm(ref) <= 1e-14
    assert h.density(xi, [], B).shape == (0, B.shape[0])
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        h.density(xi, [cfg.N], B)
    h.close()
