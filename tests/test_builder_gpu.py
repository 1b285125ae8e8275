"""NEXT-1: the GPU sketch of the Step-1 interpolative decomposition (nc_id_sketch) against the
CPU builder's numpy sketch (nc_tables/skeleton.py), and the skeleton / outgoing operator it leads to.

Y = Omega G(train, fine) on the same Omega: <= 1e-13 relative (fp64 GEMM of a well-scaled
kernel matrix).  The pivoted QR then picks the same skeleton and T reproduces the far field to the ID tolerance
(outgoing_error, eq:outgoingcompressed) like the CPU-built one."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,eps,inner", [(0, 0.02, 2.0), (1, 0.005, 2.0 * 2 ** (1 / 3))])
def test_id_sketch_matches_cpu(kind, eps, inner):
    import paper_1906_04209_b200 as nc
    from nc_tables import onepatch, skeleton
    from nc_tables.kernel import green_xyz
    op = onepatch.solve_onepatch(kind, eps, M=6, npan=8, k=10)
    fine, wf, B = onepatch.fine_grid(op)
    train = skeleton.training_grid(eps, inner=inner)
    om = skeleton.test_matrix(train.shape[0], 200)
    Yg = nc.id_sketch(kind, train, fine, om)
    Yc = om @ green_xyz(kind, train[:, None, :], fine[None, :, :])
    assert np.linalg.norm(Yg - Yc) / np.linalg.norm(Yc) <= 1e-13
    Jc, Pc = skeleton.interp_decomp(kind, train, fine, 1e-10, oversample=200)
    Jg, Pg = skeleton.interp_decomp(kind, train, fine, 1e-10, oversample=200, sketch=nc.id_sketch)
    assert len(Jg) == len(Jc) and np.array_equal(np.sort(Jg), np.sort(Jc))
    Tg = Pg @ (wf[:, None] * B)
    err = skeleton.outgoing_error(kind, fine, wf, B, fine[Jg], Tg, eps, inner=inner)
    assert err <= 1e-8


def test_id_sketch_argument_checks():
    import paper_1906_04209_b200 as nc
    with pytest.raises(nc.NcError, match="NC_EINVAL"):
        nc.id_sketch(2, np.zeros((3, 3)), np.ones((2, 3)), np.ones((1, 3)))


@pytest.mark.parametrize("kind", [0, 1])
def test_modal_kernels_match_cpu(kind):
    """The one-patch solver's modal kernels G_m(t, t') on the GPU against kernel.modal (numpy),
    including the nearly singular t ~ t' pairs the solver's graded rules produce."""
    import paper_1906_04209_b200 as nc
    from nc_tables.kernel import modal, phi_rule
    from nc_tables.onepatch import _row_rules, radial_grid
    g = radial_grid(0.02, 8, 10)
    ti = g.t[[0, 20, 55, 79]]
    tq = [np.concatenate([r[0] for r in _row_rules(g, t)]) for t in ti]
    T = np.concatenate([np.full(q.size, t) for t, q in zip(ti, tq)])
    TQ = np.concatenate(tq)
    phi, wphi = phi_rule()
    Gg = nc.modal_kernels(kind, T, TQ, 15, phi, wphi)
    Gc = modal(kind, T, TQ, 15)
    assert np.max(np.abs(Gg - Gc) / (np.abs(Gc) + np.max(np.abs(Gc), axis=1, keepdims=True))) <= 1e-13


def test_onepatch_gpu_modal_same_solution():
    from nc_tables import onepatch
    from nc_tables.kernel import modal_gpu
    a = onepatch.solve_onepatch(0, 0.05, M=8, npan=8, k=10)
    b = onepatch.solve_onepatch(0, 0.05, M=8, npan=8, k=10, modal_fn=modal_gpu)
    assert np.max(np.abs(a.sigma_radial - b.sigma_radial)) <= 1e-11 * np.max(np.abs(a.sigma_radial))
