"""Pins of the CPU oracle against what the paper and mathematics fix ("What pins
each part").  None of these compares the oracle with itself or with the CUDA path."""
import numpy as np
import pytest

from nc_inputs import CONFIGS, synthetic_tables
from nc_inputs.layouts import haar_rotation
from oracle import oracle as O


def _sphere_mean(kind, rng, n_panels=48, order=24):
    """(1/4pi) int_{S^2} G(x, x') dS(x) by dyadic Gauss panels in the polar angle about x'.

    The integrand is evaluated through the oracle's own green() on genuine 3-D points."""
    xp = rng.standard_normal(3)
    xp /= np.linalg.norm(xp)
    R = O.frames(xp[None])[0]
    gx, gw = np.polynomial.legendre.leggauss(order)
    edges = [np.pi / 2.0 ** k for k in range(n_panels)] + [0.0]
    total = 0.0
    for a, b in zip(edges[1:], edges[:-1]):
        t = 0.5 * (b - a) * gx + 0.5 * (b + a)
        w = 0.5 * (b - a) * gw
        phi = rng.random(len(t)) * 2 * np.pi            # integrand is axisymmetric about x'
        loc = np.stack([np.sin(t) * np.cos(phi), np.sin(t) * np.sin(phi), np.cos(t)], 1)
        pts = loc @ R.T
        g = O.green(kind, pts, np.broadcast_to(xp, pts.shape))
        total += np.sum(w * g * np.sin(t)) * 2 * np.pi
    return total / (4 * np.pi)


def test_green_sphere_mean_interior_is_2():
    # PAPER.md:610-612 (§2.3): (1/|dOmega|) int G_I(x, x') dS(x) = 2 for any x' on the sphere
    rng = np.random.default_rng(1)
    for _ in range(3):
        assert abs(_sphere_mean(0, rng) - 2.0) < 1e-12


def test_green_sphere_mean_exterior_is_1():
    # derived: mean of 2/d is 2, mean of log(2/d) = mean of log(1+d/2) = 1/2
    rng = np.random.default_rng(2)
    assert abs(_sphere_mean(1, rng) - 1.0) < 1e-12


def test_green_antipodal_and_symmetry():
    # d = 2: G = 1 + 0 - log 2 for both kinds (eq:Gextonsurface / eq:Gintonsurface)
    x = np.array([[0.0, 0.0, 1.0]])
    y = -x
    for kind in (0, 1):
        assert abs(O.green(kind, x, y)[0] - (1.0 - np.log(2.0))) < 1e-15
    rng = np.random.default_rng(3)
    a = rng.standard_normal((50, 3)); a /= np.linalg.norm(a, axis=1, keepdims=True)
    b = rng.standard_normal((50, 3)); b /= np.linalg.norm(b, axis=1, keepdims=True)
    for kind in (0, 1):
        np.testing.assert_array_equal(O.green(kind, a, b), O.green(kind, b, a))
    # interior minus exterior is 2 log(2/d) ("except for the sign of the second term")
    d = np.linalg.norm(a - b, axis=1)
    np.testing.assert_allclose(O.green(0, a, b) - O.green(1, a, b), 2 * np.log(2 / d), rtol=1e-13, atol=1e-13)


def test_green_flat_limit():
    # as d -> 0 the kernel is dominated by the free-space 2/d
    x = np.array([[0.0, 0.0, 1.0]])
    for d in (1e-3, 1e-5):
        t = 2 * np.arcsin(d / 2)
        y = np.array([[np.sin(t), 0.0, np.cos(t)]])
        for kind in (0, 1):
            g = O.green(kind, x, y)[0]
            assert abs(g * d / 2 - 1) < 10 * d * np.log(2 / d)


def test_frames_are_rotations_about_centre():
    c = CONFIGS["C2"].centers()
    R = O.frames(c)
    np.testing.assert_allclose(np.einsum("iab,iac->ibc", R, R), np.broadcast_to(np.eye(3), R.shape), atol=1e-14)
    np.testing.assert_allclose(np.linalg.det(R), 1.0, atol=1e-14)
    np.testing.assert_allclose(R[:, :, 2], c, atol=0)
    # a canonical node at arc t from the pole lands at arc t from the centre
    t = 0.05
    z = O.global_nodes(R, np.array([[np.sin(t), 0, np.cos(t)]]))[:, 0]
    np.testing.assert_allclose(np.sum(z * c, 1), np.cos(t), atol=1e-15)


def _tiny_tables(kind, eps, K_M=2, rng=None):
    return synthetic_tables(kind, eps, seed=11, M=K_M, p=7, n_r=3, n_theta=5)


def test_matvec_single_patch_is_identity():
    # PAPER.md:883 (Remark zerniketrunc): "In the one-patch case, the summation term vanishes"
    tab = synthetic_tables(0, 0.1, seed=5)
    x = np.random.default_rng(0).standard_normal((1, tab.K))
    np.testing.assert_array_equal(O.matvec(0, np.array([[0.0, 0, 1]]), tab, x), x)


def test_matvec_structure_single_entries():
    """T, P with one nonzero entry and pole nodes: y_i[a] - x_i[a] = G(c_i, c_j) x_j[k] (j != i only).

    Pins operand order (T vs T^T, P vs P^T), the self-exclusion and the identity term."""
    eps = 0.05
    tab = synthetic_tables(1, eps, seed=3, M=3, p=4, n_r=2, n_theta=4)
    tab.zhat[1] = [0.0, 0.0, 1.0]            # node 1 = patch centre
    tab.shat[2] = [0.0, 0.0, 1.0]            # skeleton node 2 = patch centre
    tab.T[:] = 0.0
    tab.T[2, 4] = 1.0                         # rho_{j,2} = x_{j,4}
    tab.P[:] = 0.0
    tab.P[6, 1] = 1.0                         # y_{i,6} += u_{i, node 1}
    c = CONFIGS["C1"].centers()[:4]
    x = np.zeros((4, tab.K))
    x[2, 4] = 1.5
    x[0, 6] = 0.25
    for kind in (0, 1):
        y = O.matvec(kind, c, tab, x)
        exp = x.copy()
        for i in range(4):
            if i != 2:
                exp[i, 6] += O.green(kind, c[i:i + 1], c[2:3])[0] * 1.5
        np.testing.assert_allclose(y, exp, rtol=1e-15, atol=1e-15)


def test_matvec_rotation_permutation_linearity():
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=9, M=5, p=20, n_r=6, n_theta=12)
    rng = np.random.default_rng(4)
    x = rng.standard_normal((cfg.N, tab.K))
    y = O.matvec(cfg.kind, c, tab, x)
    # global rotation of centres and frames (SURVEY.md §8(c) "Invariance under a global rotation")
    Q = haar_rotation(rng)
    R = O.frames(c)
    y_rot = O.matvec(cfg.kind, c @ Q.T, tab, x, R=np.einsum("ab,ibc->iac", Q, R))
    np.testing.assert_allclose(y_rot, y, rtol=1e-12, atol=1e-12)
    # permutation equivariance
    perm = rng.permutation(cfg.N)
    y_perm = O.matvec(cfg.kind, c[perm], tab, x[perm])
    np.testing.assert_allclose(y_perm, y[perm], rtol=1e-13, atol=1e-13)
    # linearity
    x2 = rng.standard_normal(x.shape)
    np.testing.assert_allclose(O.matvec(cfg.kind, c, tab, 2 * x - 3 * x2), 2 * y - 3 * O.matvec(cfg.kind, c, tab, x2),
                               rtol=1e-12, atol=1e-12)
    # sampled rows equal the full rows
    np.testing.assert_array_equal(O.matvec(cfg.kind, c, tab, x, rows=[3, 7]), y[[3, 7]])


def test_matvec_antipodal_pair_symmetric_blocks():
    # two antipodal patches: the configuration is symmetric under the rotation by pi that swaps them
    tab = synthetic_tables(0, 0.1, seed=2, M=4, p=9, n_r=5, n_theta=10)
    c = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])
    Rot = np.diag([1.0, -1.0, -1.0])         # rotation by pi about x maps c0 <-> c1
    R0 = np.eye(3)
    R = np.stack([R0, Rot @ R0])
    x = np.random.default_rng(5).standard_normal((1, tab.K))
    xx = np.vstack([x, x])
    y = O.matvec(0, c, tab, xx, R=R)
    np.testing.assert_allclose(y[0], y[1], rtol=1e-13, atol=1e-13)


def test_gmres_against_dense_lu_C1():
    # textbook dense solve of the assembled (I + A_off) at C1 (1360 unknowns; SURVEY.md §8(c) "GMRES")
    cfg = CONFIGS["C1"]
    c = cfg.centers()
    tab = synthetic_tables(cfg.kind, cfg.eps, seed=21, coupling=30.0)
    A = O.dense_operator(cfg.kind, c, tab)
    b = O.rhs(tab, cfg.N).ravel()
    xs = np.linalg.solve(A, b)
    r = O.solve(cfg.kind, c, tab, tol=1e-12)
    assert r["iters"] > 2
    assert np.linalg.norm(r["x"].ravel() - xs) / np.linalg.norm(xs) < 1e-10
    assert r["explicit_residual"] < 1e-11


def test_gmres_krylov_theory():
    # A = I converges in one step; diag with k distinct eigenvalues in <= k steps (Krylov theory)
    b = np.random.default_rng(0).standard_normal(40)
    x, it, _ = O.gmres(lambda v: v, b, 1e-12, 50)
    assert it == 1 and np.allclose(x, b)
    d = np.repeat([1.0, 2.0, 5.0], [10, 20, 10])
    x, it, hist = O.gmres(lambda v: d * v, b, 1e-12, 50)
    assert it <= 3 and np.allclose(x, b / d, rtol=1e-10)
    assert all(h1 <= h0 + 1e-15 for h0, h1 in zip(hist, hist[1:]))


def test_readout_scalar_maps():
    # eq:mufromsigma2: mu = 1/(3 I) - 3/5;  I = 1/3 -> 2/5; full coverage (sigma = 1/(8 pi), I = 1/2) -> 1/15
    I_row = np.array([1.0, 0.0])
    assert O.readout(0, I_row, np.array([[1.0 / 3.0, 7.0]]))[1] == pytest.approx(0.4, abs=1e-15)
    assert O.readout(0, I_row, np.array([[0.25, 0], [0.25, 0]]))[1] == pytest.approx(1.0 / 15.0, abs=1e-15)
    # exterior: J = -4 pi I_sigma (R2); full coverage has I_sigma = 1 and |J| = 4 pi (capacitance)
    assert O.readout(1, I_row, np.array([[1.0, 3.0]]))[1] == pytest.approx(-4 * np.pi, abs=1e-14)
