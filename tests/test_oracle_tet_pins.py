"""Pins of the oracle's tet4 branch (Eq. 18; NEXT-1) against what
the paper, SPEC's worked examples and mathematics fix.  Linear tetrahedra
reproduce linear fields exactly on ANY mesh, which gives exact pins that the
hex element only has on parallelepipeds."""
import numpy as np
import pytest

import oracle
from fed_inputs import (BC_CONV, BC_FLUX, FaceBC, Material, random_field, random_spd_tensor, tet_box_problem,
                        paper_tet_problem)

REF = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)


def D33(d6):
    xx, yy, zz, xy, yz, xz = d6
    return np.array([[xx, xy, xz], [xy, yy, yz], [xz, yz, zz]], dtype=np.float64)


def test_reference_tet_S127(oracle_lib):
    B, V = oracle.tet_kernel(REF)
    assert V == pytest.approx(1 / 6, rel=1e-15)
    np.testing.assert_allclose(B.T, [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], atol=1e-15)
    B2, V2 = oracle.tet_kernel(REF + 5.0)                 # translation invariance
    np.testing.assert_allclose(B2, B, atol=1e-13)
    B3, V3 = oracle.tet_kernel(2.0 * REF)                 # similarity scaling
    assert V3 == pytest.approx(8 * V, rel=1e-14)
    np.testing.assert_allclose(B3, 0.5 * B, atol=1e-15)


def test_tet_element_load_S155(oracle_lib):
    """D = 200 I, T = x on the reference tet: F_int = V B^T D B T = (-200/6, +200/6, 0, 0)
    (SPEC S:155 prints the negated load under its sign convention; reading R1)."""
    B, V = oracle.tet_kernel(REF)
    G = oracle.build_G_n(B, V)
    F = oracle.element_load_n(B, G, 200.0 * np.eye(3), np.array([0.0, 1.0, 0.0, 0.0]))
    np.testing.assert_allclose(F, [-200 / 6, 200 / 6, 0, 0], rtol=1e-14, atol=1e-13)


def _random_tets(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        x = rng.standard_normal((4, 3))
        if np.linalg.det(x[1:] - x[0]) > 0.2:
            out.append(x)
    return out


def test_tet_linear_field_exact_and_invariants(oracle_lib):
    rng = np.random.default_rng(3)
    for k, x in enumerate(_random_tets(30, 4)):
        B, V = oracle.tet_kernel(x)
        assert V == pytest.approx(np.linalg.det(x[1:] - x[0]) / 6, rel=1e-12)
        g = rng.standard_normal(3)
        np.testing.assert_allclose(B @ (x @ g + 3.0), g, rtol=1e-11, atol=1e-11)
        G = oracle.build_G_n(B, V)
        D = D33(random_spd_tensor(k))
        K = np.stack([oracle.element_load_n(B, G, D, np.eye(4)[a]) for a in range(4)], axis=1)
        np.testing.assert_allclose(K, K.T, atol=1e-12 * np.abs(K).max())
        assert np.linalg.eigvalsh(K).min() > -1e-12 * np.abs(K).max()
        np.testing.assert_allclose(K.sum(axis=0), 0, atol=1e-12 * np.abs(K).max())


def test_inverted_tet_rejected(oracle_lib):
    with pytest.raises(ValueError):
        oracle.tet_kernel(REF[[1, 0, 2, 3]])


def test_kuhn_mesh_mass_and_area(oracle_lib):
    mat = Material(7.0, 1.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0)
    p = tet_box_problem(3, 4, 2, L=(0.3, 0.4, 0.2), material=mat, side_bc={s: 0 for s in ("x0", "x1", "y0", "y1", "z0", "z1")},
                        face_bcs=[FaceBC(BC_FLUX, q=1.0)])
    assert p.n_elems == 6 * 24
    o = oracle.Oracle(p, 1.0)
    assert o.mass().sum() == pytest.approx(7.0 * 0.3 * 0.4 * 0.2, rel=1e-13)
    _, Q = o.loads(np.zeros(p.n_nodes))
    area = 2 * (0.3 * 0.4 + 0.3 * 0.2 + 0.4 * 0.2)
    assert Q.sum() == pytest.approx(area, rel=1e-13)         # flux q = 1 W/m^2 over the whole surface


@pytest.mark.parametrize("jitter", [0.0, 0.25])
def test_tet_patch_test_exact_any_mesh(oracle_lib, jitter):
    """P:228 patch test with tets: T = 200x+100y+200z pinned on the boundary is
    reproduced exactly in the interior, also on a distorted mesh."""
    mat = Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.0)
    lin = lambda x: 200 * x[:, 0] + 100 * x[:, 1] + 200 * x[:, 2]
    p = tet_box_problem(4, 4, 4, material=mat, dirichlet={s: lin for s in ("x0", "x1", "y0", "y1", "z0", "z1")},
                        T0=0.0, jitter=jitter, seed=7)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    Tl = lin(p.xyz)
    F, _ = o.loads(Tl)
    inner = np.setdiff1d(np.arange(p.n_nodes), p.dir_nodes)
    assert np.abs(F[inner]).max() <= 1e-10 * 200 * np.abs(Tl).max()
    o.step(6000)
    assert np.abs(o.T() - Tl).max() <= 1e-9 * np.abs(Tl).max()


def test_tet_dt_bound_is_conservative(oracle_lib):
    """Element bound >= exact global lambda_max (so dt_crit <= exact), and a run
    at 1.05x the EXACT global critical step diverges."""
    mat = Material(1.0, 1.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    p = tet_box_problem(3, 3, 3, L=(3, 3, 3), material=mat, T0=lambda x: random_field(x.shape[0], 2))
    o = oracle.Oracle(p, 1.0)
    N = p.n_nodes
    K = np.stack([o.loads(np.eye(N)[j])[0] for j in range(N)], axis=1)
    M = o.mass()
    lam = np.linalg.eigvalsh(K / np.sqrt(np.outer(M, M))).max()
    dtc = oracle.dt_crit(p)
    assert dtc <= 2.0 / lam * (1 + 1e-12)
    assert dtc >= 0.2 * 2.0 / lam                           # and not absurdly conservative
    bad = oracle.Oracle(p, 1.05 * 2.0 / lam)
    bad.step(3000)
    T = bad.T()
    assert (not np.isfinite(T).all()) or np.abs(T).max() > 1e3


def test_tet_lambda_matches_closed_form(oracle_lib):
    """Literal 4x4 element eigenvalue vs the closed form 4 lambda_max(L^T P L)/(rho c V)
    with P = V J^-T D J^-1 and L L^T = S S^T = I + 11^T."""
    for k, x in enumerate(_random_tets(10, 9)):
        d6 = random_spd_tensor(50 + k)
        J = x[1:] - x[0]
        Ji = np.linalg.inv(J)
        V = np.linalg.det(J) / 6
        P = V * Ji.T @ D33(d6) @ Ji
        L = np.linalg.cholesky(np.eye(3) + np.ones((3, 3)))
        lam = 4 * np.linalg.eigvalsh(L.T @ P @ L).max() / (3.0 * V)
        assert oracle.tet_lambda(x, d6, 3.0) == pytest.approx(lam, rel=1e-11)


def test_tet_flux_convection_steady_exact(oracle_lib):
    q, hc, Tinf, k = 1e5, 500.0, 20.0, 50.0
    mat = Material(1.0, 3.6e6, 0.0, (k, k, k, 0, 0, 0), 0.0)
    p = tet_box_problem(1, 1, 6, L=(0.02, 0.02, 0.1), material=mat, side_bc={"z0": 0, "z1": 1},
                        face_bcs=[FaceBC(BC_FLUX, q=q), FaceBC(BC_CONV, h=hc, T_inf=Tinf)], T0=20.0, jitter=0.0)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(30000)
    ref = Tinf + q / hc + q * (0.1 - p.xyz[:, 2]) / k
    assert np.abs(o.T() - ref).max() <= 1e-9 * ref.max()


def test_paper_tet_workload_shape(oracle_lib):
    p = paper_tet_problem()
    assert p.n_elems == 41154 and p.n_nodes == 8000          # vs 40 021 / 7 872 in P:357
    assert p.nodes_per_face == 3
