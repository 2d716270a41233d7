"""Pins of the fp64 oracle against what the paper and mathematics fix.

Nothing here compares the oracle with itself or with the CUDA path.  Each
pin is a closed form, a worked example printed in PAPER.md / SPEC.md, an
invariant, or a special case that reduces to a textbook result -- chosen so
that a plausible mistake (dropped term, wrong sign or index, transposed
operand) fails at least one of them.  Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n, 8c-k = SURVEY.md section 8(c) reading k.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from fed_inputs import (BC_CONV, BC_FLUX, BC_RAD, FaceBC, Material, box_problem, cfg3_tensor,
                        make_config, random_field, random_hexes, random_spd_tensor)

GOLD = os.path.join(os.path.dirname(__file__), "golden")

NAT = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)
UNIT = (NAT + 1.0) / 2.0   # unit cube corners in S:93 order


def D33(d6):
    xx, yy, zz, xy, yz, xz = d6
    return np.array([[xx, xy, xz], [xy, yy, yz], [xz, yz, zz]], dtype=np.float64)


# --------------------------------------------------------------------------
# Eq. 17 geometry (SPEC S:136-138 worked examples)
# --------------------------------------------------------------------------

def test_unit_cube_kernel_S136(oracle_lib):
    B, scale, det = oracle.hex_kernel(UNIT)
    assert det == pytest.approx(1 / 8, rel=1e-15)
    assert scale == pytest.approx(1.0, rel=1e-15)
    # B entries are +-1/4 with the sign of the natural coordinate
    np.testing.assert_allclose(B, NAT.T / 4.0, rtol=0, atol=1e-15)


def test_side2_cube_scale_S137(oracle_lib):
    _, scale, det = oracle.hex_kernel(2.0 * UNIT + np.array([3.0, -1.0, 0.5]))
    assert det == pytest.approx(1.0, rel=1e-15)
    assert scale == pytest.approx(8.0, rel=1e-15)


def test_parallelepiped_volume_S162(oracle_lib):
    rng = np.random.default_rng(1)
    for _ in range(20):
        A = np.eye(3) + 0.4 * rng.standard_normal((3, 3))
        if np.linalg.det(A) <= 0.1:
            continue
        x = UNIT @ A.T + rng.standard_normal(3)
        _, scale, _ = oracle.hex_kernel(x)
        assert scale == pytest.approx(np.linalg.det(A), rel=1e-13)


def test_linear_field_gradient_exact_any_hex(oracle_lib):
    """B applied to T = g.x + c gives g exactly on ANY trilinear hex (iso-
    parametric completeness); catches a transposed J^-1."""
    xyz, conn = random_hexes(50, seed=2, distort=0.3)
    rng = np.random.default_rng(3)
    for e in range(conn.shape[0]):
        x8 = xyz[conn[e]]
        B, _, _ = oracle.hex_kernel(x8)
        g = rng.standard_normal(3) * 100
        T = x8 @ g + 7.0
        np.testing.assert_allclose(B @ T, g, rtol=1e-12, atol=1e-10)
        np.testing.assert_allclose(B @ np.ones(8), 0.0, atol=1e-13 * np.abs(B).max())


def test_inverted_hex_rejected(oracle_lib):
    x = UNIT.copy()
    x[:, 2] *= -1.0  # mirror -> negative det J
    with pytest.raises(ValueError):
        oracle.hex_kernel(x)


# --------------------------------------------------------------------------
# Eq. 19/20 element load
# --------------------------------------------------------------------------

def test_element_load_uniform_box_closed_form(oracle_lib):
    """Axis-aligned box hx,hy,hz with diagonal D: the 1-point stiffness is
    K_ab = V sum_i D_ii s_ai s_bi / (16 h_i^2)  (B_ia = s_ai/(4 h_i))."""
    h = np.array([0.3, 0.7, 1.1])
    x = UNIT * h
    d6 = (3.0, 5.0, 11.0, 0, 0, 0)
    B, scale, _ = oracle.hex_kernel(x)
    G = oracle.build_G(B, scale)
    V = h.prod()
    K = np.zeros((8, 8))
    for i in range(3):
        K += V * d6[i] * np.outer(NAT[:, i], NAT[:, i]) / (16 * h[i] ** 2)
    rng = np.random.default_rng(4)
    for _ in range(5):
        Te = rng.uniform(0, 100, 8)
        F = oracle.element_load(B, G, D33(d6), Te)
        np.testing.assert_allclose(F, K @ Te, rtol=1e-13, atol=1e-12)


def test_element_load_rotated_cube_isotropic_closed_form(oracle_lib):
    """Cube of side h rotated arbitrarily, D = k I:
    K_e = (k h / 16)(xi xi^T + eta eta^T + zeta zeta^T)  (SURVEY 8c pins)."""
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    hh, k = 0.25, 42.0
    x = (UNIT * hh) @ Q.T + 1.0
    B, scale, _ = oracle.hex_kernel(x)
    G = oracle.build_G(B, scale)
    K = (k * hh / 16) * sum(np.outer(NAT[:, i], NAT[:, i]) for i in range(3))
    Te = rng.uniform(0, 100, 8)
    F = oracle.element_load(B, G, k * np.eye(3), Te)
    np.testing.assert_allclose(F, K @ Te, rtol=1e-12, atol=1e-11)


def test_element_load_zero_sum_and_symmetry(oracle_lib):
    """sum_a F_e[a] = 0 and the implied K_e = G D B is symmetric
    PSD for SPD D on distorted hexes."""
    xyz, conn = random_hexes(30, seed=6, distort=0.3)
    for e in range(conn.shape[0]):
        B, scale, _ = oracle.hex_kernel(xyz[conn[e]])
        G = oracle.build_G(B, scale)
        D = D33(random_spd_tensor(e))
        K = np.stack([oracle.element_load(B, G, D, np.eye(8)[a]) for a in range(8)], axis=1)
        np.testing.assert_allclose(K, K.T, rtol=0, atol=1e-12 * np.abs(K).max())
        assert np.linalg.eigvalsh(K).min() > -1e-12 * np.abs(K).max()
        np.testing.assert_allclose(K.sum(axis=0), 0.0, atol=1e-12 * np.abs(K).max())
        Te = random_field(8, seed=e)
        F = oracle.element_load(B, G, D, Te)
        assert abs(F.sum()) <= 1e-12 * np.abs(F).sum()
        np.testing.assert_allclose(oracle.element_load(B, G, D, np.full(8, 37.5)), 0.0,
                                   atol=1e-12 * np.abs(K).max() * 37.5)


# --------------------------------------------------------------------------
# lumping, areas, boundary loads (SPEC worked examples)
# --------------------------------------------------------------------------

def test_lumped_mass_unit_hex_S278(oracle_lib):
    p = box_problem(1, 1, 1, L=(1, 1, 1), material=Material(1000.0, 1.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0))
    o = oracle.Oracle(p, 1.0)
    np.testing.assert_allclose(o.mass(), 125.0, rtol=1e-15)


def test_mass_conservation_parallelepiped(oracle_lib):
    A = np.array([[1.0, 0.3, 0.1], [0.0, 0.9, 0.2], [0.1, 0.0, 1.2]])
    p = box_problem(3, 4, 5, L=(1, 1, 1), affine=A, material=Material(7.0, 1.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0))
    o = oracle.Oracle(p, 1.0)
    assert o.mass().sum() == pytest.approx(7.0 * np.linalg.det(A), rel=1e-13)


def test_quad_area_S59(oracle_lib):
    xyz = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 0], [2, 0, 0], [2.5, 3, 0], [0.5, 3, 0]],
                   dtype=np.float64)
    assert oracle.quad_area(xyz, [0, 1, 2, 3]) == pytest.approx(1.0, rel=1e-15)
    assert oracle.quad_area(xyz, [4, 5, 6, 7]) == pytest.approx(6.0, rel=1e-15)   # parallelogram base 2 height 3


def _one_face_problem(side_len, bc, T=37.0):
    mat = Material(1000.0, 1000.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    return box_problem(1, 1, 1, L=(side_len, side_len, side_len), material=mat, side_bc={"z1": 0},
                       face_bcs=[bc], T0=T)


def test_convection_load_S295(oracle_lib):
    """h=200, T_a=0, T=37, nodal area 8.655e-6 m^2 -> -0.0640470 W."""
    a = 8.655e-6
    p = _one_face_problem(math.sqrt(4 * a), FaceBC(BC_CONV, h=200.0, T_inf=0.0))
    o = oracle.Oracle(p, 1.0)
    F, Q = o.loads(np.full(8, 37.0))
    top = p.faces[0]
    np.testing.assert_allclose(Q[top], -0.064047, rtol=1e-12)
    assert np.all(Q[np.setdiff1d(np.arange(8), top)] == 0.0)
    np.testing.assert_allclose(F, 0.0, atol=1e-15)   # uniform T: only round-off


def test_radiation_load_S304(oracle_lib):
    """sigma=5.67e-8, eps=0.66, T_a=-50, T=37, a=3.882e-5 -> -9.84e-3 W."""
    a = 3.882e-5
    p = _one_face_problem(math.sqrt(4 * a), FaceBC(BC_RAD, eps=0.66, T_inf=-50.0))
    o = oracle.Oracle(p, 1.0)
    _, Q = o.loads(np.full(8, 37.0))
    expect = -5.67e-8 * 0.66 * (310.15 ** 4 - 223.15 ** 4) * a
    np.testing.assert_allclose(Q[p.faces[0]], expect, rtol=1e-12)
    assert Q[p.faces[0]][0] == pytest.approx(-9.84e-3, rel=1e-3)


def test_flux_load_trapezoidal(oracle_lib):
    p = _one_face_problem(0.2, FaceBC(BC_FLUX, q=1e5))
    o = oracle.Oracle(p, 1.0)
    _, Q = o.loads(np.full(8, 37.0))
    np.testing.assert_allclose(Q[p.faces[0]], 1e5 * 0.04 / 4, rtol=1e-14)
    assert Q.sum() == pytest.approx(1e5 * 0.04, rel=1e-14)


# --------------------------------------------------------------------------
# critical time step (Eq. 29 / reading 8c-13)
# --------------------------------------------------------------------------

def test_dt_uniform_grid_closed_form(oracle_lib):
    """Uniform isotropic grid: dt_crit = rho c h^2 / (2k)."""
    p = make_config(1, n=3)
    assert oracle.dt_crit(p) == pytest.approx(7800 * 460 * 0.01 / 100.0, rel=1e-13)


def test_dt_element_bound_equals_8x8_eigen(oracle_lib):
    """Closed 3x3 form == literal largest eigenvalue of M_e^-1 K_e (8x8)."""
    xyz, conn = random_hexes(20, seed=8, distort=0.3)
    for e in range(conn.shape[0]):
        d6 = random_spd_tensor(100 + e)
        p = box_problem(1, 1, 1, material=Material(3.0, 5.0, 0.0, d6, 0.0))
        p.xyz = xyz[conn[e]].copy()
        p.conn = np.arange(8, dtype=np.int32).reshape(1, 8)
        lam8 = oracle.element_lambda8(p.xyz, d6, 15.0)
        assert oracle.dt_crit(p) == pytest.approx(2.0 / lam8, rel=1e-11)


def test_dt_equals_global_lambda_max_on_uniform_grid(oracle_lib):
    """Element bound == exact 2/lambda_max(M^-1 K) of the assembled operator
    on a uniform Neumann grid (4 alpha / h^2); K is recovered column by column
    from the matrix-free loads."""
    mat = Material(2.0, 3.0, 0.0, (5.0, 5.0, 5.0, 0, 0, 0), 0.0)
    p = box_problem(4, 4, 4, L=(1, 1, 1), material=mat)
    o = oracle.Oracle(p, 1.0)
    N = p.n_nodes
    K = np.stack([o.loads(np.eye(N)[j])[0] for j in range(N)], axis=1)
    Mc = o.mass() * 3.0
    lam = np.linalg.eigvalsh(K / np.sqrt(np.outer(Mc, Mc))).max()
    h = 0.25
    assert lam == pytest.approx(4 * (5.0 / 6.0) / h ** 2, rel=1e-12)
    assert oracle.dt_crit(p) == pytest.approx(2.0 / lam, rel=1e-12)


def test_dt_td_range_cfg2(oracle_lib):
    """cfg2: crit at 500 degC = 0.065698 s, at 20 degC = 0.085913 s."""
    p = make_config(2, n=2)
    p.xyz *= 0.1 / 64 / (0.1 / 2)    # shrink so that h = 0.1/64
    assert oracle.dt_crit(p, 500.0, 500.0) == pytest.approx(0.065698, rel=2e-5)
    assert oracle.dt_crit(p, 20.0, 20.0) == pytest.approx(0.085913, rel=2e-5)
    assert oracle.dt_crit(p, 20.0, 500.0) == pytest.approx(0.065698, rel=2e-5)


def test_cfg3_tensor_and_dt_conformance(oracle_lib):
    """SURVEY 8c conformance values for the cfg3 generator + dt rule."""
    d = cfg3_tensor()
    ref = (15.690699190744347, 41.62023990177245, 32.68906090748321, 0.13819079029774411,
           -12.790318130525076, 11.742236100126187)
    np.testing.assert_allclose(d, ref, rtol=1e-13)
    assert oracle.sym_max_eig(D33(d)) == pytest.approx(52.0530340009106, rel=1e-12)
    p = make_config(3, n=2)
    p.xyz *= 2.0 / 128
    assert 0.9 * oracle.dt_crit(p) == pytest.approx(0.0189954255352859, rel=1e-12)


def test_stability_boundary(oracle_lib):
    """0.9x the critical step stays bounded, 1.1x diverges (Eq. 28/29)."""
    mat = Material(1.0, 1.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    p = box_problem(5, 5, 5, L=(5, 5, 5), material=mat, T0=lambda x: random_field(x.shape[0], 9))
    dtc = oracle.dt_crit(p)
    assert dtc == pytest.approx(0.5, rel=1e-13)
    good = oracle.Oracle(p, 0.9 * dtc)
    good.step(2000)
    assert np.abs(good.T()).max() <= 100.0 + 1e-9      # maximum principle of the stable scheme
    bad = oracle.Oracle(p, 1.1 * dtc)
    bad.step(2000)
    T = bad.T()
    assert (not np.all(np.isfinite(T))) or np.abs(T).max() > 1e6


# --------------------------------------------------------------------------
# cfg1: exact discrete closed form at every step
# --------------------------------------------------------------------------

def cfg1_closed_form(n, alpha, h, dt, k_steps):
    """1-D lumped chain with Dirichlet 100 at i=0, half mass at i=n:
    T_i^k = 100 + sum_m a_m (1 - dt lam_m)^k sin(kap_m i)."""
    i = np.arange(1, n + 1)
    w = np.ones(n)
    w[-1] = 0.5
    out = np.full(n + 1, 100.0)
    for m in range(1, n + 1):
        kap = (2 * m - 1) * np.pi / (2 * n)
        lam = 4 * alpha / h ** 2 * np.sin(kap / 2) ** 2
        a = (2.0 / n) * np.sum(w * (-100.0) * np.sin(kap * i))
        out[1:] += a * (1 - dt * lam) ** k_steps * np.sin(kap * i)
    return out


def test_cfg1_closed_form_every_column(oracle_lib):
    p = make_config(1)
    n = 10
    dt = 0.9 * oracle.dt_crit(p)
    alpha = 50.0 / (7800 * 460)
    o = oracle.Oracle(p, dt)
    o.step(1)
    T = o.T().reshape(n + 1, n + 1, n + 1)   # [k][j][i]
    assert T[0, 0, 1] == pytest.approx(45.0, abs=1e-12)
    done = 1
    for ks in (10, 100, 500, 2000):
        o.step(ks - done)
        done = ks
        T = o.T().reshape(n + 1, n + 1, n + 1)
        ref = cfg1_closed_form(n, alpha, 0.1, dt, ks)
        err = np.abs(T - ref[None, None, :]).max()
        assert err <= 1.5e-13 * 100, (ks, err)


def test_cfg1_conformance_golden(oracle_lib):
    """Values printed in SURVEY 8c (harness conformance) -- golden fixture."""
    with open(os.path.join(GOLD, "cfg1_closed_form.json")) as f:
        g = json.load(f)
    p = make_config(1)
    dt = 0.9 * oracle.dt_crit(p)
    assert dt == pytest.approx(g["dt"], rel=1e-12)
    o = oracle.Oracle(p, dt)
    done = 0
    for rec in g["checkpoints"]:
        o.step(rec["step"] - done)
        done = rec["step"]
        T = o.T()
        for i, v in zip(rec["i"], rec["T"]):
            assert T[i] == pytest.approx(v, abs=1e-11), (rec["step"], i)


def test_continuous_series_sanity(oracle_lib):
    """Discretisation sanity vs the continuous series solution:
    at step 2000 the field is within 1e-6 of the steady 100 degC."""
    p = make_config(1)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(2000)
    assert np.abs(o.T() - 100.0).max() < 1e-6


def test_sine_decay_S498(oracle_lib):
    """Bar with zero ends and sin initial field, alpha = 1e-4, L = 0.1: the
    midpoint decays by exp(-pi^2 alpha t / L^2) = 0.372708 at t = 10 s
    within 2 % (SPEC acceptance 5)."""
    n = 40
    L = 0.1
    mat = Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.0)
    p = box_problem(n, 1, 1, L=(L, L / n, L / n), material=mat, dirichlet={"x0": 0.0, "x1": 0.0},
                    T0=lambda x: np.sin(np.pi * x[:, 0] / L))
    dtc = oracle.dt_crit(p)
    nsteps = int(math.ceil(10.0 / (0.5 * dtc)))
    dt = 10.0 / nsteps
    o = oracle.Oracle(p, dt)
    o.step(nsteps)
    T = o.T().reshape(2, 2, n + 1)
    assert T[0, 0, n // 2] == pytest.approx(math.exp(-math.pi ** 2 / 10), rel=0.02)
    assert math.exp(-math.pi ** 2 / 10) == pytest.approx(0.372708, rel=1e-6)


# --------------------------------------------------------------------------
# steady states (patch test P:226-236, Kirchhoff, flux+convection/radiation)
# --------------------------------------------------------------------------

def _lin(x):
    return 200 * x[:, 0] + 100 * x[:, 1] + 200 * x[:, 2]


@pytest.mark.parametrize("affine", [None, [[1.0, 0.25, 0.1], [0.0, 0.9, -0.2], [0.15, 0.0, 1.1]]])
def test_patch_test_parallelepiped(oracle_lib, affine):
    """Linear T is reproduced exactly: zero interior load and the Dirichlet-
    pinned steady field equals T = 200x+100y+200z."""
    mat = Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.0)
    sides = {s: _lin for s in ("x0", "x1", "y0", "y1", "z0", "z1")}
    p = box_problem(4, 4, 4, material=mat, dirichlet=sides, T0=0.0,
                    affine=None if affine is None else np.array(affine))
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    T_lin = _lin(p.xyz)
    F, _ = o.loads(T_lin)
    interior = np.setdiff1d(np.arange(p.n_nodes), p.dir_nodes)
    assert np.abs(F[interior]).max() <= 1e-12 * np.abs(T_lin).max() * 200
    o.step(3000)
    assert np.abs(o.T() - T_lin).max() <= 1e-10 * np.abs(T_lin).max()


def test_patch_test_jittered_reports_method_limit(oracle_lib):
    """Jittered hexes: the 1-point element does not pass exactly (SURVEY V5,
    paper's own 1.7e-3 hex error P:228).  Report-only bound."""
    mat = Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.0)
    sides = {s: _lin for s in ("x0", "x1", "y0", "y1", "z0", "z1")}
    p = box_problem(4, 4, 4, material=mat, dirichlet=sides, T0=0.0, jitter=0.2, seed=7)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    F, _ = o.loads(_lin(p.xyz))
    interior = np.setdiff1d(np.arange(p.n_nodes), p.dir_nodes)
    assert np.abs(F[interior]).max() > 1e-3      # genuinely non-zero
    o.step(4000)
    err = np.abs(o.T() - _lin(p.xyz)).max()
    assert 1e-4 < err < 20.0


def test_kirchhoff_td_steady_state(oracle_lib):
    """TD conductivity k = 50(1+0.002 T), Dirichlet 500 / 20 on x = 0 / L,
    adiabatic elsewhere: nodal Phi(T) = T + beta T^2/2 is exactly linear in x
    at steady state -- pins the nodal-average rule of P:301."""
    beta = 0.002
    mat = Material(7800.0, 460.0, 0.001, (50.0, 50.0, 50.0, 0, 0, 0), beta)
    L = 0.08
    p = box_problem(8, 8, 8, L=(L, L, L), material=mat, dirichlet={"x0": 500.0, "x1": 20.0}, T0=20.0)
    dt = 0.9 * oracle.dt_crit(p, 20.0, 500.0)
    o = oracle.Oracle(p, dt)
    o.step(6000)
    T = o.T()
    x = p.xyz[:, 0]
    phi = T + beta * T ** 2 / 2
    phi_ref = (500 + beta * 500 ** 2 / 2) + ((20 + beta * 20 ** 2 / 2) - (500 + beta * 500 ** 2 / 2)) * x / L
    assert np.abs(phi - phi_ref).max() <= 1e-11 * 750


def test_flux_convection_steady_1d(oracle_lib):
    """Column, flux q on z=0, convection (h, T_inf) on z=L, adiabatic sides:
    T(z) = T_inf + q/h + q (L - z)/k at the nodes."""
    q, hc, Tinf, k = 1e5, 500.0, 20.0, 50.0
    L = 0.1
    mat = Material(1.0, 3.6e6, 0.0, (k, k, k, 0, 0, 0), 0.0)
    p = box_problem(1, 1, 8, L=(0.0125, 0.0125, L), material=mat, side_bc={"z0": 0, "z1": 1},
                    face_bcs=[FaceBC(BC_FLUX, q=q), FaceBC(BC_CONV, h=hc, T_inf=Tinf)], T0=20.0)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(8000)
    z = p.xyz[:, 2]
    ref = Tinf + q / hc + q * (L - z) / k
    assert np.abs(o.T() - ref).max() <= 1e-10 * ref.max()


def test_flux_radiation_steady_bisection_S595(oracle_lib):
    """Column with flux q in at z=0 and radiation out at z=L: the top
    temperature is the root of sigma eps [(T-T_z)^4 - (T_a-T_z)^4] = q found
    by bisection (SPEC acceptance 8), and T(z) = T_top + q (L-z)/k."""
    q, eps, Ta, k = 1e5, 0.8, 20.0, 50.0
    L = 0.1
    mat = Material(1.0, 3.6e6, 0.0, (k, k, k, 0, 0, 0), 0.0)
    p = box_problem(1, 1, 4, L=(0.025, 0.025, L), material=mat, side_bc={"z0": 0, "z1": 1},
                    face_bcs=[FaceBC(BC_FLUX, q=q), FaceBC(BC_RAD, eps=eps, T_inf=Ta)], T0=900.0)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(20000)
    lo, hi = Ta, 5000.0
    f = lambda T: 5.67e-8 * eps * ((T + 273.15) ** 4 - (Ta + 273.15) ** 4) - q
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(mid) > 0:
            hi = mid
        else:
            lo = mid
    Ttop = 0.5 * (lo + hi)
    z = p.xyz[:, 2]
    ref = Ttop + q * (L - z) / k
    assert np.abs(o.T() - ref).max() <= 1e-6


# --------------------------------------------------------------------------
# invariants
# --------------------------------------------------------------------------

def test_adiabatic_conservation_S418(oracle_lib):
    """No BC, no Dirichlet, TI: sum M c T is constant (SPEC acceptance 10)."""
    mat = Material(1000.0, 2000.0, 0.0, random_spd_tensor(3, 50, 300), 0.0)
    p = box_problem(5, 4, 3, material=mat, jitter=0.15, seed=4, T0=lambda x: random_field(x.shape[0], 5))
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    M = o.mass()
    e0 = (M * 2000 * o.T()).sum()
    o.step(1000)
    e1 = (M * 2000 * o.T()).sum()
    assert abs(e1 - e0) <= 1e-12 * abs(e0)


def test_energy_identity_per_step_td(oracle_lib):
    """sum_free M c(T^k)(T^{k+1}-T^k) = dt sum_free (Q - F) and sum F = 0."""
    mat = Material(7800.0, 460.0, 0.001, (50.0, 40.0, 30.0, 5.0, 2.0, 1.0), 0.002)
    bcs = [FaceBC(BC_FLUX, q=1e4), FaceBC(BC_CONV, h=25.0, T_inf=20.0), FaceBC(BC_RAD, eps=0.5, T_inf=10.0)]
    p = box_problem(4, 3, 5, L=(0.1, 0.1, 0.1), material=mat, side_bc={"z0": 0, "x1": 1, "y1": 2},
                    face_bcs=bcs, dirichlet={"x0": 50.0}, T0=lambda x: 20 + random_field(x.shape[0], 6, 0, 60),
                    q_vol=lambda x: 1e6 * np.ones(x.shape[0]), jitter=0.1, seed=2)
    dt = 0.5 * oracle.dt_crit(p, 0.0, 200.0)
    o = oracle.Oracle(p, dt)
    M = o.mass()
    free = np.ones(p.n_nodes, bool)
    free[p.dir_nodes] = False
    for _ in range(3):
        T0 = o.T()
        F, Q = o.loads(T0)
        assert abs(F.sum()) <= 1e-11 * np.abs(F).sum()
        o.step(1)
        T1 = o.T()
        lhs = (M * 460 * (1 + 0.001 * T0) * (T1 - T0))[free].sum()
        rhs = dt * (Q - F)[free].sum()
        assert lhs == pytest.approx(rhs, rel=1e-10)
        np.testing.assert_array_equal(T1[p.dir_nodes], 50.0)


def test_symmetry_cfg2_like(oracle_lib):
    """cfg2 is symmetric under x<->y, x->L-x, y->L-y."""
    n = 6
    p = make_config(2, n=n, steps=50)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(50)
    T = o.T().reshape(n + 1, n + 1, n + 1)
    s = np.abs(T).max()
    assert np.abs(T - T.transpose(0, 2, 1)).max() <= 1e-13 * s
    assert np.abs(T - T[:, :, ::-1]).max() <= 1e-13 * s
    assert np.abs(T - T[:, ::-1, :]).max() <= 1e-13 * s


def test_permutation_invariance(oracle_lib):
    """Renumbering nodes and elements does not change the physics."""
    mat = Material(7800.0, 460.0, 0.001, (50.0, 50.0, 50.0, 0, 0, 0), 0.002)
    kw = dict(L=(0.1, 0.1, 0.1), material=mat, side_bc={s: 0 for s in ("x0", "x1", "y0", "y1", "z0", "z1")},
              face_bcs=[FaceBC(BC_CONV, h=50.0, T_inf=20.0)],
              T0=lambda x: 20 + 80 * np.sin(np.pi * x[:, 0] / 0.1) * np.sin(np.pi * x[:, 1] / 0.1),
              jitter=0.2, seed=7)
    a = box_problem(5, 5, 5, **kw)
    b = box_problem(5, 5, 5, shuffle_seed=11, **kw)
    assert oracle.dt_crit(b, 20.0, 100.0) == oracle.dt_crit(a, 20.0, 100.0)
    dt = 0.9 * oracle.dt_crit(a, 20.0, 100.0)
    oa, ob = oracle.Oracle(a, dt), oracle.Oracle(b, dt)
    oa.step(100)
    ob.step(100)
    Ta, Tb = oa.T(), ob.T()
    perm = b.meta["node_perm"]
    assert np.abs(Tb - Ta[perm]).max() <= 1e-12 * np.abs(Ta).max()


def test_cfg2_flux_heats_convection_cools(oracle_lib):
    """Sign reading 8c-11: flux raises T, convection pulls toward T_inf."""
    p = make_config(2, n=4, steps=20)
    o = oracle.Oracle(p, 0.9 * oracle.dt_crit(p))
    o.step(20)
    T = o.T().reshape(5, 5, 5)
    assert T[0].mean() > 20.0 and T[0].mean() > T[-1].mean()


def test_cfg4_generator_and_dt_conformance(oracle_lib):
    """cfg4 jitter recipe (seed 7) + element-bound dt over [20,100] on the full
    256^3 mesh: 1.75477136965634e-3 s (SURVEY 8c conformance, V11)."""
    p = make_config(4, renumber=False)
    assert oracle.dt_crit(p, 20.0, 100.0) == pytest.approx(1.75477136965634e-3, rel=1e-12)
