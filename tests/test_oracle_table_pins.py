"""Pins of the oracle's tabulated-property branch (NEXT-2; "a linear
interpolation between points is employed", P:301 nodal evaluation then
element average; SPEC S:197-231 worked examples)."""
import numpy as np
import pytest

import oracle
from fed_inputs import Material, box_problem, paper_td_material, tet_box_problem

KT = ((37.0, 337.0), (200.0, 2000.0))
CT = ((37.0, 337.0), (2000.0, 8000.0))


def test_table_eval_S203():
    assert oracle.table_eval(*KT, 37.0) == 200.0
    assert oracle.table_eval(*KT, 38.0) == pytest.approx(206.0, rel=1e-15)   # S:204 (6 per degC)
    assert oracle.table_eval(*KT, 400.0) == 2000.0          # S:205 clamped
    assert oracle.table_eval(*KT, -50.0) == 200.0           # clamped below
    assert oracle.table_eval((5.0,), (7.5,), 123.0) == 7.5  # single row -> constant


def test_c_table_S229():
    assert oracle.table_eval(*CT, 37.0) == 2000.0
    assert oracle.table_eval(*CT, 337.0) == 8000.0
    assert oracle.table_eval(*CT, 87.0) == pytest.approx(3000.0, rel=1e-15)


def test_midpoint_property_S234():
    Tt, vt = (0.0, 10.0, 30.0, 35.0), (1.0, 4.0, -2.0, 9.0)
    for i in range(3):
        mid = 0.5 * (Tt[i] + Tt[i + 1])
        assert oracle.table_eval(Tt, vt, mid) == pytest.approx(0.5 * (vt[i] + vt[i + 1]), rel=1e-13)


def test_element_conductivity_average_S222(oracle_lib):
    """Reference tet with nodes at (37, 37, 337, 337): element k = mean of the
    nodal table values = 1100, so F = V * 1100 * B^T B T with the
    textbook reference-tet gradients."""
    mat = Material(1000.0, 2000.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0, k_table=KT)
    p = tet_box_problem(1, 1, 1, material=mat)
    p.xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    p.conn = np.array([[0, 1, 2, 3]], dtype=np.int32)
    p.faces = np.zeros((0, 3), np.int32)
    p.face_bc = np.zeros(0, np.int32)
    p.dir_nodes = np.zeros(0, np.int32)
    p.dir_T = np.zeros(0)
    p.T0 = np.zeros(4)
    o = oracle.Oracle(p, 1.0)
    T = np.array([37.0, 37.0, 337.0, 337.0])
    F, _ = o.loads(T)
    B = np.array([[-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1]], dtype=np.float64)
    np.testing.assert_allclose(F, (1 / 6) * 1100.0 * B.T @ B @ T, rtol=1e-13)


def test_steady_flux_is_constant_with_nonlinear_table(oracle_lib):
    """1-D column, Dirichlet at both ends, a k table with a kink inside the
    temperature range: at steady state the discrete flux
    (k(T_i)+k(T_i+1))/2 (T_i+1 - T_i)/h is the same between every pair of
    node planes (conservation), and it is NOT the linear profile."""
    kt = ((0.0, 60.0, 100.0), (50.0, 150.0, 60.0))
    ct = ((0.0, 100.0), (400.0, 600.0))
    mat = Material(7800.0, 460.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0, k_table=kt, c_table=ct)
    n, L = 10, 0.05
    p = box_problem(1, 1, n, L=(0.005, 0.005, L), material=mat, dirichlet={"z0": 100.0, "z1": 0.0}, T0=50.0)
    dt = 0.9 * oracle.dt_crit(p, 0.0, 100.0)
    o = oracle.Oracle(p, dt)
    o.step(40000)
    T = o.T().reshape(n + 1, 2, 2)[:, 0, 0]
    h = L / n
    k = np.array([oracle.table_eval(*kt, t) for t in T])
    q = 0.5 * (k[1:] + k[:-1]) * (T[1:] - T[:-1]) / h
    assert np.abs(q - q.mean()).max() <= 1e-9 * np.abs(q).max()
    assert np.abs(T - np.linspace(100, 0, n + 1)).max() > 1.0


def test_dt_crit_with_tables_checks_breakpoints(oracle_lib):
    """Uniform grid: dt_crit = rho c(T*) h^2 / (2 k(T*)) at the worst T* in
    [T_lo, T_hi]; with a k peak at an interior breakpoint T* is that breakpoint."""
    kt = ((0.0, 50.0, 100.0), (1.0, 3.0, 1.0))
    mat = Material(2.0, 5.0, 0.0, (10.0, 10.0, 10.0, 0, 0, 0), 0.0, k_table=kt)
    p = box_problem(3, 3, 3, L=(0.3, 0.3, 0.3), material=mat)
    h = 0.1
    assert oracle.dt_crit(p, 0.0, 100.0) == pytest.approx(2.0 * 5.0 * h * h / (2 * 10.0 * 3.0), rel=1e-12)
    assert oracle.dt_crit(p, 60.0, 100.0) == pytest.approx(2.0 * 5.0 * h * h / (2 * 10.0 * 2.6), rel=1e-12)
    pm = paper_td_material()
    q = box_problem(2, 2, 2, L=(0.2, 0.2, 0.2), material=pm)
    # paper's tables on [37, 137]: k/c = 0.1 at 37, 800/4000 = 0.2 at 137 -> worst at 137
    assert oracle.dt_crit(q, 37.0, 137.0) == pytest.approx(1000.0 * 4000.0 * 0.01 / (2 * 800.0), rel=1e-12)
