"""Pins of the oracle's volumetric source term Q_vol,n = q_vol(x_n) V_n.

The source Q enters the strong form (Eq. 1) and the semi-discrete
system C dT/dt + K T = Q; the oracle lumps it by nodal quadrature
with the same equal-split volumes as the capacity (reading R3 / SURVEY 8c-16:
Q_vol,n = s(x_n) V_n, V_n = sum over the node's elements of 8 det J_e / 8).
Every expected value here is a closed form in the mesh parameters or a
textbook integral -- never a value read back from the oracle -- chosen so that
a dropped multiply, V_n replaced by M_n = rho V_n, a wrong node index or a
missing element share fails at least one pin.

`Oracle.loads(T)` returns (F_int, Q) at a field T; with no face loads (or with
T equal to the ambient temperature of every convection face) Q is the source
term alone.
"""
import math

import numpy as np
import pytest

import oracle
from fed_inputs import BC_CONV, FaceBC, Material, box_problem, make_config

RHO = 7.0   # != 1, so V_n and M_n = rho V_n cannot be confused


def _incident_elements(nx, ny, nz):
    """Number of hex elements touching each node of an nx x ny x nz grid
    (natural x-fastest numbering): product over the axes of 1 at an end, 2 inside."""
    def f(n):
        c = np.full(n + 1, 2.0)
        c[0] = c[-1] = 1.0
        return c
    cx, cy, cz = f(nx), f(ny), f(nz)
    return (cz[:, None, None] * cy[None, :, None] * cx[None, None, :]).ravel()


def _source_only(prob, T=0.0):
    o = oracle.Oracle(prob, 1.0)
    _, Q = o.loads(np.full(prob.n_nodes, T))
    return Q


def test_uniform_source_affine_box_per_node(oracle_lib):
    """Uniform q on an affine (parallelepiped) grid: every element has volume
    |det A| hx hy hz, so Q_n = q |det A| hx hy hz (#elements at n) / 8 exactly."""
    A = np.array([[1.0, 0.3, 0.1], [0.0, 0.9, 0.2], [0.1, 0.0, 1.2]])
    nx, ny, nz, L = 3, 4, 5, (0.3, 0.2, 0.5)
    q = 2.5e6
    mat = Material(RHO, 460.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0)
    p = box_problem(nx, ny, nz, L=L, affine=A, material=mat, q_vol=lambda x: np.full(x.shape[0], q))
    Q = _source_only(p)
    ve = np.linalg.det(A) * (L[0] / nx) * (L[1] / ny) * (L[2] / nz)
    exp = q * ve * _incident_elements(nx, ny, nz) / 8.0
    np.testing.assert_allclose(Q, exp, rtol=1e-13, atol=0)
    # total power = q x box volume (closed form)
    assert Q.sum() == pytest.approx(q * np.linalg.det(A) * L[0] * L[1] * L[2], rel=1e-13)


def test_linear_source_integrated_exactly(oracle_lib):
    """Nodal quadrature with equal-split volumes integrates a LINEAR density
    exactly on a parallelepiped grid (the mean of an element's corner values of
    a linear function is its centroid value): sum_n Q_n = Vol q(centroid)."""
    A = np.array([[1.1, 0.2, 0.0], [0.1, 0.8, -0.3], [0.0, 0.2, 1.0]])
    nx, ny, nz, L = 5, 3, 4, (0.5, 0.3, 0.4)
    a, b = 3.0e5, np.array([2.0e6, -1.5e6, 4.0e6])
    mat = Material(RHO, 460.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0)
    p = box_problem(nx, ny, nz, L=L, affine=A, material=mat, q_vol=lambda x: a + x @ b)
    Q = _source_only(p)
    vol = np.linalg.det(A) * L[0] * L[1] * L[2]
    centroid = A @ (0.5 * np.array(L))
    assert Q.sum() == pytest.approx(vol * (a + centroid @ b), rel=1e-13)
    # and it is node-local: a source on one node only loads that node
    qv = np.zeros(p.n_nodes)
    qv[17] = 1.0e6
    p1 = box_problem(nx, ny, nz, L=L, affine=A, material=mat, q_vol=qv)
    Q1 = _source_only(p1)
    assert np.count_nonzero(Q1) == 1 and Q1[17] > 0


def test_uniform_source_proportional_to_lumped_mass_any_mesh(oracle_lib):
    """On ANY mesh (jittered, renumbered), a uniform density gives
    Q_n = (q / rho) M_n: the source uses the same lumped volume as the capacity
    (R3), and M_n itself is pinned by the S:278 worked example and by exact
    mass conservation on parallelepipeds (test_oracle_pins.py)."""
    q = 4.0e5
    mat = Material(RHO, 460.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0)
    p = box_problem(6, 5, 4, L=(0.06, 0.05, 0.04), material=mat, jitter=0.2, seed=3, shuffle_seed=8,
                    q_vol=lambda x: np.full(x.shape[0], q))
    o = oracle.Oracle(p, 1.0)
    _, Q = o.loads(np.zeros(p.n_nodes))
    np.testing.assert_allclose(Q, (q / RHO) * o.mass(), rtol=1e-14, atol=0)


def test_source_adds_to_face_loads(oracle_lib):
    """Q_n = Q_vol,n + face loads: with a convection face away from T_inf the two
    terms add (the convection part is pinned in test_oracle_pins.py)."""
    q = 1.0e6
    mat = Material(RHO, 460.0, 0.0, (1, 1, 1, 0, 0, 0), 0.0)
    kw = dict(L=(0.2, 0.2, 0.2), material=mat, q_vol=lambda x: np.full(x.shape[0], q))
    p_src = box_problem(2, 2, 2, **kw)
    p_both = box_problem(2, 2, 2, side_bc={"z1": 0}, face_bcs=[FaceBC(BC_CONV, h=30.0, T_inf=15.0)], **kw)
    p_conv = box_problem(2, 2, 2, L=(0.2, 0.2, 0.2), material=mat, side_bc={"z1": 0},
                         face_bcs=[FaceBC(BC_CONV, h=30.0, T_inf=15.0)])
    T = 40.0
    np.testing.assert_allclose(_source_only(p_both, T), _source_only(p_src, T) + _source_only(p_conv, T),
                               rtol=1e-14, atol=1e-9)
    # top-face nodes lose h (T - T_inf) x (their tributary area) on top of the source
    top = np.isclose(p_both.xyz[:, 2], 0.2)
    Qc = _source_only(p_conv, T)
    assert Qc[top].sum() == pytest.approx(-30.0 * (T - 15.0) * 0.04, rel=1e-13)


def test_cfg5_total_source_power(oracle_lib):
    """cfg5's Gaussian source (1e8 W/m^3 peak, sigma = 0.01 m at
    the centre of the 0.1 m cube) at n = 64: the total nodal source power equals
    the integral of the density over the cube,
        1e8 (2 pi)^{3/2} sigma^3 erf(L / (2 sqrt(2) sigma))^3 = 1574.96 W.
    The nodal quadrature is the tensor trapezoidal rule here (uniform grid,
    equal split); for a Gaussian with sigma / h = 6.4 its aliasing error is
    ~exp(-2 pi^2 (sigma/h)^2) and its end corrections scale with the density's
    derivatives on the faces (~exp(-12.5) of the peak), both far below the
    2e-6 tolerance used (SURVEY 8c-16's "1 575 W")."""
    p = make_config(5, n=64)
    Q = _source_only(p, T=20.0)     # T = T_inf: the convection faces carry no load
    sig, L = 0.01, 0.1
    exact = 1e8 * (2 * math.pi) ** 1.5 * sig ** 3 * math.erf(L / (2 * math.sqrt(2) * sig)) ** 3
    assert exact == pytest.approx(1574.96, abs=0.01)
    assert Q.sum() == pytest.approx(exact, rel=2e-6)
    # peak node: the cube centre (n even) carries q_peak x h^3
    h = L / 64
    c = np.argmin(((p.xyz - 0.05) ** 2).sum(axis=1))
    assert Q[c] == pytest.approx(1e8 * h ** 3, rel=1e-12)
