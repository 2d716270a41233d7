"""Pins of the oracle's "concentrated" boundary loads (NEXT-3; the paper's
convention in Secs. 4.3/4.4, "calculating the sum of convection surface
areas ... dividing by the number of nodes")."""
import math

import numpy as np
import pytest

import oracle
from fed_inputs import BC_CONV, BC_FLUX, FaceBC, Material, box_problem

MAT = Material(1000.0, 1000.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)


def _faces_problem(nx, ny, bc):
    """nx x ny x 1 box, BC on the top side (z = 1): nx*ny unit quads."""
    return box_problem(nx, ny, 1, L=(nx, ny, 1.0), material=MAT, side_bc={"z1": 0}, face_bcs=[bc], T0=37.0)


def test_one_quad_S71(oracle_lib):
    p = _faces_problem(1, 1, FaceBC(BC_FLUX, q=1.0, area_mode=1))
    _, Q = oracle.Oracle(p, 1.0).loads(np.full(p.n_nodes, 37.0))
    np.testing.assert_allclose(Q[p.faces[0]], 0.25, rtol=1e-15)          # 1.0 / 4 nodes


def test_two_quads_S72(oracle_lib):
    p = _faces_problem(2, 1, FaceBC(BC_FLUX, q=1.0, area_mode=1))
    _, Q = oracle.Oracle(p, 1.0).loads(np.full(p.n_nodes, 37.0))
    top = np.unique(p.faces)
    assert top.size == 6
    np.testing.assert_allclose(Q[top], 2.0 / 6.0, rtol=1e-14)              # 2.0 / 6 unique nodes
    # per-face tributary mode: shared-edge nodes 0.5, corners 0.25 (R9)
    q = _faces_problem(2, 1, FaceBC(BC_FLUX, q=1.0, area_mode=0))
    _, Q0 = oracle.Oracle(q, 1.0).loads(np.full(q.n_nodes, 37.0))
    assert sorted(np.round(Q0[top], 12)) == [0.25, 0.25, 0.25, 0.25, 0.5, 0.5]


@pytest.mark.parametrize("n", [3, 7])
def test_uniform_area_times_count_is_total_area_S77(oracle_lib, n):
    p = _faces_problem(n, n + 1, FaceBC(BC_FLUX, q=2.5, area_mode=1))
    _, Q = oracle.Oracle(p, 1.0).loads(np.full(p.n_nodes, 37.0))
    top = np.unique(p.faces)
    assert top.size == (n + 1) * (n + 2)
    np.testing.assert_allclose(Q[top], 2.5 * n * (n + 1) / top.size, rtol=1e-13)
    assert Q.sum() == pytest.approx(2.5 * n * (n + 1), rel=1e-13)


def test_fin_cooler_nodal_area_S295(oracle_lib):
    """h = 200, T_a = 0, T = 37 with the paper's uniform nodal area 8.655e-6 m^2
     gives -0.0640470 W per node."""
    a = 8.655e-6
    s = math.sqrt(2 * 3 * a / 2)       # 2 x 1 quads of side s: area 2 s^2 over 6 nodes = a
    p = box_problem(2, 1, 1, L=(2 * s, s, s), material=MAT, side_bc={"z1": 0},
                    face_bcs=[FaceBC(BC_CONV, h=200.0, T_inf=0.0, area_mode=1)], T0=37.0)
    _, Q = oracle.Oracle(p, 1.0).loads(np.full(p.n_nodes, 37.0))
    np.testing.assert_allclose(Q[np.unique(p.faces)], -0.064047, rtol=1e-12)
