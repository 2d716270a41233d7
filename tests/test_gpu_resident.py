"""GPU parity of resident mode (fed_options.resident): one cooperative launch per
fed_step call, chunks ordered by per-chunk dataflow, shared-node updates recomputed
by every touching chunk, last step finalised by the node kernel.  Results must
match the fp64 oracle within the north_star tolerances (reading 8c-19) and the
streaming (per-step launch) path; calls of 1, 2, 3 ... steps exercise the
step % 3 rotation of the partial-load buffers and the finalize pass.
"""
import numpy as np
import pytest

import oracle
from fed_inputs import FaceBC, BC_CONV, BC_FLUX, Material, box_problem, make_config, random_field
from parity_util import TOL, oracle_dt, rel_err, trajectory_parity
from test_gpu_parity import _rich_problem, _rich_tet, _table_material

pytestmark = pytest.mark.gpu

CHECKS = [1, 2, 3, 5, 8, 17, 60, 200]   # uneven call lengths


@pytest.fixture(scope="module", autouse=True)
def built():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1909_03355_b200.build import build
    build()
    oracle.build_oracle()


def _check(prob, precision, checks=CHECKS, **kw):
    res = trajectory_parity(prob, precision, checks, resident=1, **kw)
    for k, e in res:
        assert e <= TOL[precision], res
    return res


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("case", ["rich_td", "rich_ti", "tables", "concentrated", "cfg1", "cfg2", "cfg5",
                                  "tet_td", "tet_ti", "tet_paper_td"])
def test_resident_trajectory(case, precision):
    if case == "rich_td":
        p = _rich_problem(8, shuffle=2, n=(12, 10, 9))
    elif case == "rich_ti":
        p = _rich_problem(3, n=(12, 10, 9), td=False)   # near-cubic cells: 8 parity colours
    elif case == "tables":
        p = _rich_problem(9, shuffle=4, n=(10, 9, 8))
        p.material = _table_material(9)
        p.T_lo, p.T_hi = 0.0, 200.0
    elif case == "concentrated":
        p = _rich_problem(6, shuffle=2, n=(9, 8, 7))
        for b in p.face_bcs:
            b.area_mode = 1
    elif case == "cfg1":
        p = make_config(1)
    elif case == "cfg2":
        p = make_config(2, n=24, steps=200)
    elif case == "tet_td":
        p = _rich_tet(6, shuffle=2)
    elif case == "tet_ti":
        p = _rich_tet(7, td=False, n=(7, 6, 8))
    elif case == "tet_paper_td":
        from fed_inputs import paper_tet_problem
        p = paper_tet_problem(td=True, n=12)
    else:
        p = make_config(5, n=24, steps=200)
    _check(p, precision)


def test_resident_matches_streaming_and_reports_mode():
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=32, steps=300)
    dt = oracle_dt(p)
    a = fed.Fed.from_problem(p, precision=64, dt=dt, resident=1)
    b = fed.Fed.from_problem(p, precision=64, dt=dt, resident=-1)
    assert a.info()["resident"] == 1 and b.info()["resident"] == 0
    for n in (1, 7, 64, 228):
        a.step(n)
        b.step(n)
    assert rel_err(a.temperature(), b.temperature()) <= 1e-13
    assert a.info()["step"] == 300


def test_resident_mixed_with_streaming_steps_and_set_temperature():
    """Resident calls, timed (streaming) calls, a steady-state check and a new
    field set in between must compose exactly like one oracle trajectory."""
    from paper_1909_03355_b200 import fed
    p = _rich_problem(4, shuffle=1, n=(12, 10, 9))
    dt = oracle_dt(p)
    o = oracle.Oracle(p, dt)
    g = fed.Fed.from_problem(p, precision=64, dt=dt, resident=1)
    g.step(5)
    o.step(5)
    g.set_timing(True)          # streaming path while timing is on
    g.step(4)
    o.step(4)
    g.set_timing(False)
    g.step(11)
    o.step(11)
    assert rel_err(g.temperature(), o.T()) <= TOL[64]
    T = 20 + random_field(p.n_nodes, 21, 0, 60)
    g.set_temperature(T)
    Td = T.copy()
    Td[p.dir_nodes] = p.dir_T
    o.set_T(Td)
    g.step(3)
    o.step(3)
    assert rel_err(g.temperature(), o.T()) <= TOL[64]
    n, d = g.run_until_steady(tol=1e-12, max_steps=30, check_every=10)   # monitored steps (streaming)
    o.step(n)
    assert rel_err(g.temperature(), o.T()) <= TOL[64]


def test_resident_required_but_impossible():
    from paper_1909_03355_b200 import fed
    p = _rich_problem(3, n=(6, 5, 4))
    with pytest.raises(fed.FedError) as e:       # staged compare-and-swap scatter: not a register mode
        fed.Fed.from_problem(p, precision=64, resident=1, scatter=3)
    assert e.value.status == fed.FED_ERR_INVALID
    big = make_config(3)          # 2.1 M elements: chunks do not all fit at once
    g = fed.Fed.from_problem(big, precision=32, device=0)
    assert g.info()["resident"] == 0


def test_resident_instability_detected():
    from paper_1909_03355_b200 import fed
    mat = Material(1.0, 1.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    p = box_problem(6, 6, 6, L=(6, 6, 6), material=mat, T0=lambda x: random_field(x.shape[0], 9))
    dtc = oracle.dt_crit(p)
    g = fed.Fed.from_problem(p, precision=64, dt=1.1 * dtc, T_abort=1e6, resident=1)
    with pytest.raises(fed.FedError) as e:
        g.step(2000)
    assert e.value.status == fed.FED_ERR_UNSTABLE
    assert 0 < g.info()["fail_step"] < 2000


def test_resident_cfg1_closed_form():
    """cfg1 in resident mode against the exact discrete solution (independent of the oracle)."""
    from paper_1909_03355_b200 import fed
    from test_oracle_pins import cfg1_closed_form
    p = make_config(1)
    dt = 0.9 * oracle.dt_crit(p)
    g = fed.Fed.from_problem(p, precision=64, dt=dt, resident=1)
    alpha = 50.0 / (7800 * 460)
    done = 0
    for ks in (1, 10, 100, 2000):
        g.step(ks - done)
        done = ks
        T = g.temperature().reshape(11, 11, 11)
        ref = cfg1_closed_form(10, alpha, 0.1, dt, ks)
        assert np.abs(T - ref[None, None, :]).max() <= 1e-11 * 100
