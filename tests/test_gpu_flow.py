"""GPU parity of flow mode (fed_options.flow): one cooperative launch of a
persistent CTA pool per fed_step call, chunks streamed step after step and
ordered by per-chunk dataflow (no kernel boundary or node kernel between steps).
Results must match the fp64 oracle within the north_star tolerances (reading
8c-19) and the streaming path; uneven call lengths exercise the call-relative
step % 2 / step % 3 buffers and the finalize pass.
"""
import pytest

import oracle
from fed_inputs import make_config, random_field
from parity_util import TOL, oracle_dt, rel_err, trajectory_parity
from test_gpu_parity import _rich_problem, _table_material

pytestmark = pytest.mark.gpu

CHECKS = [1, 2, 3, 5, 8, 17, 60, 200]


@pytest.fixture(scope="module", autouse=True)
def built():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1909_03355_b200.build import build
    build()
    oracle.build_oracle()


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("case", ["rich_td", "tables", "cfg4", "cfg5"])
def test_flow_trajectory(case, precision):
    if case == "rich_td":
        p = _rich_problem(8, shuffle=2, n=(12, 10, 9))
    elif case == "tables":
        p = _rich_problem(9, shuffle=4, n=(12, 10, 9))
        p.material = _table_material(9)
        p.T_lo, p.T_hi = 0.0, 200.0
    elif case == "cfg4":
        p = make_config(4, n=16, steps=200)
    else:
        p = make_config(5, n=24, steps=200)
    res = trajectory_parity(p, precision, CHECKS, flow=1, resident=-1, chunk_elems=128)
    for k, e in res:
        assert e <= TOL[precision], res


def test_flow_matches_streaming_and_mixes_with_it():
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=32, steps=300)
    dt = oracle_dt(p)
    a = fed.Fed.from_problem(p, precision=64, dt=dt, flow=1, resident=-1, chunk_elems=256)
    b = fed.Fed.from_problem(p, precision=64, dt=dt, resident=-1, chunk_elems=256)
    assert a.info()["flow"] == 1 and b.info()["flow"] == 0
    for n in (1, 7, 64):
        a.step(n)
        b.step(n)
    a.set_timing(True)      # streaming path while timing is on
    a.step(5)
    b.step(5)
    a.set_timing(False)
    T = 20 + random_field(p.n_nodes, 3, 0, 50)
    a.set_temperature(T)
    b.set_temperature(T)
    a.step(23)
    b.step(23)
    assert rel_err(a.temperature(), b.temperature()) <= 1e-13
    assert a.info()["step"] == 100


def test_flow_full_size_cfg5_sampled():
    """cfg5 at full size in flow mode vs streaming after a few steps (fp32)."""
    from paper_1909_03355_b200 import fed
    p = make_config(5)
    a = fed.Fed.from_problem(p, precision=32, flow=1)
    a.step(20)
    Ta = a.temperature()
    a.close()
    b = fed.Fed.from_problem(p, precision=32)
    b.step(20)
    Tb = b.temperature()
    assert rel_err(Ta, Tb) <= 1e-6
