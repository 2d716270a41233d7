"""GPU parity of the partitioned (z-slab) path on one GPU.

`fed_options.local_ranks = P` makes one context hold the P slabs of P ranks on
one device: each slab is planned, stored and stepped exactly as on its own GPU
(interface chunks first, interior chunks, exchange, node kernel), and the
interface partial loads travel either as the device copy an ncclSend/ncclRecv
pair would make (FED_TRANSPORT_NCCL) or through the fused peer-load path
(FED_TRANSPORT_PEER: step flags raised by the interface-chunk launch, loads read
from the neighbour's buffer by the node kernel) on same-device pointers.  All
kernels run in one stream in an order where no kernel waits for another
(B200_PROFILING.md: ranks whose kernels wait on one another must not share a
GPU).  Results must match the fp64 oracle within the north_star tolerances
(reading 8c-19) and the single-rank run.
"""
import numpy as np
import pytest

import oracle
from fed_inputs import make_config, random_field
from parity_util import TOL, oracle_dt, rel_err, trajectory_parity
from test_gpu_parity import _rich_problem, _rich_tet, _table_material

pytestmark = pytest.mark.gpu

NCCL, PEER = 0, 1


@pytest.fixture(scope="module", autouse=True)
def built():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1909_03355_b200.build import build
    build()
    oracle.build_oracle()


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("transport", [NCCL, PEER])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_group_rich_trajectory(P, transport, precision):
    """Jittered, renumbered box with Dirichlet, flux, convection, radiation and a
    source: interface nodes carry face loads and Dirichlet values too."""
    p = _rich_problem(8, shuffle=2, n=(9, 8, 12))
    res = trajectory_parity(p, precision, [1, 10, 100, 300], chunk_elems=128, local_ranks=P, transport=transport)
    for k, e in res:
        assert e <= TOL[precision], (P, transport, res)


@pytest.mark.parametrize("transport", [NCCL, PEER])
@pytest.mark.parametrize("scatter", [2, 3, 4, 5])
def test_group_scatter_strategies(scatter, transport):
    p = _rich_problem(3, shuffle=7, n=(8, 7, 10))
    res = trajectory_parity(p, 64, [1, 50, 200], scatter=scatter, chunk_elems=64, local_ranks=3,
                            transport=transport)
    for k, e in res:
        assert e <= TOL[64], (scatter, transport, res)


def test_group_atomic_scatter_nccl():
    p = _rich_problem(4, shuffle=1, n=(7, 7, 9))
    res = trajectory_parity(p, 64, [1, 50, 200], scatter=1, local_ranks=3, transport=NCCL)
    for k, e in res:
        assert e <= TOL[64], res


def test_group_peer_needs_chunks():
    from paper_1909_03355_b200 import fed
    p = _rich_problem(4, n=(4, 4, 6))
    with pytest.raises(fed.FedError) as e:
        fed.Fed.from_problem(p, precision=64, scatter=1, local_ranks=2, transport=PEER)
    assert e.value.status == fed.FED_ERR_INVALID


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_group_cfg5_scaled(P, precision):
    """cfg5 physics (TD k, c; convection on 5 faces; Gaussian source) at 24^3,
    z-slabs of 12 / 6 / 3 layers -- the strong-scaling configuration in small."""
    p = make_config(5, n=24, steps=500)
    res = trajectory_parity(p, precision, [1, 50, 200, 500], local_ranks=P, transport=PEER)
    for k, e in res:
        assert e <= TOL[precision], (P, res)


def test_group_cfg4_scaled_renumbered():
    p = make_config(4, n=16, steps=300)
    for transport in (NCCL, PEER):
        res = trajectory_parity(p, 32, [1, 100, 300], local_ranks=4, transport=transport)
        for k, e in res:
            assert e <= TOL[32], (transport, res)


@pytest.mark.parametrize("transport", [NCCL, PEER])
def test_group_tet(transport):
    p = _rich_tet(6, shuffle=3, n=(6, 5, 9))
    res = trajectory_parity(p, 64, [1, 20, 200], local_ranks=3, transport=transport)
    for k, e in res:
        assert e <= TOL[64], res


def test_group_tables_and_concentrated_bcs():
    p = _rich_problem(9, shuffle=4, n=(8, 7, 10))
    p.material = _table_material(9)
    for b in p.face_bcs:
        b.area_mode = 1
    res = trajectory_parity(p, 64, [1, 20, 200], local_ranks=3, transport=PEER)
    for k, e in res:
        assert e <= TOL[64], res


def test_group_matches_single_rank_and_graphs():
    """P = 4 slabs vs the unpartitioned run, CUDA graphs vs eager launches."""
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=16, steps=200)
    dt = oracle_dt(p)
    one = fed.Fed.from_problem(p, precision=64, dt=dt)
    grp = fed.Fed.from_problem(p, precision=64, dt=dt, local_ranks=4, transport=PEER)
    eag = fed.Fed.from_problem(p, precision=64, dt=dt, local_ranks=4, transport=PEER, graph_steps=-1)
    for g in (one, grp, eag):
        g.step(200)
    T1 = one.temperature()
    assert rel_err(grp.temperature(), T1) <= 1e-13
    assert rel_err(eag.temperature(), T1) <= 1e-13
    info = grp.info()
    assert info["nranks"] == 4 and info["rank"] == -1 and info["step"] == 200
    assert info["n_elems_local"] == p.conn.shape[0]
    assert info["n_interface"] == 2 * 3 * 17 * 17
    assert info["kernel_launches_per_step"] == 4 * 2   # per slab: one element launch (PEER) + node


def test_group_steady_state_and_roundtrip():
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=8, steps=100)
    dt = oracle_dt(p)
    a = fed.Fed.from_problem(p, precision=64, dt=dt)
    b = fed.Fed.from_problem(p, precision=64, dt=dt, local_ranks=2, transport=PEER)
    T = 20 + random_field(p.n_nodes, 17, 0, 50)
    a.set_temperature(T)
    b.set_temperature(T)
    np.testing.assert_array_equal(a.temperature(), b.temperature())
    sa = a.run_until_steady(tol=1e-2, max_steps=3000, check_every=100)
    sb = b.run_until_steady(tol=1e-2, max_steps=3000, check_every=100)
    assert sa[0] == sb[0]
    assert sb[1] == pytest.approx(sa[1], rel=1e-6)
    assert rel_err(b.temperature(), a.temperature()) <= 1e-12


def test_group_rank_timing():
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=32)
    g = fed.Fed.from_problem(p, precision=32, local_ranks=4, transport=PEER)
    g.set_timing(True)
    g.step(10)
    tot = g.timing()
    per = [g.rank_timing(r) for r in range(4)]
    for r, t in enumerate(per):
        assert t["element_launches"] == 10 and t["element_ms"] > 0, (r, t)
        assert t["node_launches"] == 10 and t["node_ms"] > 0, (r, t)
    assert tot["element_ms"] == pytest.approx(sum(t["element_ms"] for t in per))
    with pytest.raises(fed.FedError):
        g.rank_timing(4)


def test_group_instability_detected():
    from fed_inputs import Material, box_problem
    from paper_1909_03355_b200 import fed
    mat = Material(1.0, 1.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    p = box_problem(5, 5, 8, L=(5, 5, 8), material=mat, T0=lambda x: random_field(x.shape[0], 9))
    dtc = oracle.dt_crit(p)
    g = fed.Fed.from_problem(p, precision=64, dt=1.1 * dtc, local_ranks=2, transport=PEER)
    with pytest.raises(fed.FedError) as e:
        g.step(3000)
    assert e.value.status == fed.FED_ERR_UNSTABLE
    assert 0 < g.info()["fail_step"] < 3000


@pytest.mark.parametrize("transport", [NCCL, PEER])
def test_debug_time_rank_alone(transport):
    """fed_debug_time_rank replays one slab's kernel sequence alone (timing only)
    and leaves the context unusable for stepping."""
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=24)
    g = fed.Fed.from_problem(p, precision=32, local_ranks=3, transport=transport, chunk_elems=128)
    g.step(4)
    ms = [g.debug_time_rank(r, 8) for r in range(3)]
    assert all(m > 0 for m in ms)
    with pytest.raises(fed.FedError) as e:
        g.step(1)
    assert e.value.status == fed.FED_ERR_STATE
