"""GPU parity: the CUDA path (through the C ABI, paper_1909_03355_b200.fed)
against the fp64 oracle on the same seeded inputs.

Tolerances (north_star, reading 8c-19): max_n |T_gpu - T_ora| / max_n |T_ora|
<= 1e-11 for the fp64 path and <= 1e-4 for the fp32 path.
"""
import numpy as np
import pytest

import oracle
from fed_inputs import (BC_CONV, BC_FLUX, BC_RAD, FaceBC, Material, box_problem, make_config, random_field,
                        random_spd_tensor)
from parity_util import TOL, multi_parity, oracle_dt, patch_problem, rel_err, trajectory_parity

pytestmark = pytest.mark.gpu

SCATTERS = [2, 3, 4, 5, 1]   # CHUNK, CHUNK_CAS, CHUNK_REG, CHUNK_REGC, ATOMIC


@pytest.fixture(scope="module", autouse=True)
def built():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1909_03355_b200.build import build
    build()
    oracle.build_oracle()


def _rich_problem(seed=0, shuffle=None, n=(7, 6, 5), td=True):
    mat = Material(7800.0, 460.0, 0.001 if td else 0.0, random_spd_tensor(seed, 20, 80), 0.002 if td else 0.0)
    bcs = [FaceBC(BC_FLUX, q=2e4), FaceBC(BC_CONV, h=40.0, T_inf=15.0), FaceBC(BC_RAD, eps=0.7, T_inf=30.0)]
    p = box_problem(*n, L=(0.07, 0.06, 0.05), material=mat, side_bc={"z0": 0, "x1": 1, "y0": 1, "z1": 2},
                    face_bcs=bcs, dirichlet={"x0": 80.0}, T0=lambda x: 20 + random_field(x.shape[0], seed, 0, 60),
                    q_vol=lambda x: 5e5 * np.exp(-((x - 0.03) ** 2).sum(axis=1) / 1e-3), jitter=0.2, seed=seed,
                    shuffle_seed=shuffle)
    p.T_lo, p.T_hi = 0.0, 200.0
    return p


# ---------------------------------------------------------------- one step, many meshes
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter", SCATTERS)
@pytest.mark.parametrize("case", ["single", "affine", "jitter_shuffled", "rich_td", "rich_ti", "ragged"])
def test_one_step_from_random_field(precision, scatter, case):
    if case == "single":
        p = box_problem(1, 1, 1, material=Material(2.0, 3.0, 0.0, random_spd_tensor(1), 0.0))
    elif case == "affine":
        p = box_problem(4, 3, 5, affine=[[1.0, 0.3, 0.1], [0.0, 0.8, -0.2], [0.2, 0.1, 1.2]],
                        material=Material(2.0, 3.0, 0.0, random_spd_tensor(2), 0.0))
    elif case == "jitter_shuffled":
        p = box_problem(6, 6, 6, jitter=0.2, seed=4, shuffle_seed=9,
                        material=Material(2.0, 3.0, 0.0, random_spd_tensor(3), 0.0))
    elif case == "rich_td":
        p = _rich_problem(5, shuffle=3)
    elif case == "rich_ti":
        p = _rich_problem(6, td=False)
    else:
        p = _rich_problem(7, n=(13, 11, 9))
    T = 20 + random_field(p.n_nodes, 11, 0, 80)
    dt = oracle_dt(p)
    res = trajectory_parity(p, precision, [1], dt=dt, T_start=T, scatter=scatter, chunk_elems=64)
    assert res[0][1] <= TOL[precision], res


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter,resident", [(s, -1) for s in SCATTERS] + [(5, 1)])
def test_rich_trajectory(precision, scatter, resident):
    """resident = -1: the streaming kernels bench.py times; 1: resident_kernel."""
    p = _rich_problem(8, shuffle=2, n=(12, 10, 9))
    res = trajectory_parity(p, precision, [1, 10, 100, 400], scatter=scatter, chunk_elems=128, resident=resident)
    for k, e in res:
        assert e <= TOL[precision], res


# ---------------------------------------------------------------- configs (scaled) trajectories
CFG_SCALED = [(1, None, 2000, [1, 10, 100, 500, 2000]),
              (2, 16, 3000, [1, 100, 1000, 3000]),
              (3, 16, 2000, [1, 100, 1000, 2000]),
              (4, 16, 1000, [1, 10, 100, 1000]),
              (5, 24, 500, [1, 50, 200, 500])]


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("cfg,n,steps,checks", CFG_SCALED)
def test_config_trajectory(cfg, n, steps, checks, precision):
    """Every scaled config against the oracle in BOTH execution modes: the
    streaming element_chunk_kernel + node_kernel that bench.py times
    (resident = -1) and the one-launch resident_kernel (resident = 1), side by
    side on one oracle trajectory."""
    p = make_config(cfg, n=n, steps=steps)
    res, infos = multi_parity(p, [(precision, {"resident": -1}), (precision, {"resident": 1})], checks)
    assert infos[0]["resident"] == 0 and infos[1]["resident"] == 1
    for i in res:
        for k, e in res[i]:
            assert e <= TOL[precision], (cfg, i, res)


@pytest.mark.parametrize("precision", [32, 64])
def test_cfg5_streaming_1024_chunks_500_steps(precision):
    """cfg5 at n = 96 (864 chunks of 1024 elements: above the resident-mode cap,
    so the automatic choice is the streaming path) -- the benched kernel
    instantiation (element_chunk_kernel, colour phases, 1024-element chunks,
    CUDA-graph replay) for the config's full 500 steps against the oracle."""
    p = make_config(5, n=96)
    res, infos = multi_parity(p, [(precision, {})], [1, 50, 200, 500], dt=DT_FULL[5])
    assert infos[0]["resident"] == 0 and infos[0]["chunk_elems"] == 1024 and infos[0]["n_chunks"] == 864
    assert infos[0]["scatter"] == 5
    for i in res:
        for k, e in res[i]:
            assert e <= TOL[precision], res


@pytest.mark.parametrize("chunk", [2048, 2624])
@pytest.mark.parametrize("case", ["cfg5", "rich"])
def test_packed_record_large_chunks(chunk, case):
    """The fp32 streaming kernel's 12-bit packed positions at their upper range:
    chunks of 2048 / 2624 elements (up to 3 200 / 4 064 local nodes, so bit 11 of the
    fields is set) on cfg5's physics and on a jittered, shuffled mesh with every BC
    kind, trajectory against the oracle (colours of > 128 elements: the kernel's
    general colour loop)."""
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=40) if case == "cfg5" else _rich_problem(8, shuffle=5, n=(26, 24, 22))
    R = fed.FED_SCATTER_CHUNK_REGC
    g = fed.Fed.from_problem(p, precision=32, device=-1, scatter=R, chunk_elems=chunk, resident=-1)
    _, _, c16 = g.debug_chunks()
    assert g.info()["scatter"] == R and int(c16.max()) >= 2048, int(c16.max())
    g.close()
    res = trajectory_parity(p, 32, [1, 20, 100], dt=DT_FULL[5] if case == "cfg5" else None, scatter=R,
                            chunk_elems=chunk, resident=-1)
    for k, e in res:
        assert e <= TOL[32], res


def test_cfg1_closed_form_on_gpu():
    """GPU cfg1 against the exact discrete solution (independent of the oracle)."""
    from paper_1909_03355_b200 import fed
    from test_oracle_pins import cfg1_closed_form
    p = make_config(1)
    dt = 0.9 * oracle.dt_crit(p)
    g = fed.Fed.from_problem(p, precision=64, dt=dt)
    alpha = 50.0 / (7800 * 460)
    done = 0
    for ks in (1, 10, 100, 2000):
        g.step(ks - done)
        done = ks
        T = g.temperature().reshape(11, 11, 11)
        ref = cfg1_closed_form(10, alpha, 0.1, dt, ks)
        assert np.abs(T - ref[None, None, :]).max() <= 1e-11 * 100


# ---------------------------------------------------------------- full-size configs
DT_FULL = {2: 0.059128, 3: 0.0189954, 4: 1.57929e-3, 5: 2.0075e-3}


@pytest.mark.parametrize("cfg,precision", [(2, 32), (2, 64), (3, 32)])
def test_full_size_trajectory_small_configs(cfg, precision):
    """cfg2 (64^3) and cfg3 (128^3) at full size, bench launch configuration."""
    p = make_config(cfg)
    steps = [1, 20, 100] if cfg == 2 else [1, 10, 20]
    res = trajectory_parity(p, precision, steps, dt=DT_FULL[cfg])
    for k, e in res:
        assert e <= TOL[precision], res


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_sampled_step(cfg):
    """cfg4 (256^3, jittered + renumbered) and cfg5 (384^3) at full size, fp32,
    in the launch configuration bench.py times: one step from a seeded random
    field, checked at sampled nodes against the oracle run on the patch of
    elements / faces around them."""
    from paper_1909_03355_b200 import fed
    p = make_config(cfg)
    T = 20 + random_field(p.n_nodes, 123, 0, 80)
    g = fed.Fed.from_problem(p, precision=32, dt=DT_FULL[cfg])
    g.set_temperature(T)
    g.step(1)
    Tg = g.temperature()
    g.close()
    rng = np.random.default_rng(5)
    sample = np.concatenate([rng.choice(p.n_nodes, 60, replace=False),
                             np.unique(p.faces[rng.choice(p.faces.shape[0], 20, replace=False)].ravel())])
    sub, ls, nodes = patch_problem(p, sample)
    o = oracle.Oracle(sub, DT_FULL[cfg])
    o.set_T(T[nodes])
    o.step(1)
    ref = o.T()[ls]
    got = Tg[np.unique(sample)]
    assert rel_err(got, ref) <= TOL[32]
    # and the change itself is resolved (not just T0 echoed back)
    dT_ref = ref - T[np.unique(sample)]
    assert np.abs(dT_ref).max() > 0
    assert np.abs((got - T[np.unique(sample)]) - dT_ref).max() <= 1e-3 * np.abs(dT_ref).max() + 1e-4 * 100


def test_full_size_cfg5_properties():
    """cfg5 full size, 100 steps: the x<->y / x->L-x symmetry of the problem
    and the global energy balance (properties that hold at any size)."""
    from paper_1909_03355_b200 import fed
    p = make_config(5)
    g = fed.Fed.from_problem(p, precision=32)
    info = g.info()
    T0 = g.temperature()
    g.step(100)
    T = g.temperature()
    n = 385
    Tg = T.reshape(n, n, n)
    scale = np.abs(Tg).max()
    assert np.abs(Tg - Tg.transpose(0, 2, 1)).max() <= 1e-5 * scale
    assert np.abs(Tg - Tg[:, :, ::-1]).max() <= 1e-5 * scale
    assert Tg.max() > 20.0 and np.isfinite(Tg).all()
    # energy: heat gained ~ source power x time (convection losses are tiny at these T)
    V, coef = g.debug_nodal()
    rhoc = 7800.0 * 460.0
    dE = (V * 7800.0 * 460.0 * ((T - 20.0) + 0.001 * (T ** 2 - 400.0) / 2)).sum()  # integral of rho c(T) dT
    P_src = (p.q_vol * V).sum()
    assert dE == pytest.approx(P_src * 100 * info["dt"], rel=2e-3)
    assert rhoc > 0


# ---------------------------------------------------------------- edge cases
def test_zero_steps_and_roundtrip():
    from paper_1909_03355_b200 import fed
    p = box_problem(3, 3, 3, shuffle_seed=4, dirichlet={"x0": 5.0})
    g = fed.Fed.from_problem(p, precision=64)
    g.step(0)
    T = random_field(p.n_nodes, 1)
    g.set_temperature(T)
    got = g.temperature()
    exp = T.copy()
    exp[p.dir_nodes] = 5.0
    np.testing.assert_array_equal(got, exp)
    assert g.info()["step"] == 0


def test_all_dirichlet_is_fixed_point():
    from paper_1909_03355_b200 import fed
    sides = {s: 37.0 for s in ("x0", "x1", "y0", "y1", "z0", "z1")}
    p = box_problem(1, 1, 1, dirichlet=sides, T0=0.0)
    g = fed.Fed.from_problem(p, precision=64)
    g.step(50)
    np.testing.assert_array_equal(g.temperature(), 37.0)


def test_instability_detected():
    from paper_1909_03355_b200 import fed
    mat = Material(1.0, 1.0, 0.0, (1.0, 1.0, 1.0, 0, 0, 0), 0.0)
    p = box_problem(5, 5, 5, L=(5, 5, 5), material=mat, T0=lambda x: random_field(x.shape[0], 9))
    dtc = oracle.dt_crit(p)
    g = fed.Fed.from_problem(p, precision=64, dt=1.1 * dtc, T_abort=1e6)
    with pytest.raises(fed.FedError) as e:
        g.step(2000)
    assert e.value.status == fed.FED_ERR_UNSTABLE
    fs = g.info()["fail_step"]
    assert 0 < fs < 2000
    ok = fed.Fed.from_problem(p, precision=64, dt=0.9 * dtc)
    ok.step(2000)
    assert ok.info()["fail_step"] == -1


def test_graph_and_eager_agree():
    """Streaming mode (resident = -1, where graph_steps applies): eager launches
    and CUDA-graph replays (16-step graphs, plus an eager remainder) give the same
    field, and both match the oracle."""
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=12, steps=101)
    dt = oracle_dt(p)
    a = fed.Fed.from_problem(p, precision=64, dt=dt, graph_steps=-1, resident=-1)
    b = fed.Fed.from_problem(p, precision=64, dt=dt, graph_steps=16, resident=-1)
    assert a.info()["resident"] == 0 and b.info()["resident"] == 0
    n0 = b.info()["kernel_launches_total"]
    a.step(101)
    b.step(101)
    ib = b.info()
    L = ib["kernel_launches_per_step"]
    # 6 graph replays of 16 steps (2 kernels each + 1 counter advance) + 5 eager steps + 1 advance
    assert L == 2 and ib["kernel_launches_total"] - n0 == 6 * (16 * L + 1) + 5 * L + 1
    assert rel_err(a.temperature(), b.temperature()) <= 1e-13
    assert a.info()["step"] == ib["step"] == 101
    o = oracle.Oracle(p, dt)
    o.step(101)
    assert rel_err(b.temperature(), o.T()) <= TOL[64]


def test_timing_api():
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=32)
    g = fed.Fed.from_problem(p, precision=32)
    g.set_timing(True)
    g.step(10)
    t = g.timing()
    assert t["element_launches"] == 10 and t["node_launches"] == 10
    assert t["element_ms"] > 0 and t["node_ms"] > 0


def test_mode_switches_and_readouts():
    """A resident context switches to streaming steps while timing is on: readouts
    between calls, single steps, set_temperature and resident <-> streaming switches
    all reproduce the oracle's sequence."""
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=12, steps=100)
    dt = oracle_dt(p)
    o = oracle.Oracle(p, dt)
    g = fed.Fed.from_problem(p, precision=64, dt=dt)        # resident candidate
    assert g.info()["resident"] == 1
    T_set = 20 + random_field(p.n_nodes, 31, 0, 90)
    seq = [("step", 7, False), ("read",), ("step", 1, True), ("step", 13, True), ("read",), ("step", 5, False),
           ("set",), ("step", 1, True), ("read",), ("step", 9, False), ("step", 3, True), ("step", 2, False), ("read",)]
    for op in seq:
        if op[0] == "step":
            g.set_timing(op[2])        # True: streaming steps; False: resident mode
            g.step(op[1])
            o.step(op[1])
        elif op[0] == "read":
            assert rel_err(g.temperature(), o.T()) <= TOL[64], op
        else:
            g.set_temperature(T_set)
            o.set_T(T_set)
    assert g.info()["step"] == 41


# ---------------------------------------------------------------- tet4 (NEXT-1, Eq. 18)
def _rich_tet(seed=0, td=True, shuffle=None, n=(6, 5, 7)):
    from fed_inputs import tet_box_problem
    mat = Material(7800.0, 460.0, 0.001 if td else 0.0, random_spd_tensor(seed, 20, 80), 0.002 if td else 0.0)
    bcs = [FaceBC(BC_FLUX, q=2e4), FaceBC(BC_CONV, h=40.0, T_inf=15.0), FaceBC(BC_RAD, eps=0.7, T_inf=30.0)]
    p = tet_box_problem(*n, L=(0.06, 0.05, 0.07), material=mat, side_bc={"z0": 0, "x1": 1, "y0": 1, "z1": 2},
                        face_bcs=bcs, dirichlet={"x0": 80.0}, T0=lambda x: 20 + random_field(x.shape[0], seed, 0, 60),
                        q_vol=lambda x: 5e5 * np.exp(-((x - 0.03) ** 2).sum(axis=1) / 1e-3), jitter=0.2, seed=seed,
                        shuffle_seed=shuffle)
    p.T_lo, p.T_hi = 0.0, 200.0
    return p


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter", [4, 5, 1])
@pytest.mark.parametrize("td", [True, False])
def test_tet_one_step_from_random_field(precision, scatter, td):
    p = _rich_tet(3, td=td, shuffle=5)
    T = 20 + random_field(p.n_nodes, 12, 0, 80)
    res = trajectory_parity(p, precision, [1], dt=oracle_dt(p), T_start=T, scatter=scatter, chunk_elems=128)
    assert res[0][1] <= TOL[precision], res


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter", [4, 5])
def test_tet_trajectory(precision, scatter):
    p = _rich_tet(4, shuffle=1, n=(9, 8, 10))
    res = trajectory_parity(p, precision, [1, 10, 100, 300], scatter=scatter)
    for k, e in res:
        assert e <= TOL[precision], res


@pytest.mark.parametrize("td", [False, True])
def test_paper_tet_workload_trajectory(td):
    """Shape of the paper's Sec. 4.6 timing workload (41 154 tets), 200 steps."""
    from fed_inputs import paper_tet_problem
    p = paper_tet_problem(td=td)
    res = trajectory_parity(p, 64, [1, 50, 200])
    for k, e in res:
        assert e <= TOL[64], res


def test_tet_patch_test_on_gpu():
    """Linear field pinned on the boundary of a jittered tet mesh is reproduced
    exactly in the interior, on the GPU path."""
    from fed_inputs import tet_box_problem
    from paper_1909_03355_b200 import fed
    mat = Material(1000.0, 2000.0, 0.0, (200.0, 200.0, 200.0, 0, 0, 0), 0.0)
    lin = lambda x: 200 * x[:, 0] + 100 * x[:, 1] + 200 * x[:, 2]
    p = tet_box_problem(5, 5, 5, material=mat, dirichlet={s: lin for s in ("x0", "x1", "y0", "y1", "z0", "z1")},
                        T0=0.0, jitter=0.25, seed=7)
    g = fed.Fed.from_problem(p, precision=64, dt=0.9 * oracle.dt_crit(p))
    g.step(8000)
    Tl = lin(p.xyz)
    assert np.abs(g.temperature() - Tl).max() <= 1e-9 * np.abs(Tl).max()


# ---------------------------------------------------------------- tables (NEXT-2)
def _table_material(seed):
    kt = ((10.0, 40.0, 70.0, 120.0), (0.8, 1.6, 1.1, 2.0))
    ct = ((0.0, 50.0, 150.0), (400.0, 700.0, 520.0))
    return Material(7800.0, 460.0, 0.0, random_spd_tensor(seed, 20, 80), 0.0, k_table=kt, c_table=ct)


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter", [2, 4, 5, 1])
def test_table_hex_trajectory(precision, scatter):
    p = _rich_problem(9, shuffle=4, n=(10, 9, 8))
    p.material = _table_material(9)
    p.T_lo, p.T_hi = 0.0, 200.0
    res = trajectory_parity(p, precision, [1, 10, 100, 300], scatter=scatter, chunk_elems=128)
    for k, e in res:
        assert e <= TOL[precision], res


@pytest.mark.parametrize("precision", [64, 32])
def test_table_tet_paper_422(precision):
    """The paper's Sec. 4.2.2 TD tables (k 200->2000, c 2000->8000 over 37->337 degC)
    on the Sec. 4.6-shaped tet cube with a hot flux face."""
    from fed_inputs import paper_td_material, paper_tet_problem
    p = paper_tet_problem(n=12)
    p.material = paper_td_material()
    p.face_bcs[0].q = 2e6
    p.T_lo, p.T_hi = 37.0, 337.0
    res = trajectory_parity(p, precision, [1, 20, 200, 600])
    for k, e in res:
        assert e <= TOL[precision], res


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("case", ["two_point_tables", "collinear_three_point", "k_table_c_law", "constant_c"])
def test_clamped_linear_tables(precision, case):
    """Tables of <= 2 points are clamped linear functions: the library evaluates them
    like the linear laws (temperature_dependent = 3), a 3-point table through the same
    line takes the general table path (2); both against the oracle, which always
    interpolates the table, over a range that crosses both clamps."""
    from paper_1909_03355_b200 import fed
    p = _rich_problem(10, shuffle=6, n=(10, 9, 8))
    rho = 7800.0
    kt2 = ((30.0, 90.0), (0.8, 2.0))
    if case == "two_point_tables":
        m, td = Material(rho, 460.0, 0.0, random_spd_tensor(10, 20, 80), 0.0, k_table=kt2,
                         c_table=((25.0, 110.0), (420.0, 610.0))), 3
    elif case == "collinear_three_point":
        m, td = Material(rho, 460.0, 0.0, random_spd_tensor(10, 20, 80), 0.0, k_table=((30.0, 60.0, 90.0), (0.8, 1.4, 2.0)),
                         c_table=((25.0, 110.0), (420.0, 610.0))), 2
    elif case == "k_table_c_law":
        m, td = Material(rho, 460.0, 0.001, random_spd_tensor(10, 20, 80), 0.0, k_table=kt2), 3
    else:
        m, td = Material(rho, 460.0, 0.0, random_spd_tensor(10, 20, 80), 0.002, c_table=((50.0,), (500.0,))), 3
    p.material = m
    p.T_lo, p.T_hi = 0.0, 200.0
    g = fed.Fed.from_problem(p, precision=precision, device=-1)
    assert g.info()["temperature_dependent"] == td
    g.close()
    for resident in (-1, 1):
        res = trajectory_parity(p, precision, [1, 10, 100, 300], resident=resident)
        for k, e in res:
            assert e <= TOL[precision], (case, resident, res)


# ---------------------------------------------------------------- concentrated BCs (NEXT-3)
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("tet", [False, True])
def test_concentrated_bc_trajectory(precision, tet):
    p = _rich_tet(6, shuffle=2) if tet else _rich_problem(6, shuffle=2, n=(9, 8, 7))
    for b in p.face_bcs:
        b.area_mode = 1
    p.face_bcs[1].area_mode = 0          # mixed: one record keeps per-face tributary areas
    res = trajectory_parity(p, precision, [1, 10, 100, 300])
    for k, e in res:
        assert e <= TOL[precision], res


# ---------------------------------------------------------------- steady-state mode (NEXT-4)
def test_run_until_steady_matches_oracle_criterion():
    from paper_1909_03355_b200 import fed
    q, hc, Tinf, k = 1e5, 500.0, 20.0, 50.0
    mat = Material(1.0, 3.6e6, 0.0, (k, k, k, 0, 0, 0), 0.0)
    p = box_problem(2, 2, 8, L=(0.025, 0.025, 0.1), material=mat, side_bc={"z0": 0, "z1": 1},
                    face_bcs=[FaceBC(BC_FLUX, q=q), FaceBC(BC_CONV, h=hc, T_inf=Tinf)], T0=20.0)
    dt = 0.9 * oracle.dt_crit(p)
    tol, every = 1e-3, 50                                      # the paper's 0.001 degC
    g = fed.Fed.from_problem(p, precision=64, dt=dt)
    steps, last = g.run_until_steady(tol=tol, max_steps=200000, check_every=every)
    # oracle emulation of the same criterion (max per-step change at each check)
    o = oracle.Oracle(p, dt)
    done = 0
    while True:
        o.step(every - 1)
        T0 = o.T()
        o.step(1)
        done += every
        d = np.abs(o.T() - T0).max()
        if d <= tol:
            break
    assert steps == done and 0 < last <= tol
    assert last == pytest.approx(d, rel=1e-6)
    assert rel_err(g.temperature(), o.T()) <= 1e-11
    # near the analytic steady profile T(z) = Tinf + q/h + q (L - z)/k
    ref = Tinf + q / hc + q * (0.1 - p.xyz[:, 2]) / k
    assert np.abs(g.temperature() - ref).max() < 10.0
    steps2, last2 = g.run_until_steady(tol=1e-9, max_steps=400000, check_every=500)
    assert last2 <= 1e-9 and np.abs(g.temperature() - ref).max() <= 1e-5 * ref.max()


# ---------------------------------------------------------------- scatter baselines (measured)
BASELINES = [6, 7, 8]   # ATOMIC_WARP, COLOR_PASSES, GATHER


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("scatter", BASELINES)
@pytest.mark.parametrize("case", ["rich_td", "jitter_shuffled", "cfg5"])
def test_scatter_baselines_trajectory(case, scatter, precision):
    if case == "rich_td":
        p = _rich_problem(8, shuffle=2, n=(12, 10, 9))
    elif case == "jitter_shuffled":
        p = box_problem(9, 8, 10, jitter=0.2, seed=4, shuffle_seed=9, L=(0.09, 0.08, 0.1),
                        material=Material(2.0, 3.0, 0.0, random_spd_tensor(3), 0.0),
                        T0=lambda x: random_field(x.shape[0], 2, 0, 50))
    else:
        p = make_config(5, n=24, steps=200)
    res = trajectory_parity(p, precision, [1, 10, 100], scatter=scatter, resident=-1)
    for k, e in res:
        assert e <= TOL[precision], (scatter, res)


@pytest.mark.parametrize("precision", [64, 32])
def test_gather_baseline_tets(precision):
    p = _rich_tet(3, shuffle=5)
    res = trajectory_parity(p, precision, [1, 20, 100], scatter=8, resident=-1)
    for k, e in res:
        assert e <= TOL[precision], res


def test_color_passes_rejects_invalid_global_colouring():
    from paper_1909_03355_b200 import fed
    p = _rich_tet(3, shuffle=5)       # Kuhn tets: chunk colours are not a global colouring
    with pytest.raises(fed.FedError) as e:
        fed.Fed.from_problem(p, precision=64, scatter=7, resident=-1)
    assert e.value.status == fed.FED_ERR_INVALID
