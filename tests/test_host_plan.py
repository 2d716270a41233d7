"""CPU tests of libfed.so's host side (no GPU): exported C-ABI symbols, the
dry-run plan (device = -1), the fp64 pre-computation against the oracle, and
error handling.  The planner's arithmetic (critical step, lumped volumes) is
independent code from the oracle's; agreement is checked here to round-off.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from fed_inputs import (BC_CONV, BC_FLUX, BC_RAD, FaceBC, Material, box_problem, make_config,
                        random_spd_tensor)
from paper_1909_03355_b200 import fed
from paper_1909_03355_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return fed.load()


def dry(prob, **kw):
    kw.setdefault("device", -1)
    return fed.Fed.from_problem(prob, **kw)


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "fed.h")).read()
    decl = set(re.findall(r"^\s*(?:fed_status|void|const char \*)\s*(fed_\w+)\s*\(", hdr, re.M))
    assert {"fed_create", "fed_step", "fed_get_temperature"} <= decl
    assert decl == set(fed.EXPORTED)
    for name in decl:
        assert hasattr(lib, name), name
        getattr(lib, name)


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg3", "jitter_aniso"])
def test_dt_crit_matches_oracle(lib, oracle_lib, case):
    if case == "jitter_aniso":
        p = box_problem(6, 5, 4, material=Material(3.0, 5.0, 0.001, random_spd_tensor(4), 0.002), jitter=0.2, seed=3)
        p.T_lo, p.T_hi = 10.0, 150.0
    else:
        p = make_config(int(case[-1]), n=5)
    f = dry(p)
    info = f.info()
    ref = oracle.dt_crit(p, p.T_lo, p.T_hi)
    assert info["dt_crit"] == pytest.approx(ref, rel=1e-12)
    assert info["dt"] == pytest.approx(0.9 * ref, rel=1e-12)


def test_explicit_dt_used_verbatim(lib):
    p = make_config(2, n=4)
    f = dry(p, dt=0.0123456789)
    assert f.info()["dt"] == 0.0123456789


def test_lumped_volume_and_coef_match_oracle(lib, oracle_lib):
    p = box_problem(5, 4, 3, L=(0.1, 0.2, 0.3), material=Material(7800.0, 460.0, 0.0, (50, 50, 50, 0, 0, 0), 0.0),
                    jitter=0.2, seed=1, shuffle_seed=5)
    dt = 0.5
    f = dry(p, dt=dt)
    V, coef = f.debug_nodal()
    o = oracle.Oracle(p, dt)
    M = o.mass()
    np.testing.assert_allclose(V * 7800.0, M, rtol=1e-13)
    np.testing.assert_allclose(coef, dt / (M * 460.0), rtol=1e-13)


@pytest.mark.parametrize("chunk", [0, 32, 64, 256])
@pytest.mark.parametrize("shuffle", [None, 11])
def test_plan_is_valid_partition_and_colouring(lib, chunk, shuffle):
    p = box_problem(13, 11, 9, L=(1.3, 1.1, 0.9), jitter=0.15, seed=2, shuffle_seed=shuffle,
                    side_bc={"z0": 0}, face_bcs=[FaceBC(BC_FLUX, q=1.0)], dirichlet={"x0": 1.0})
    f = dry(p, chunk_elems=chunk)
    info = f.info()
    d = f.debug_plan()
    el = d["slot_elem"]
    real = el >= 0
    assert np.array_equal(np.sort(el[real]), np.arange(p.n_elems))          # every element once
    nm = d["node_map"]
    assert (nm >= 0).all() and np.unique(nm).size == p.n_nodes              # injective node map
    assert nm.max() < info["n_nodes_local"]
    conn = p.conn
    ch, co = d["slot_chunk"][real], d["slot_color"][real]
    maxl = info["chunk_elems"] + info["chunk_elems"] // 2 + 128 - 7
    for c in np.unique(ch):
        sel = el[real][ch == c]
        assert sel.size <= info["chunk_elems"]
        assert np.unique(conn[sel]).size <= maxl
        for col in np.unique(co[ch == c]):
            e = sel[co[ch == c] == col]
            nodes = conn[e].ravel()
            assert np.unique(nodes).size == nodes.size, "colour phase with a shared node"
    # chunk-interior nodes are touched by exactly one chunk and carry no BC
    n_int = info["n_interior"]
    slot_chunk_of_elem = np.empty(p.n_elems, np.int64)
    slot_chunk_of_elem[el[real]] = ch
    chunks_of_node = {}
    for e in range(p.n_elems):
        for n in conn[e]:
            chunks_of_node.setdefault(int(n), set()).add(int(slot_chunk_of_elem[e]))
    bc_nodes = set(p.faces[p.face_bc >= 0].ravel().tolist()) | set(p.dir_nodes.tolist())
    for n in range(p.n_nodes):
        if nm[n] < n_int:
            assert len(chunks_of_node[n]) == 1 and n not in bc_nodes
    if info["max_colors"] > 8 or shuffle is None:
        pass
    assert info["max_colors"] <= 32


def test_structured_grid_gets_eight_balanced_colours(lib):
    p = make_config(5, n=32)
    info = dry(p, chunk_elems=512).info()
    assert info["max_colors"] == 8
    assert info["n_chunks"] == 32 ** 3 // 512


def test_errors(lib):
    p = box_problem(2, 2, 2)
    bad = box_problem(2, 2, 2)
    bad.conn = bad.conn[:, [4, 5, 6, 7, 0, 1, 2, 3]].copy()     # inverted elements
    with pytest.raises(fed.FedError) as e:
        dry(bad)
    assert e.value.status == fed.FED_ERR_MESH
    oob = box_problem(2, 2, 2)
    oob.conn = oob.conn.copy()
    oob.conn[3, 2] = 10_000
    with pytest.raises(fed.FedError) as e:
        dry(oob)
    assert e.value.status == fed.FED_ERR_MESH
    orphan = box_problem(2, 2, 2)
    orphan.xyz = np.vstack([orphan.xyz, [[9.0, 9.0, 9.0]]])
    orphan.T0 = np.append(orphan.T0, 0.0)
    with pytest.raises(fed.FedError) as e:
        dry(orphan)
    assert e.value.status == fed.FED_ERR_MESH
    with pytest.raises(fed.FedError) as e:
        dry(p, precision=16)
    assert e.value.status == fed.FED_ERR_INVALID
    notspd = box_problem(2, 2, 2, material=Material(1.0, 1.0, 0.0, (1.0, -1.0, 1.0, 0, 0, 0), 0.0))
    with pytest.raises(fed.FedError) as e:
        dry(notspd)
    assert e.value.status == fed.FED_ERR_INVALID
    empty = box_problem(2, 2, 2)
    empty.conn = empty.conn[:0].copy()                            # no elements
    with pytest.raises(fed.FedError) as e:
        dry(empty)
    assert e.value.status == fed.FED_ERR_INVALID
    for kw in (dict(dt=float("nan")), dict(dt=float("inf")), dict(chunk_elems=33), dict(chunk_elems=8192)):
        with pytest.raises(fed.FedError) as e:
            dry(p, **kw)
        assert e.value.status == fed.FED_ERR_INVALID, kw
    assert dry(p, dt=-1.0).info()["dt"] == pytest.approx(0.9 * dry(p).info()["dt_crit"], rel=1e-15)
    f = dry(p)
    with pytest.raises(fed.FedError) as e:
        f.step(1)
    assert e.value.status == fed.FED_ERR_STATE
    assert "dry-run" in fed.fed_last_error()
    # device-memory hook: both functions or neither; the wait bound must be a number
    o = fed.options(device=-1)
    o.dev_alloc = fed.DEV_ALLOC(lambda n, d, c: None)
    with pytest.raises(fed.FedError) as e:
        fed.Fed.from_problem(p, opts=o)
    assert e.value.status == fed.FED_ERR_INVALID and "dev_free" in fed.fed_last_error()
    with pytest.raises(fed.FedError) as e:
        dry(p, wait_timeout_s=float("nan"))
    assert e.value.status == fed.FED_ERR_INVALID


def test_destroy_null_is_noop(lib):
    lib.fed_destroy(None)


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_slab_partition_dry_run(lib, nranks):
    """Every element on exactly one rank; interface nodes shared by exactly the
    two neighbouring ranks, in the same (caller-id sorted) order on both."""
    n = 8
    p = make_config(5, n=n)
    owners = np.zeros(p.n_elems, np.int64)
    lists = []
    for r in range(nranks):
        f = dry(p, rank=r, nranks=nranks)
        info = f.info()
        d = f.debug_plan()
        el = d["slot_elem"][d["slot_elem"] >= 0]
        owners[el] += 1
        nm = d["node_map"]
        lo, hi = info["n_interior"], info["n_interior"] + info["n_interface"]
        ids = np.nonzero((nm >= lo) & (nm < hi))[0]
        ids = ids[np.argsort(nm[ids])]
        lists.append(ids)
        # slab of n/nranks layers (+ the interface planes)
        z = p.xyz[np.nonzero(nm >= 0)[0], 2]
        assert z.max() - z.min() <= 0.1 / nranks + 1e-12 + 0.1 / n
    assert np.all(owners == 1)
    plane = (n + 1) ** 2
    assert lists[0].size == plane and lists[-1].size == plane
    for r in range(nranks - 1):
        # rank r's upper group == rank r+1's lower group, same order
        up = lists[r][-plane:]
        low = lists[r + 1][:plane]
        assert np.array_equal(up, low)
        assert np.all(np.diff(up) > 0)


@pytest.mark.parametrize("P", [2, 3, 5])
@pytest.mark.parametrize("transport", [0, 1])
def test_local_group_dry_run(lib, P, transport):
    """local_ranks = P plans the P slabs of a P-rank run inside one context: the
    totals add up to the mesh plus the duplicated interface planes."""
    n = 10
    p = make_config(5, n=n)
    g = dry(p, local_ranks=P, transport=transport)
    info = g.info()
    plane = (n + 1) ** 2
    assert info["nranks"] == P and info["rank"] == -1
    assert info["n_elems_local"] == p.n_elems
    assert info["n_nodes_local"] >= p.n_nodes + (P - 1) * plane     # + alignment padding
    assert info["n_interface"] == 2 * (P - 1) * plane
    assert info["n_elems_global"] == p.n_elems and info["n_nodes_global"] == p.n_nodes
    # every slab agrees with the stand-alone rank contexts of a real P-GPU run
    single = [dry(p, rank=r, nranks=P).info() for r in range(P)]
    assert sum(s["n_chunks"] for s in single) == info["n_chunks"]
    assert sum(s["n_interface"] for s in single) == info["n_interface"]
    with pytest.raises(fed.FedError) as e:
        g.debug_plan()
    assert e.value.status == fed.FED_ERR_STATE
    with pytest.raises(fed.FedError) as e:
        g.step(1)
    assert e.value.status == fed.FED_ERR_STATE


def test_local_group_errors(lib):
    p = make_config(5, n=6)
    for kw in (dict(local_ranks=2, nranks=2, rank=0),          # group inside a multi-process run
               dict(local_ranks=2, transport=7),                 # unknown transport
               dict(nranks=2, rank=0, transport=7),
               dict(local_ranks=2, transport=1, scatter=1),      # PEER needs a chunk scatter
               dict(local_ranks=9)):                            # more slabs than z layers allow
        with pytest.raises(fed.FedError) as e:
            dry(p, **kw)
        assert e.value.status == fed.FED_ERR_INVALID, kw


# ---------------------------------------------------------------- tet4 (NEXT-1)
def test_tet_dt_volume_and_plan(lib, oracle_lib):
    from fed_inputs import tet_box_problem
    p = tet_box_problem(5, 4, 6, L=(0.5, 0.4, 0.6), material=Material(3.0, 5.0, 0.001, random_spd_tensor(8), 0.002),
                        jitter=0.2, seed=5, shuffle_seed=3, side_bc={"z0": 0}, face_bcs=[FaceBC(BC_FLUX, q=1.0)])
    p.T_lo, p.T_hi = 10.0, 150.0
    f = dry(p, dt=0.25)
    info = f.info()
    assert info["nodes_per_elem"] == 4
    assert info["dt_crit"] == pytest.approx(oracle.dt_crit(p, 10.0, 150.0), rel=1e-11)
    V, coef = f.debug_nodal()
    o = oracle.Oracle(p, 0.25)
    np.testing.assert_allclose(V * 3.0, o.mass(), rtol=1e-12)
    d = f.debug_plan()
    el = d["slot_elem"]
    assert np.array_equal(np.sort(el[el >= 0]), np.arange(p.n_elems))
    if info["colored"]:
        hdr, col, c16 = f.debug_chunks()
        ch, co = d["slot_chunk"][el >= 0], d["slot_color"][el >= 0]
        for c in np.unique(ch):
            sel = el[el >= 0][ch == c]
            for k in np.unique(co[ch == c]):
                nodes = p.conn[sel[co[ch == c] == k]].ravel()
                assert np.unique(nodes).size == nodes.size


# ---------------------------------------------------------------- dataflow tables (resident / flow modes)
def _touchers_from_plan(p, g):
    """chunks touching every caller node, from the slot -> element map (independent of the tables)"""
    d = g.debug_plan()
    el, ch = d["slot_elem"], d["slot_chunk"]
    m = el >= 0
    nodes = p.conn[el[m]]                               # [slots, npe] caller node ids
    chunks = np.repeat(ch[m], nodes.shape[1])
    pairs = np.unique(np.stack([nodes.ravel(), chunks]), axis=1)
    return d["node_map"], pairs


@pytest.mark.parametrize("case", ["cfg5", "jitter_shuffled", "tet"])
def test_dataflow_tables(lib, case):
    from fed_inputs import tet_box_problem
    if case == "cfg5":
        p = make_config(5, n=16)
    elif case == "jitter_shuffled":
        p = box_problem(12, 10, 9, jitter=0.2, seed=4, shuffle_seed=9, L=(0.07, 0.06, 0.05))
    else:
        p = tet_box_problem(6, 5, 7, jitter=0.2, seed=3, shuffle_seed=5)
    g = dry(p, precision=32)
    t = g.debug_dataflow()
    assert t is not None
    ptr, adj, spl, own = t
    info = g.info()
    nch = info["n_chunks"]
    hdr, _, _ = g.debug_chunks()
    # adjacency: symmetric, no self loops, sorted and unique per chunk
    A = set()
    for c in range(nch):
        row = adj[ptr[c]:ptr[c + 1]]
        assert np.all(np.diff(row) > 0) and c not in row
        A.update((c, int(x)) for x in row)
    assert all((b, a) in A for (a, b) in A)
    # independent touchers of every shared node from the slot map
    node_map, pairs = _touchers_from_plan(p, g)
    N_int = info["n_interior"]
    sp_of_node = node_map[pairs[0]] - N_int
    shared = sp_of_node >= 0
    touch = {}
    for s, c in zip(sp_of_node[shared], pairs[1][shared]):
        touch.setdefault(int(s), set()).add(int(c))
    # every shared node: listed by exactly its touchers, owned by exactly the lowest one
    owners = {}
    listed = {}
    for c in range(nch):
        off, n = hdr[c, 5], hdr[c, 6]
        for j in range(n):
            s = int(spl[off + j])
            if s < 0:
                continue
            listed.setdefault(s, set()).add(c)
            if own[off + j]:
                owners.setdefault(s, []).append(c)
    assert listed == touch
    for s, cs in touch.items():
        assert owners.get(s) == [min(cs)], (s, owners.get(s), cs)
    # chunks are adjacent iff they share a node
    B = set()
    for cs in touch.values():
        B.update((a, b) for a in cs for b in cs if a != b)
    assert A == B


def test_bank_layout_is_conflict_free(lib):
    """Simulated shared-memory conflicts of the colour phases (scripts/bank_sim.py)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bank_sim", os.path.join(ROOT, "scripts", "bank_sim.py"))
    bs = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bs)
    for p in (make_config(5, n=32), make_config(4, n=24)):
        g = dry(p, precision=32, scatter=5, chunk_elems=1024)
        hdr, col, c16 = g.debug_chunks()
        assert bs.simulate(hdr, col, c16, True, max_chunks=40) <= 1.05
        info = g.info()
        # holes of the layout (padding nodes in the interior ranges) stay small
        d = g.debug_plan()
        interior_nodes = int(((d["node_map"] >= 0) & (d["node_map"] < info["n_interior"])).sum())
        assert info["n_interior"] <= 1.10 * interior_nodes + 8 * info["n_chunks"]


@pytest.mark.parametrize("n", [(9, 9, 9), (10, 8, 9), (13, 11, 9), (7, 6, 5)])
def test_parity_colouring_on_non_cubic_cells(lib, n):
    """Per-axis quantisation: structured boxes with non-cubic, jittered cells keep
    the 8 parity colours (<= 128 elements per colour) the fast paths need."""
    p = box_problem(*n, L=(0.07, 0.06, 0.05), jitter=0.2, seed=3)
    g = dry(p, precision=32)
    info = g.info()
    assert info["max_colors"] == 8
    hdr, col, _ = g.debug_chunks()
    assert np.diff(col[:, :9], axis=1).max() <= 128


def test_temperature_dependence_classification(lib):
    """The planner's choice of material evaluation: TI (0), linear laws (1), general
    tables (2), tables of <= 2 points as clamped linear laws (3)."""
    from fed_inputs import Material, random_spd_tensor
    D = random_spd_tensor(1, 20, 80)
    cases = [(Material(1.0, 2.0, 0.0, D, 0.0), 0), (Material(1.0, 2.0, 0.001, D, 0.0), 1),
             (Material(1.0, 2.0, 0.0, D, 0.002), 1),
             (Material(1.0, 2.0, 0.0, D, 0.0, k_table=((1.0, 2.0, 3.0), (1.0, 2.0, 2.5))), 2),
             (Material(1.0, 2.0, 0.0, D, 0.0, c_table=((1.0, 2.0, 3.0), (1.0, 2.0, 2.5)),
                       k_table=((1.0, 2.0), (1.0, 3.0))), 2),
             (Material(1.0, 2.0, 0.0, D, 0.0, k_table=((1.0, 2.0), (1.0, 3.0))), 3),
             (Material(1.0, 2.0, 0.001, D, 0.0, k_table=((5.0,), (1.5,))), 3),
             (Material(1.0, 2.0, 0.0, D, 0.0, k_table=((0.0, 9.0), (1.0, 3.0)), c_table=((2.0, 4.0), (5.0, 7.0))), 3)]
    for mat, td in cases:
        p = box_problem(2, 2, 2, material=mat)
        p.T_lo, p.T_hi = 0.0, 10.0
        assert dry(p).info()["temperature_dependent"] == td, (mat, td)


def test_packed_connectivity_chunk_limit(lib):
    """The streaming hex colour-phase kernel reads 12-bit packed chunk-local positions
    (<= 4096 local nodes per chunk, i.e. chunk_elems <= 2624): larger chunks take the
    compare-and-swap mode under AUTO (which already prefers it for colours of more than
    128 elements) and are refused for an explicit CHUNK_REGC."""
    p = make_config(5, n=40)
    R = fed.FED_SCATTER_CHUNK_REGC
    assert dry(p, chunk_elems=2048, scatter=R).info()["scatter"] == R
    assert dry(p, chunk_elems=4096, resident=-1).info()["scatter"] == fed.FED_SCATTER_CHUNK_REG
    with pytest.raises(fed.FedError) as e:
        dry(p, chunk_elems=4096, scatter=fed.FED_SCATTER_CHUNK_REGC)
    assert e.value.status == fed.FED_ERR_INVALID and "12-bit" in fed.fed_last_error()


@pytest.mark.parametrize("bnd_first", ["1", "0"])
def test_special_node_order(lib, bnd_first, monkeypatch):
    """The shared ("special") region is laid out in two groups, each in one piece:
    nodes with face BCs or Dirichlet values, then plain chunk-shared nodes (the
    default, so the node kernel's slow boundary blocks start in its first wave),
    or the reverse with FED_BND_FIRST=0 (the round-1 order, kept for A/B)."""
    monkeypatch.setenv("FED_BND_FIRST", bnd_first)
    p = box_problem(13, 11, 9, L=(1.3, 1.1, 0.9), jitter=0.15, seed=2,
                    side_bc={"z0": 0, "x1": 0}, face_bcs=[FaceBC(BC_CONV, h=25.0, T_inf=20.0)],
                    dirichlet={"x0": 1.0})
    f = dry(p, chunk_elems=128)
    info = f.info()
    nm = f.debug_plan()["node_map"]
    n_int = info["n_interior"]
    bc_nodes = set(p.faces[p.face_bc >= 0].ravel().tolist()) | set(p.dir_nodes.tolist())
    sp = np.flatnonzero(nm >= n_int)
    order = np.argsort(nm[sp])
    is_bnd = np.array([int(n) in bc_nodes for n in sp[order]])
    assert is_bnd.any() and (~is_bnd).any()
    first = is_bnd if bnd_first == "1" else ~is_bnd
    k = int(first.sum())
    assert first[:k].all() and not first[k:].any(), "special groups interleaved"
    assert all(nm[n] >= n_int for n in bc_nodes)
