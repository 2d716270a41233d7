"""World-size-2 CPU test of the multi-GPU (z-slab) host logic with gloo.

Each rank plans its slab with libfed in dry-run mode (device = -1, the same
planner the GPU path uses), computes the partial internal loads of ITS
elements with the oracle, exchanges the interface slices over gloo in the
library's interface order, and combines them lower-rank-first exactly as the
node kernel does.  The combined loads must equal the single-domain oracle,
and both ranks must hold bit-identical interface values.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sub_problem(prob, elems):
    from fed_inputs import Problem
    ce = prob.conn[elems]
    nodes = np.unique(ce)
    loc = np.full(prob.n_nodes, -1, np.int64)
    loc[nodes] = np.arange(nodes.size)
    sub = Problem("slab", prob.xyz[nodes].copy(), loc[ce].astype(np.int32), np.zeros((0, 4), np.int32),
                  np.zeros(0, np.int32), [], np.zeros(0, np.int32), np.zeros(0), None, prob.T0[nodes].copy(),
                  prob.material, 1, prob.precisions, prob.T_lo, prob.T_hi)
    return sub, nodes


def _worker(rank, world, port, n, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from fed_inputs import make_config, random_field
        from paper_1909_03355_b200 import fed
        p = make_config(5, n=n)
        T = 20 + random_field(p.n_nodes, 3, 0, 80)
        g = fed.Fed.from_problem(p, device=-1, rank=rank, nranks=world)
        info = g.info()
        d = g.debug_plan()
        nm = d["node_map"]
        my_elems = np.sort(d["slot_elem"][d["slot_elem"] >= 0])
        lo, n_if = info["n_interior"], info["n_interface"]
        if_ids = np.nonzero((nm >= lo) & (nm < lo + n_if))[0]
        if_ids = if_ids[np.argsort(nm[if_ids])]          # library order
        # partial loads of this rank's elements (oracle on the slab sub-mesh)
        sub, nodes = _sub_problem(p, my_elems)
        o = oracle.Oracle(sub, 1.0)
        F_sub, _ = o.loads(T[nodes])
        F_part = np.zeros(p.n_nodes)
        F_part[nodes] = F_sub
        mine = torch.from_numpy(F_part[if_ids].copy())
        other = torch.zeros_like(mine)
        peer = 1 - rank
        ids_other = torch.zeros(if_ids.size, dtype=torch.int64)
        if rank == 0:
            dist.send(torch.from_numpy(if_ids.astype(np.int64)), peer)
            dist.send(mine, peer)
            dist.recv(ids_other, peer)
            dist.recv(other, peer)
        else:
            dist.recv(ids_other, peer)
            dist.recv(other, peer)
            dist.send(torch.from_numpy(if_ids.astype(np.int64)), peer)
            dist.send(mine, peer)
        same_order = bool(np.array_equal(ids_other.numpy(), if_ids))
        # combine lower rank first (node_kernel order)
        comb = (other.numpy() + mine.numpy()) if rank == 1 else (mine.numpy() + other.numpy())
        # reference: single-domain oracle
        o_all = oracle.Oracle(p, 1.0)
        F_all, _ = o_all.loads(T)
        err = float(np.abs(comb - F_all[if_ids]).max() / np.abs(F_all).max())
        # interior (non-interface) nodes of the slab need no exchange
        own = np.setdiff1d(nodes, if_ids)
        err_own = float(np.abs(F_part[own] - F_all[own]).max() / np.abs(F_all).max())
        dist.barrier()
        q.put((rank, same_order, err, err_own, comb.tobytes(), if_ids.size, my_elems.size))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.parametrize("n", [8, 12])
def test_two_rank_interface_exchange_gloo(oracle_lib, n):
    import torch.multiprocessing as mp
    from paper_1909_03355_b200.build import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
    res = sorted(res, key=lambda r: r[0])
    for r in res:
        assert r[1] != "error", r
    (_, o0, e0, w0, c0, n0, m0), (_, o1, e1, w1, c1, n1, m1) = res
    assert o0 and o1, "interface order differs between ranks"
    assert n0 == n1 == (n + 1) ** 2
    assert m0 + m1 == n ** 3
    assert e0 <= 1e-13 and e1 <= 1e-13
    assert w0 <= 1e-13 and w1 <= 1e-13
    assert c0 == c1, "interface loads not bit-identical on both ranks"


def _gather_worker(rank, world, port, n, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from fed_inputs import make_config, random_field
        from paper_1909_03355_b200 import fed
        p = make_config(4, n=n)                       # jittered + renumbered: caller ids are not z-ordered
        g = fed.Fed.from_problem(p, device=-1, rank=rank, nranks=world, precision=32)
        off, ids, pack = g.debug_gather()
        d = g.debug_plan()
        nm = d["node_map"]
        my_elems = d["slot_elem"][d["slot_elem"] >= 0]
        # the fed_get_temperature algorithm on host data: internal field -> packed own slice
        # -> all-gather (padded to the largest slice) -> caller order
        field = 20 + random_field(p.n_nodes, 4, 0, 80)
        node_global = np.full(int(nm.max()) + 1, -1, np.int64)
        node_global[nm[nm >= 0]] = np.nonzero(nm >= 0)[0]
        T_int = field[node_global]
        stride = int(np.diff(off).max())
        send = torch.zeros(stride, dtype=torch.float64)
        send[:pack.size] = torch.from_numpy(T_int[pack])
        recv = [torch.zeros(stride, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, send)
        out = np.full(p.n_nodes, np.nan)
        for r in range(world):
            out[ids[off[r]:off[r + 1]]] = recv[r].numpy()[:off[r + 1] - off[r]]
        touched = [None] * world
        dist.all_gather_object(touched, np.unique(p.conn[my_elems]).tolist())
        layouts = [None] * world
        dist.all_gather_object(layouts, (off.tolist(), ids.tobytes()))
        dist.barrier()
        q.put((rank, bool(np.array_equal(out, field)), touched, layouts, pack.size, off.tolist(),
               bool(np.array_equal(nm[ids[off[rank]:off[rank + 1]]], pack))))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


def test_multi_rank_readout_layout_gloo():
    """fed_get_temperature with nranks > 1 (fed.h): every node is packed by exactly
    one rank -- the lowest rank whose elements touch it -- in increasing caller id,
    all ranks agree on the layout, and one all-gather of the packed slices
    reconstructs the full field (3 ranks, gloo, renumbered jittered mesh)."""
    import torch.multiprocessing as mp
    from paper_1909_03355_b200.build import build
    build()
    world, n = 3, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    N = (n + 1) ** 3
    for rank, ok, touched, layouts, npack, off, own in res:
        assert ok, f"rank {rank}: gathered field differs"
        assert own, f"rank {rank}: pack list is not its slice"
        assert all(l == layouts[0] for l in layouts), "ranks disagree on the readout layout"
        ids = np.frombuffer(layouts[0][1], np.int32)
        assert np.array_equal(np.sort(ids), np.arange(N))
        owner = np.full(N, world)
        for r in range(world - 1, -1, -1):
            owner[np.asarray(touched[r])] = r
        for r in range(world):
            sl = ids[off[r]:off[r + 1]]
            assert np.all(owner[sl] == r) and np.all(np.diff(sl) > 0)
        assert npack == off[rank + 1] - off[rank]
