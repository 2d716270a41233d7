"""Helpers for GPU-vs-oracle parity tests (test infrastructure).

The oracle always receives generator-produced inputs (fed_inputs) and a dt
computed by the oracle itself; nothing flows from the CUDA path into it.
"""
from __future__ import annotations

import numpy as np

import oracle
from fed_inputs import Problem

TOL = {64: 1e-11, 32: 1e-4}   # north_star: max relative error (inf-norm / max|T_oracle|), reading 8c-19


def rel_err(T, ref):
    return float(np.abs(T - ref).max() / max(np.abs(ref).max(), 1e-300))


def oracle_dt(prob, factor=None):
    return (prob.dt_factor if factor is None else factor) * oracle.dt_crit(prob, prob.T_lo, prob.T_hi)


def trajectory_parity(prob, precision, checkpoints, dt=None, T_start=None, **opt_kw):
    """Run GPU (through the C ABI) and oracle side by side; return
    [(step, rel_err)] at the checkpoints (cumulative step counts)."""
    from paper_1909_03355_b200 import fed
    dt = oracle_dt(prob) if dt is None else dt
    o = oracle.Oracle(prob, dt)
    g = fed.Fed.from_problem(prob, precision=precision, dt=dt, device=0, **opt_kw)
    if T_start is not None:
        o.set_T(_with_dirichlet(prob, T_start))
        g.set_temperature(T_start)
    out = []
    done = 0
    for k in checkpoints:
        o.step(k - done)
        g.step(k - done)
        done = k
        out.append((k, rel_err(g.temperature(), o.T())))
    g.close()
    return out


def multi_parity(prob, variants, checkpoints, dt=None):
    """One oracle trajectory against several GPU contexts (precision, options)
    stepped side by side; returns {variant index: [(step, rel_err)]} and the
    contexts' fed_info dicts (taken after creation)."""
    from paper_1909_03355_b200 import fed
    dt = oracle_dt(prob) if dt is None else dt
    o = oracle.Oracle(prob, dt)
    gs = [fed.Fed.from_problem(prob, precision=prec, dt=dt, device=0, **kw) for prec, kw in variants]
    infos = [g.info() for g in gs]
    out = {i: [] for i in range(len(gs))}
    done = 0
    for k in checkpoints:
        o.step(k - done)
        ref = o.T()
        for i, g in enumerate(gs):
            g.step(k - done)
            out[i].append((k, rel_err(g.temperature(), ref)))
        done = k
    for g in gs:
        g.close()
    return out, infos


def _with_dirichlet(prob, T):
    T = np.array(T, dtype=np.float64, copy=True)
    if prob.dir_nodes.size:
        T[prob.dir_nodes] = prob.dir_T
    return T


def patch_problem(prob: Problem, sample: np.ndarray):
    """Sub-problem made of every element and boundary face touching the
    sampled nodes, renumbered locally.  The sampled nodes keep their full
    neighbourhood, so one oracle step on the patch reproduces their update
    exactly.  Returns (sub_problem, local ids of the samples, global ids of
    the patch nodes)."""
    sample = np.unique(np.asarray(sample, dtype=np.int64))
    touch = np.isin(prob.conn, sample).any(axis=1)
    ce = prob.conn[touch]
    nodes = np.unique(ce)
    loc = np.full(prob.n_nodes, -1, np.int64)
    loc[nodes] = np.arange(nodes.size)
    conn = loc[ce].astype(np.int32)
    if prob.faces.size:
        ft = np.isin(prob.faces, sample).any(axis=1)
        faces = loc[prob.faces[ft]].astype(np.int32)
        face_bc = prob.face_bc[ft].copy()
        assert (faces >= 0).all()
    else:
        faces = np.zeros((0, 4), np.int32)
        face_bc = np.zeros(0, np.int32)
    dmask = np.isin(prob.dir_nodes, nodes)
    sub = Problem(prob.name + "_patch", prob.xyz[nodes].copy(), conn, faces, face_bc, prob.face_bcs,
                  loc[prob.dir_nodes[dmask]].astype(np.int32), prob.dir_T[dmask].copy(),
                  None if prob.q_vol is None else prob.q_vol[nodes].copy(), prob.T0[nodes].copy(),
                  prob.material, 1, prob.precisions, prob.T_lo, prob.T_hi, prob.dt_factor)
    return sub, loc[sample], nodes
