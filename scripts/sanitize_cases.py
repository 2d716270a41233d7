#!/usr/bin/env python
"""Small runs of every execution mode of libfed.so, for the checked build.

    FED_LIB=paper_1909_03355_b200/libfed_checked.so python scripts/sanitize_cases.py --case CASE

compute-sanitizer is closed on this pool (runs under it left GPUs needing a
reset), so libfed_checked.so (-DFED_DEVICE_CHECKS) bounds-checks every
plan-driven index on the device and checks colour phases for write conflicts;
fed_step fails with FED_ERR_CUDA if a check fires.

Cases (each a few steps on a small mesh, through the C ABI; the result is
checked for finiteness and against the streaming path where both apply, no
oracle involved):
  stream      cfg5-shaped 16^3 mesh, streaming element_chunk_kernel + node_kernel
  stream64    same in fp64
  resident    cfg1 (10^3), resident_kernel (cooperative, per-chunk dataflow)
  peer        cfg5-shaped 16^3 mesh as a 4-slab local rank group, PEER transport
  nccl        same, NCCL-transport group (device-copy exchange)
  tables      tabulated k(T), c(T) (TDK 2) streaming
  tet         Kuhn tets, register compare-and-swap chunks
  atomic      ATOMIC / GATHER baselines
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    from fed_inputs import Material, make_config, paper_td_material, paper_tet_problem
    from paper_1909_03355_b200 import fed
    K = a.steps
    ref_kw = {"resident": -1, "graph_steps": -1}

    def run(p, prec=32, **kw):
        if p.name == "cfg5":
            kw.setdefault("dt", 2.0e-3)
        g = fed.Fed.from_problem(p, precision=prec, **kw)
        info = g.info()
        g.step(K)
        T = g.temperature()
        g.close()
        assert np.isfinite(T).all()
        return T, info

    c = a.case
    if c in ("stream", "stream64"):
        p = make_config(5, n=16)
        prec = 64 if c == "stream64" else 32
        T, info = run(p, prec, resident=-1, chunk_elems=256)
        assert info["resident"] == 0
        T2, _ = run(p, prec, resident=-1, chunk_elems=256, graph_steps=-1)
        assert np.abs(T - T2).max() <= 1e-5 * np.abs(T).max()
    elif c == "resident":
        p = make_config(1)
        T, info = run(p, 64, resident=1)
        assert info["resident"] == 1
        T2, _ = run(p, 64, **ref_kw)
        assert np.abs(T - T2).max() <= 1e-12 * max(1.0, np.abs(T).max())
    elif c in ("peer", "nccl"):
        p = make_config(5, n=16)
        tr = fed.FED_TRANSPORT_PEER if c == "peer" else fed.FED_TRANSPORT_NCCL
        T, info = run(p, 32, local_ranks=4, transport=tr, chunk_elems=128)
        T2, _ = run(p, 32, resident=-1, chunk_elems=128)
        assert np.abs(T - T2).max() <= 1e-5 * np.abs(T).max()
    elif c == "tables":
        p = make_config(2, n=12)
        p.material = paper_td_material()
        p.T_lo, p.T_hi = 20.0, 400.0
        T, info = run(p, 32, resident=-1, chunk_elems=128)
    elif c == "tet":
        p = paper_tet_problem(n=8, td=True)
        T, info = run(p, 32, resident=-1)
        T2, _ = run(p, 32, resident=1)
        assert np.abs(T - T2).max() <= 1e-5 * np.abs(T).max()
    elif c == "atomic":
        p = make_config(5, n=12)
        for sc in (1, 6, 7, 8):
            run(p, 32, scatter=sc, resident=-1)
    else:
        raise SystemExit(f"unknown case {c}")
    print(f"case {c}: ok")


if __name__ == "__main__":
    main()
