#!/usr/bin/env python
"""Per-rank cost of the z-slab partition of cfg5, measured on ONE GPU.

    python scripts/slab_projection.py [--n 384] [--ranks 1 2 4 8] [--steps 50] [--chunk 1024]

For each P, one context holds the P slabs of a P-GPU run (fed_options.local_ranks,
PEER transport).  Each slab is planned, stored and launched exactly as on its
own GPU; with per-kernel CUDA-event timing on, fed_get_rank_timing gives every
rank's element + node kernel time per step.  In a P-GPU run the ranks run
concurrently, so the step takes about max_r(rank time) + the exchange latency;
this script reports that PROJECTION (labelled as such) next to the measured
1-GPU step, and the measured time of the whole emulated group (all slabs back
to back on one GPU, CUDA graphs), whose excess over the 1-GPU step is the
partitioning overhead (duplicated interface nodes, extra launches).
It is not a multi-GPU measurement: this run has one GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def group_graph_ms(g, K, stream):
    """K steps replayed from CUDA graphs, CUDA events on the library's stream."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    g.step(K)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--chunk", type=int, default=0, help="fed_options.chunk_elems (0 = auto)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build

    build()
    prob = make_config(5, n=args.n)
    E = prob.n_elems
    rows = []
    base = base_alone = None
    for P in args.ranks:
        t0 = time.perf_counter()
        stream = torch.cuda.Stream()
        kw = dict(precision=args.precision, device=0, chunk_elems=args.chunk, resident=-1,
                  stream=stream.cuda_stream)
        tr = fed.FED_TRANSPORT_PEER if args.transport == "peer" else fed.FED_TRANSPORT_NCCL
        if P > 1:
            kw.update(local_ranks=P, transport=tr)
        g = fed.Fed.from_problem(prob, **kw)
        create_s = time.perf_counter() - t0
        g.step(16)
        torch.cuda.synchronize()
        # measured: the whole group back to back on one GPU (graphs), wall of K steps
        K = args.steps
        group_ms = group_graph_ms(g, K, stream)
        # per-rank kernel times (eager, CUDA events on the launching stream)
        g.set_timing(True)
        g.step(K)
        per = []
        for r in range(P):
            t = g.rank_timing(r)
            per.append({"rank": r, "element_ms": t["element_ms"] / K, "node_ms": t["node_ms"] / K,
                        "element_launches_per_step": t["element_launches"] / K})
        g.set_timing(False)
        info = g.info()
        # each slab's own kernel sequence replayed ALONE in a CUDA graph (what the rank
        # launches on its own GPU, neighbour waits skipped): the per-GPU step time
        alone = [g.debug_time_rank(r, K) for r in range(P)] if P > 1 else [group_graph_ms(g, K, stream)]
        g.close()
        rank_ms = [p["element_ms"] + p["node_ms"] for p in per]
        proj = max(rank_ms)
        if P == 1:
            base = proj
            base_alone = alone[0]
        row = {"P": P, "elements": E, "precision": args.precision, "create_s": round(create_s, 1),
               "group_ms_per_step_1gpu": group_ms,
               "rank_kernel_ms_per_step": rank_ms,
               "projected_ms_per_step": proj,
               "projected_elem_steps_per_s": E / (proj / 1e3),
               "projected_efficiency_vs_P1": (base / (P * proj)) if base else None,
               "alone_ms_per_step": alone, "projected_alone_ms_per_step": max(alone),
               "projected_alone_efficiency_vs_P1": (base_alone / (P * max(alone))) if base_alone else None,
               "per_rank": per, "n_interface_total": info["n_interface"],
               "kernel_launches_per_step": info["kernel_launches_per_step"],
               "note": "projection: max over ranks of measured per-rank kernel time; excludes exchange latency"}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
