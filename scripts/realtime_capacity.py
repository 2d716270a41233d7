#!/usr/bin/env python
"""Real-time capacity (the paper's criterion, P:385 / P:369: the largest mesh whose
compute time per step stays within the simulated step, Dt = 5 ms in its Sec. 4.6
runs) of one B200: cfg5's physics (TD k(T) and c(T), convection, Gaussian source)
on n^3 hex8 cubes of growing n, fp32, timed like bench.py (CUDA events on the
library's stream around K graph-replayed steps after warm-up).

    python scripts/realtime_capacity.py [--sizes 384 512 640 768] [--steps 20] [--budget-ms 5]

Prints one JSON line per size and a summary line with the largest measured mesh
within the budget and the element count at which the measured ms/step (linear
in elements on this HBM-bound path) reaches the budget.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[384, 512, 640, 768])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--budget-ms", type=float, default=5.0)
    ap.add_argument("--precision", type=int, default=32)
    a = ap.parse_args()
    import torch
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build
    build()
    rows = []
    for n in a.sizes:
        t0 = time.perf_counter()
        p = make_config(5, n=n)
        stream = torch.cuda.Stream()
        g = fed.Fed.from_problem(p, precision=a.precision, device=0, stream=stream.cuda_stream)  # dt = 0.9 x crit
        create_s = time.perf_counter() - t0
        g.step(16)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.step(a.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        info = g.info()
        row = {"n": n, "elements": p.n_elems, "nodes": p.n_nodes, "precision": a.precision, "ms_per_step": ms,
               "element_steps_per_s": p.n_elems / (ms / 1e3), "within_budget": ms <= a.budget_ms,
               "device_bytes": info["device_bytes"], "create_s": round(create_s, 1), "fail_step": info["fail_step"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
        g.close()
        del p
    ok = [r for r in rows if r["within_budget"]]
    rate = max(r["element_steps_per_s"] for r in rows)
    summary = {"budget_ms": a.budget_ms, "largest_measured_within_budget": max(ok, key=lambda r: r["elements"]) if ok else None,
               "elements_at_budget_from_best_rate": rate * a.budget_ms / 1e3,
               "paper_capacity": "14 164 nodes / 73 025 tets TI, 8 360 nodes / 42 600 elements TD, i7-6700 1 thread (P:369, P:385)"}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
