#!/usr/bin/env python
"""Where the per-rank step time of an 8-slab partition goes (cfg5 fp32, one GPU).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv \
        python scripts/slab_launches.py --steps 3          # kernel durations, one by one
    python scripts/slab_launches.py --summarize L.csv --alone PROJ.jsonl

Under ncu, every kernel of a few eager steps of a P-slab rank group runs alone
(serialised, cold): their durations are the kernels' own time.  The per-rank step
measured by scripts/slab_projection.py (each slab's kernel sequence replayed alone
in a CUDA graph) minus the sum of its kernels' durations is what launch
boundaries, ramps and tails cost per step.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    p = make_config(5)
    g = fed.Fed.from_problem(p, precision=32, device=0, local_ranks=a.ranks, transport=fed.FED_TRANSPORT_PEER,
                             graph_steps=-1, resident=-1)
    g.step(a.steps)
    g.close()


def summarize(a):
    rows = list(csv.reader(open(a.summarize)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i], rows[i + 1:]
    kn, mn, mv, mu = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    dur = []
    for r in data:
        if len(r) > mv and r[mn] == "gpu__time_duration.sum":
            v = float(r[mv].replace(",", ""))
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[mu], 1.0)
            dur.append((r[kn], v))
    elem = [d for n, d in dur if "element_chunk" in n]
    node = [d for n, d in dur if "node_kernel" in n]
    P = a.ranks
    steps = len(elem) // P
    out = {"ranks": P, "steps_profiled": steps,
           "element_us_per_slab": [round(x, 2) for x in elem[-P:]], "node_us_per_slab": [round(x, 2) for x in node[-P:]]}
    kernel_sum = max(e + n for e, n in zip(elem[-P:], node[-P:]))
    out["max_slab_kernel_sum_us"] = round(kernel_sum, 2)
    if a.alone:
        for l in open(a.alone):
            d = json.loads(l)
            if d["P"] == P:
                alone = 1e3 * max(d["alone_ms_per_step"])
                out["alone_step_us"] = round(alone, 2)
                out["boundary_cost_us"] = round(alone - kernel_sum, 2)
                out["note"] = ("alone step = the slab's kernel sequence replayed in a CUDA graph (PDL); kernel durations "
                               "from ncu are cold, serialised launches")
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--summarize", default=None)
    ap.add_argument("--alone", default=None)
    a = ap.parse_args()
    if a.summarize:
        summarize(a)
    else:
        run(a)


if __name__ == "__main__":
    main()
