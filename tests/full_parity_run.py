#!/usr/bin/env python
"""Full-length parity runs of the BASELINE configs the oracle can finish in
minutes: cfg1 (10^3, 2000 steps, fp64) and cfg2 (64^3, 10 000 steps, fp32 and
fp64), GPU (through the C ABI, default execution mode) against the fp64 oracle
on the same seeded inputs and the same dt, at checkpoints along the run.

    python tests/full_parity_run.py [--out profiles/r1_full_parity.jsonl]

(Test infrastructure: lives under tests/ because it runs the oracle; not collected by pytest.)

Metric (reading 8c-19): max_n |T_gpu - T_oracle| / max_n |T_oracle|.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TOL = {64: 1e-11, 32: 1e-4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import oracle
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build
    build()
    oracle.build_oracle()
    runs = [(1, [64], [1, 10, 100, 500, 2000]), (2, [32, 64], [1, 100, 1000, 5000, 10000])]
    rows = []
    for cfg, precs, checks in runs:
        p = make_config(cfg)
        dt = p.dt_factor * oracle.dt_crit(p, p.T_lo, p.T_hi)
        o = oracle.Oracle(p, dt)
        gs = {prec: fed.Fed.from_problem(p, precision=prec, dt=dt, device=0) for prec in precs}
        done = 0
        t_or = 0.0
        for k in checks:
            t0 = time.perf_counter()
            o.step(k - done)
            t_or += time.perf_counter() - t0
            ref = o.T()
            for prec, g in gs.items():
                g.step(k - done)
                T = g.temperature()
                err = float(np.abs(T - ref).max() / np.abs(ref).max())
                row = {"cfg": cfg, "precision": prec, "step": k, "rel_err": err, "tol": TOL[prec],
                       "ok": err <= TOL[prec], "mode": "resident" if g.info()["resident"] else "streaming",
                       "Tmin": float(ref.min()), "Tmax": float(ref.max())}
                rows.append(row)
                print(json.dumps(row), flush=True)
            done = k
        print(json.dumps({"cfg": cfg, "oracle_seconds": t_or, "elements": p.n_elems, "steps": done}), flush=True)
        for g in gs.values():
            g.close()
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    assert all(r["ok"] for r in rows), "parity failure"


if __name__ == "__main__":
    main()
