#!/usr/bin/env python
"""Cost of the NEXT rows on the headline mesh (cfg5, 384^3 hex8, fp32, one GPU):
tabulated k(T)/c(T) (NEXT-2, the paper's Sec. 4.2.2 tables), concentrated face
loads (NEXT-3) and the steady-state monitor (NEXT-4, a max-|dT| check every
`check_every` steps) against the plain cfg5 step.  Wall clock of K graph-launched
steps after warm-up, synchronised on both sides.

    python scripts/next_rows_perf.py [--steps 200] [--n 384]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--only", default=None, help="run one variant: base | tables | tables4 | concentrated | steady100 | steady10")
    a = ap.parse_args()
    import torch
    from fed_inputs import make_config, paper_td_material
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build

    build()
    K = a.steps

    def run(name, p, steady=0, key=None):
        if a.only and key != a.only:
            return
        g = fed.Fed.from_problem(p, precision=a.precision, device=0)
        g.step(20)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if steady:
            n, _ = g.run_until_steady(tol=1e-30, max_steps=K, check_every=steady)   # never converges: K monitored steps
            assert n == K, n
        else:
            g.step(K)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        info = g.info()
        g.close()
        print(json.dumps({"variant": name, "precision": a.precision, "elements": p.n_elems, "steps": K,
                          "ms_per_step": 1e3 * wall / K, "elem_steps_per_s": p.n_elems * K / wall,
                          "scatter": info.get("scatter"), "fail_step": info["fail_step"]}), flush=True)

    p = make_config(5, n=a.n)
    run("cfg5", p, key="base")
    pt = make_config(5, n=a.n)
    m = paper_td_material()
    # make_config shares one Material object between calls: replace, never mutate
    pt.material = dataclasses.replace(pt.material, k_table=m.k_table, c_table=m.c_table)
    pt.T_lo, pt.T_hi = 20.0, 100.0
    run("cfg5 + tabulated k(T), c(T) (NEXT-2; the paper's 2-point tables)", pt, key="tables")
    p4 = make_config(5, n=a.n)
    # general tables (> 2 points: the table path with per-node phi in shared memory)
    p4.material = dataclasses.replace(p4.material, k_table=((20.0, 40.0, 70.0, 100.0), (1.0, 1.05, 1.2, 1.3)),
                                      c_table=((20.0, 60.0, 100.0), (460.0, 480.0, 500.0)))
    p4.T_lo, p4.T_hi = 20.0, 100.0
    run("cfg5 + tabulated k(T), c(T) with 4 / 3 points (NEXT-2 general tables)", p4, key="tables4")
    pc = make_config(5, n=a.n)
    for b in pc.face_bcs:
        b.area_mode = 1
    run("cfg5 + concentrated face loads (NEXT-3)", pc, key="concentrated")
    run("cfg5 + steady-state check every 100 steps (NEXT-4)", make_config(5, n=a.n), steady=100, key="steady100")
    run("cfg5 + steady-state check every 10 steps (NEXT-4)", make_config(5, n=a.n), steady=10, key="steady10")


if __name__ == "__main__":
    main()
