"""Throughput of every BASELINE config on one GPU (timing only; parity is in
tests/).  One JSON line per (config, precision).

    python scripts/all_configs.py [--configs 1,2,3,4,5] [--max-steps 500]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--max-steps", type=int, default=1000)
    ap.add_argument("--precisions", default="")
    ap.add_argument("--graph-steps", type=int, default=0)
    ap.add_argument("--scatter", type=int, default=0)
    a = ap.parse_args()
    import torch

    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build
    build()
    from fed_inputs import paper_tet_problem, tet_box_problem, K_T
    def problem(name):
        if name.startswith("tet"):          # tetN: Kuhn tet cube of N^3 cells (cfg5 physics, TD)
            n = int(name[3:])
            return tet_box_problem(n, n, n, L=(0.1, 0.1, 0.1), material=K_T, side_bc={"z1": 0, "x0": 0},
                                   face_bcs=[__import__("fed_inputs").FaceBC(2, h=25.0, T_inf=20.0)], T0=20.0,
                                   steps=500, name=name)
        if name.startswith("paper"):        # paper_ti / paper_td: Sec. 4.6 workload shape
            return paper_tet_problem(td=name.endswith("td"))
        return make_config(int(name))
    for cfg in a.configs.split(","):
        p = problem(cfg)
        if cfg.startswith("tet"):
            p.T_lo, p.T_hi = 20.0, 100.0
        precs = [int(x) for x in a.precisions.split(",")] if a.precisions else list(p.precisions)
        for prec in precs:
            t0 = time.perf_counter()
            g = fed.Fed.from_problem(p, precision=prec, graph_steps=a.graph_steps, scatter=a.scatter)
            tc = time.perf_counter() - t0
            K = min(p.steps, a.max_steps)
            g.step(min(20, K))
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            t0 = time.perf_counter()
            g.step(K)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            g.set_timing(True)
            g.step(min(K, 100))
            t = g.timing()
            info = g.info()
            T = g.temperature()
            g.close()
            kk = min(K, 100)
            print(json.dumps({"cfg": cfg, "precision": prec, "elements": p.n_elems, "steps": K,
                              "ms_per_step": 1e3 * wall / K, "elem_steps_per_s": p.n_elems * K / wall,
                              "elem_kernel_us": 1e3 * t["element_ms"] / kk, "node_kernel_us": 1e3 * t["node_ms"] / kk,
                              "chunk": info["chunk_elems"], "n_chunks": info["n_chunks"],
                              "resident": info["resident"],
                              "max_colors": info["max_colors"], "Tmin": float(T.min()), "Tmax": float(T.max()),
                              "fail_step": info["fail_step"], "create_s": round(tc, 2)}), flush=True)


if __name__ == "__main__":
    main()
