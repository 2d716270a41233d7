"""Tuning sweep: one problem, several (scatter, chunk, precision) variants.

    python scripts/sweep.py --config 5 --steps 50 --variants chunk:1024,cas:512,...

Prints one JSON line per variant with ms/step and per-kernel times.  Not the
benchmark of record (that is bench.py); used to choose defaults by
measurement.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--variants", default="chunk:0,cas:0,atomic:0")
    a = ap.parse_args()
    import torch

    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build
    build()
    p = make_config(a.config, n=a.n)
    E = p.n_elems
    sc = {"auto": 0, "atomic": 1, "chunk": 2, "cas": 3, "reg": 4, "regc": 5}
    for v in a.variants.split(","):
        name, chunk = v.split(":")
        prec = a.precision
        if name.endswith("64"):
            name, prec = name[:-2], 64
        t0 = time.perf_counter()
        g = fed.Fed.from_problem(p, precision=prec, scatter=sc[name], chunk_elems=int(chunk))
        tc = time.perf_counter() - t0
        g.step(5)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        t0 = time.perf_counter()
        g.step(a.steps)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / a.steps
        g.set_timing(True)
        g.step(a.steps)
        t = g.timing()
        info = g.info()
        g.close()
        print(json.dumps({"variant": v, "precision": prec, "ms_step_wall": 1e3 * wall,
                          "Gelem_s": E / wall / 1e9, "elem_ms": t["element_ms"] / a.steps,
                          "node_ms": t["node_ms"] / a.steps, "chunk": info["chunk_elems"],
                          "n_special": info["n_special"], "n_interior": info["n_interior"],
                          "max_colors": info["max_colors"], "create_s": round(tc, 1)}), flush=True)


if __name__ == "__main__":
    main()
