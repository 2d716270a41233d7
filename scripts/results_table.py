#!/usr/bin/env python
"""Markdown results table from the round's measurement files:
profiles/r2_all_configs.jsonl (throughput per config), r2_full_parity.jsonl (GPU vs
oracle after the full step count; oracle speed on the box's host core),
r2_ncu_full_cfg5_fp32.json (DRAM traffic of the headline kernels), and the bench lines.

    python scripts/results_table.py [--profiles profiles]
"""
import argparse
import json
import os


def jl(path):
    return [json.loads(l) for l in open(path) if l.strip()] if os.path.exists(path) else []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profiles", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                        "profiles"))
    a = ap.parse_args()
    P = a.profiles
    cfgs = jl(os.path.join(P, "r2_all_configs.jsonl"))
    par = jl(os.path.join(P, "r2_full_parity.jsonl"))
    peak = json.load(open(os.path.join(os.path.dirname(P), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.6) \
        if os.path.exists(os.path.join(os.path.dirname(P), "MEASURED_PEAKS.json")) else 6552.6
    traffic = {}
    for prec in (32, 64):
        f = os.path.join(P, f"r2_ncu_full_cfg5_fp{prec}.json")
        if os.path.exists(f):
            ks = json.load(open(f))["kernels"]
            tot_b, tot_t = 0.0, 0.0
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tsc = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
            for k in ks.values():
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot_b += float(k[m][0].replace(",", "")) * scale[k[m][1]]
                d = k["gpu__time_duration.sum"]
                tot_t += float(d[0].replace(",", "")) * tsc.get(d[1], 1e-6)
            traffic[prec] = (tot_b, tot_t)
    print("| cfg | precision | GPUs | element-steps/s | ms/step | mode | HBM GB/s (ncu, element + node kernels) | % of "
          f"{peak:.0f} GB/s | parity err vs oracle (final step) | oracle ms/step (1 core) | host cores |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    osum = {r["cfg"]: r for r in par if "oracle_step_seconds" in r}
    for r in cfgs:
        cfg = int(r["cfg"]) if str(r["cfg"]).isdigit() else r["cfg"]
        prec = r["precision"]
        errs = [p for p in par if p.get("cfg") == cfg and p.get("precision") == prec and "rel_err" in p]
        last = max((p["step"] for p in errs), default=None)
        err = max((p["rel_err"] for p in errs if p["step"] == last), default=None)
        o = osum.get(cfg)
        oms = 1e3 * o["oracle_step_seconds"] / o["steps"] if o else None
        gbs, frac = "—", "—"
        if cfg == 5 and prec in traffic:
            b, t = traffic[prec]
            gbs = f"{b / t / 1e9:.0f}"
            frac = f"{100 * b / t / 1e9 / peak:.0f} %"
        print(f"| {cfg} | fp{prec} | 1 | {r['elem_steps_per_s'] / 1e9:.1f} G | {r['ms_per_step']:.4f} | "
              f"{'resident' if r.get('resident') else 'streaming'} | {gbs} | {frac} | "
              f"{'—' if err is None else f'{err:.1e} (step {last})'} | {'—' if oms is None else f'{oms:.1f}'} | "
              f"16 (1 used) |")


if __name__ == "__main__":
    main()
