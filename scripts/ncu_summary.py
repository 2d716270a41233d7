"""Summarise an `ncu --set full` capture of the element and node kernels into the
JSON kept under profiles/ (and the per-launch DRAM traffic file bench.py reads
for `roofline.traffic`).

  python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep \
      --out profiles/r1_ncu_full_cfg5_fp32.json \
      --traffic profiles/traffic_cfg5_fp32.json --source "..."
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_red.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "gpc__cycles_elapsed.avg.per_second",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--source", default="")
    ap.add_argument("--source-hash", default="", help="libfed source hash of the captured build "
                    "(default: the tree's current one)")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    kcol = head.index("Kernel Name")
    kernels = {}
    for r in data:                      # last launch of each kernel wins
        kernels[r[kcol]] = {m: [r[head.index(m)], units[head.index(m)]] for m in METRICS if m in head}
    json.dump({"source": a.source, "kernels": kernels}, open(a.out, "w"), indent=1)
    if a.traffic:
        name = next(k for k in kernels if "element_chunk" in k)
        k = kernels[name]
        b = sum(float(k[m][0].replace(",", "")) * SCALE[k[m][1]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        import os
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_1909_03355_b200.build import source_hash
        json.dump({"kernel": name, "dram_bytes_per_launch": b, "source": f"ncu --set full ({a.out})",
                   "source_hash": a.source_hash or source_hash()},
                  open(a.traffic, "w"), indent=1)
    for n, k in kernels.items():
        print(n, k["gpu__time_duration.sum"], k["launch__registers_per_thread"])


if __name__ == "__main__":
    main()
