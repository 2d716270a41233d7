"""Per-source-line warp-stall samples and executed instructions of one kernel in an
ncu report (cuda,sass source view), top N lines.

    python scripts/ncu_lines.py REPORT [--top 25]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--kernel", default=None, help="substring of the kernel name (default: first)")
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if a.kernel:
        cmd += ["--kernel-name", "regex:" + a.kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_samp, i_inst = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lines, cur = {}, None
    for r in rows:
        if len(r) < 4 or r[0] == "Line No":
            continue
        if r[0] and r[2] == "-":          # a CUDA source line; its SASS rows follow
            cur = (int(r[0]), r[1].strip())
            lines.setdefault(cur, [0.0, 0.0])
        elif r[2].startswith("0x") and cur is not None and len(r) >= len(hdr):
            try:
                lines[cur][0] += float(r[i_samp])
                lines[cur][1] += float(r[i_inst])
            except ValueError:
                pass
    ts = sum(v[0] for v in lines.values()) or 1
    ti = sum(v[1] for v in lines.values()) or 1
    print(f"samples {ts:.0f}, warp instructions {ti:.0f}")
    for (ln, src), (s, i) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{100 * s / ts:5.1f}% stalls {100 * i / ti:5.1f}% inst  L{ln}: {src[:100]}")


if __name__ == "__main__":
    main()
