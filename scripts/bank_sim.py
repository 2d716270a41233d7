"""Offline simulation of the element kernel's shared-memory bank conflicts
for a plan (dry run, no GPU): for every warp instruction that reads sT / sF
through the chunk-local connectivity, the conflict degree is the max number
of distinct 4-byte words (fp32) hitting one of the 32 banks."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def simulate(hdr, col, c16, colored=True, threads=128, max_chunks=400, word=1):
    tot_wf = 0
    tot_ideal = 0
    for c in range(min(max_chunks, hdr.shape[0])):
        off, ne = hdr[c, 0], hdr[c, 1]
        groups = []
        if colored:
            for k in range(32):
                a, b = col[c, k], col[c, k + 1]
                if b > a:
                    for base in range(a, b, threads):
                        groups.append(np.arange(base, min(b, base + threads)))
        else:
            for base in range(0, ne, threads):
                groups.append(np.arange(base, min(ne, base + threads)))
        for g in groups:
            for w0 in range(0, g.size, 32):
                lanes = g[w0:w0 + 32]
                idx = c16[off + lanes].astype(np.int64)     # (lanes, 8)
                for q in range(8):
                    a = idx[:, q] * word
                    wf = 0
                    for half in range(word):
                        banks = (a + half) % 32
                        # distinct words per bank
                        m = 0
                        for bk in np.unique(banks):
                            m = max(m, np.unique(a[banks == bk]).size)
                        wf += m
                    tot_wf += wf
                    tot_ideal += word
    return tot_wf / max(tot_ideal, 1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=96)
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--scatter", type=int, default=2)
    a = ap.parse_args()
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    p = make_config(a.config, n=a.n)
    g = fed.Fed.from_problem(p, device=-1, chunk_elems=a.chunk, scatter=a.scatter, precision=32)
    hdr, col, c16 = g.debug_chunks()
    print("colored conflict factor", round(simulate(hdr, col, c16, True), 3))
    print("uncolored conflict factor", round(simulate(hdr, col, c16, False), 3))
