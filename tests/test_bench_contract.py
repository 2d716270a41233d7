"""CPU test of bench.py's reference arm: one JSON line with the contract's keys
(the GPU arm is exercised by the driver on a B200)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(oracle_lib):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "element-steps/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multi_rank_control_flow_dry_run():
    """bench.py's N > 1 control flow under torchrun (2 ranks, gloo, planning-only
    contexts): env parsing, process group, the per-rank slab plans, barriers and
    max-over-ranks, both transports, and exactly ONE JSON line from rank 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--grid", "24", "--dry-run"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["config"]["parallelism"] == "z-slab x2"
    assert set(d["transports"]) == {"peer", "nccl"}
    ranks = d["ranks"]
    assert len(ranks) == 2 and sum(r["n_elems_local"] for r in ranks) == d["config"]["elements"] == 24 ** 3
    # both ranks hold the shared interface plane: (n + 1)^2 nodes each
    assert ranks[0]["n_interface"] == ranks[1]["n_interface"] == 25 ** 2


def test_multi_rank_transport_fallback_dry_run():
    """A transport that fails on one rank only (injected on the last rank) is abandoned
    by every rank: the line is measured with the other transport and names the error."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--grid", "16", "--dry-run"]
    env = dict(os.environ, FED_BENCH_FAIL_TRANSPORT="peer")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["config"]["exchange"] == "nccl" and set(d["transports"]) == {"nccl"}
    assert "injected" in d["transport_errors"]["peer"] or "another rank" in d["transport_errors"]["peer"]


def test_layout_bytes_accounting():
    """bench.py's compulsory-bytes figure for the roofline (DESIGN.md sec. 5
    "Measurement"), on a planning-only context: fp32 streaming hex = 12 B packed
    positions + 6 operator words per element, the chunk tables (64-B header + the
    shared-node list padded to 16 B) per chunk, T r/w + coef + Q per interior node and
    the T read per shared node; fp64 keeps the 16 B of uint16 byte offsets."""
    sys.path.insert(0, ROOT)
    import bench
    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=24)
    for prec, conn in ((32, 12), (64, 16)):
        g = fed.Fed.from_problem(p, precision=prec, device=-1, resident=-1, chunk_elems=256)
        info = g.info()
        assert info["scatter"] == fed.FED_SCATTER_CHUNK_REGC
        hdr, _, _ = g.debug_chunks()
        tables = bench.chunk_table_bytes(g, info)
        assert tables == 64 * len(hdr) + 4 * int(((hdr[:, 6].astype(np.int64) + 3) // 4 * 4).sum())
        w = prec // 8
        elem, node, elem_survey, _, chunk_mode = bench.layout_bytes(info, prec, 1, tables)
        assert chunk_mode
        assert elem == (info["n_elems_local"] * (conn + 6 * w) + info["n_interior"] * 4 * w
                        + info["n_special"] * w + tables)
        assert node == info["n_special"] * 3 * w
        assert elem_survey == elem - tables + info["n_elems_local"] * (32 - conn)
        g.close()
