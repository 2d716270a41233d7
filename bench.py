#!/usr/bin/env python
"""Benchmark of the FED-FEM per-time-step hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fed|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload: BASELINE.json config 5 ("Multi-GPU strong scaling": 384^3 hex8 block,
56.6M elements, k(T), c(T), convection on 5 faces, Gaussian source, fp32) --
the configuration the headline metric (element-steps/s at 1/2/4/8 B200) is
quoted on; it fits one GPU.  A "step" is one explicit time step of the whole
hot path (element loads + face loads + nodal update [+ interface exchange]).
Inputs are synthetic (seeded generators in fed_inputs), resident in HBM; the
per-step traffic (~4 GB) is far larger than the 126 MB L2, so no flush is
needed between steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "element-steps/s"
UNIT = "element-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fed", choices=["fed", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", "--grid", dest="n", type=int, default=None,
                    help="override grid size (not the headline workload)")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--scatter", default="auto",
                    choices=["auto", "atomic", "chunk", "cas", "reg", "regc", "atomic_warp", "color", "gather"])
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="interface exchange for N > 1: fused peer-memory loads (default) or NCCL send/recv")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--chunk-order", type=int, default=0, choices=[0, 1],
                    help="fed_options.chunk_order: 0 layer-major launch order (default), 1 Morton (baseline)")
    ap.add_argument("--one-transport", action="store_true",
                    help="N > 1: time only --transport (default: both transports in the same line)")
    ap.add_argument("--dry-run", action="store_true",
                    help="host control flow only (gloo, planning contexts, no device work): for CPU tests")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampler running during the timed region (recipe's clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index, enabled=True):
        self.dev = device_index
        self.proc = None
        self.enabled = enabled
        self.path = None

    def start(self):
        if not self.enabled:
            return
        fd, self.path = tempfile.mkstemp(prefix="clk", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # the sampler's start-up (NVML initialisation) happens before the timed region:
        # wait for its first sample, then the timed steps run while it keeps sampling
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count()


# ------------------------------------------------------------------ oracle (CPU) timing
def oracle_sample_rate(steps, warmup=2, n=128):
    """Time the fp64 oracle, as it stands, on a bounded sample of the same
    workload: BASELINE cfg5's problem on an n^3 grid (same physics, BCs,
    source; fewer elements), `steps` explicit steps on one host thread."""
    import oracle
    from fed_inputs import make_config
    p = make_config(5, n=n)
    o = oracle.Oracle(p, 2.0075e-3)
    o.step(warmup)
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    return p.n_elems * steps / dt, p.n_elems, dt


def run_reference(args, rank):
    if rank != 0:
        return
    model, ncpu = host_info()
    K, W = args.steps, args.warmup
    # size the sample so that K + W steps take ~30 s at ~12M element-steps/s
    n = int(max(16, min(128, round((3.6e8 / max(1, K + W)) ** (1 / 3)))))
    rate, E, secs = oracle_sample_rate(K, W, n)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * secs / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg5 sample {n}^3 ({E} hex8 elements), oracle fp64 single thread",
                   "steps": K},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"cfg5 physics on {n}^3 grid ({E} elements), {K} steps after {W} warm-up, "
                                   f"host {model} ({ncpu} logical cores, 1 used)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def chunk_table_bytes(g, info):
    """Per-step bytes of the chunk tables the element kernel reads (chunk modes): the
    64-byte header of every chunk and its shared-node list (int32 per entry, bank-layout
    holes included, padded to 16 B) -- the part of the stored connectivity that names
    the chunk's shared nodes (chunk-local positions alone do not)."""
    import ctypes as C
    import numpy as np
    from paper_1909_03355_b200 import fed
    if info["scatter"] not in (2, 3, 4, 5) or info["n_chunks"] == 0:
        return 0
    lib = fed.load()
    nc = C.c_int64(0)
    if lib.fed_debug_chunks(g._h, C.byref(nc), None, None, None) != 0:
        return 0
    hdr = np.empty((nc.value, 8), np.int32)
    if lib.fed_debug_chunks(g._h, C.byref(nc), hdr.ctypes.data, None, None) != 0:
        return 0
    n_sp = hdr[:, 6].astype(np.int64)
    return int(64 * nc.value + 4 * ((n_sp + 3) & ~3).sum())


def layout_bytes(info, precision, q, tables=0):
    """Compulsory DRAM bytes of one element-kernel launch and of the node kernel
    in the library's data layout (DESIGN.md sec. 5 "Measurement"): per element the
    connectivity as stored (chunk-local uint16: 2 B per corner; atomic-family
    baselines: int32, 4 B per corner) and the 6-word operator; per node T read,
    T write, coef (+ Q with a source).  SURVEY 8d's figure counts int32
    connectivity (32 B per hex) for every layout; it is reported next to it."""
    w = precision // 8
    npe = info["nodes_per_elem"]
    E_loc, N_int, N_sp = info["n_elems_local"], info["n_interior"], info["n_special"]
    chunk_mode = info["scatter"] in (2, 3, 4, 5)
    # fp32 streaming colour-phase hex kernel (REGC): 12-bit packed positions, 12 B per element
    conn = (12 if info["scatter"] == 5 and npe == 8 and precision == 32 else (2 if chunk_mode else 4) * npe)
    if chunk_mode:   # chunk-interior nodes are updated by the element kernel, shared nodes by the node kernel
        elem = E_loc * (conn + 6 * w) + N_int * (3 + q) * w + N_sp * w + tables
        node = N_sp * (2 + q) * w
        elem_survey = elem - tables + E_loc * (4 * npe - conn)   # SURVEY: int32 global ids, no lists
    else:
        elem = E_loc * (conn + 6 * w)
        node = (N_int + N_sp) * (3 + q) * w
        elem_survey = elem
    step_survey = E_loc * (4 * npe + 6 * w) + (N_int + N_sp) * (3 + q) * w
    return elem, node, elem_survey, step_survey, chunk_mode


def traffic_record(config, precision, n):
    """Measured DRAM bytes per element-kernel launch (ncu, profiles/traffic_*.json),
    used only if it was captured from the current kernel sources."""
    from paper_1909_03355_b200.build import source_hash
    tpath = os.path.join(ROOT, "profiles", f"traffic_cfg{config}_fp{precision}.json")
    if n is not None or not os.path.exists(tpath):
        return None, "no capture for this workload"
    try:
        t = json.load(open(tpath))
    except Exception:
        return None, "unreadable traffic file"
    if t.get("source_hash") != source_hash():
        return None, f"stale: {os.path.basename(tpath)} was captured from other kernel sources"
    return t.get("dram_bytes_per_launch"), f"ncu --set full of these sources ({os.path.basename(tpath)})"


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from fed_inputs import make_config
    from paper_1909_03355_b200 import fed
    from paper_1909_03355_b200.build import build

    dry = args.dry_run      # host control flow only (CPU test): plans, no device work
    if rank == 0:
        build()
    if not dry:
        torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            obj = [fed.fed_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        dist.barrier()
    prob = make_config(args.config, n=args.n)
    E, N = prob.n_elems, prob.n_nodes
    scatter = {"auto": 0, "atomic": 1, "chunk": 2, "cas": 3, "reg": 4, "regc": 5, "atomic_warp": 6, "color": 7,
               "gather": 8}[args.scatter]
    K, W = args.steps, max(3, args.warmup)
    tr_code = {"peer": fed.FED_TRANSPORT_PEER, "nccl": fed.FED_TRANSPORT_NCCL}

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if dry else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = None if dry else torch.cuda.Stream()

    def create(transport):
        if os.environ.get("FED_BENCH_FAIL_TRANSPORT") == transport and rank == world - 1:
            raise RuntimeError("injected failure (FED_BENCH_FAIL_TRANSPORT, control-flow test)")
        return fed.Fed.from_problem(prob, precision=args.precision, device=-1 if dry else local,
                                    stream=None if dry else stream.cuda_stream, rank=rank, nranks=world,
                                    nccl_id=nccl_id, scatter=scatter, chunk_elems=args.chunk,
                                    transport=tr_code[transport], chunk_order=args.chunk_order)

    def timed_steps(g, k):
        """k steps between CUDA events on the library's stream, max over ranks (ms)."""
        barrier()
        if dry:
            return max_over_ranks(0.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.step(k)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    def all_ok(ok):
        """Every rank's verdict on a fallible phase (create + warm-up): either all ranks
        go on with this transport or all abandon it (the library's create already agrees
        across ranks; a step error -- e.g. a bounded PEER flag wait -- is raised on each)."""
        if world == 1:
            return ok
        t = torch.tensor([0.0 if ok else 1.0], dtype=torch.float64, device="cpu" if dry else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) == 0.0

    def create_and_warm(transport):
        """(context, create seconds, error string or None)."""
        t0 = time.perf_counter()
        g, err = None, None
        try:
            g = create(transport)
            if not dry:
                g.step(W)                  # warm-up (also builds the CUDA graph)
                torch.cuda.synchronize()
        except Exception as e:            # noqa: BLE001 -- reported in the JSON line
            err = f"{type(e).__name__}: {e}"
        if not all_ok(err is None):
            if g is not None:
                try:
                    g.close()
                except Exception:
                    pass
            return None, 0.0, err or "failed on another rank"
        return g, time.perf_counter() - t0, None

    # ---- primary transport: the full measurement.  At N > 1 a transport that fails on
    # real hardware (this path first runs multi-GPU at the driver) is reported and the
    # other one takes its place, so the line still measures the partitioned step.
    transport_errors = {}
    g, t_create, err = create_and_warm(args.transport)
    if g is None:
        if world == 1:
            raise RuntimeError(err)
        transport_errors[args.transport] = err
        args.transport = "nccl" if args.transport == "peer" else "peer"
        g, t_create, err = create_and_warm(args.transport)
        if g is None:
            raise RuntimeError(f"both transports failed: {transport_errors} / {args.transport}: {err}")
    info = g.info()
    clk = Clocks(local, enabled=not (args.no_clocks or dry))
    launches0 = info["kernel_launches_total"]
    clk.start()
    ms = timed_steps(g, K)
    clocks = clk.stop()
    launches = g.info()["kernel_launches_total"] - launches0
    value = E * K / (ms / 1e3) if ms > 0 else None

    # ---- per-kernel timing pass (CUDA events around each launch, same stream)
    q = 1 if prob.q_vol is not None else 0
    tables = 0 if dry else chunk_table_bytes(g, info)
    elem_bytes, node_bytes, elem_bytes_survey, step_bytes_survey, chunk_mode = layout_bytes(info, args.precision, q,
                                                                                            tables)
    roof = None
    if not dry:
        g.set_timing(True)
        barrier()
        g.step(K)
        tim = g.timing()
        g.set_timing(False)
        elem_ms = tim["element_ms"] / max(1, tim["element_launches"])
        elem_launches_per_step = tim["element_launches"] / K
        node_ms = tim["node_ms"] / max(1, tim["node_launches"])
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
        per_launch = elem_bytes / elem_launches_per_step
        achieved = per_launch / (elem_ms / 1e3) / 1e9
        traffic, traffic_src = traffic_record(args.config, args.precision, args.n) if world == 1 else \
            (None, "single-GPU capture only")
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "traffic_over_alg": (traffic / per_launch) if traffic else None,
                "kernel": "element_chunk_kernel" if chunk_mode else "element_atomic_kernel",
                "peak_source": peak_src, "alg_bytes_per_launch": per_launch,
                "alg_bytes_note": "compulsory bytes of the stored layout: per element 12 B of 12-bit packed "
                                  "chunk-local connectivity + 6 operator words; per chunk its 64-B header and "
                                  "shared-node list; per node T read/write, coef, Q (DESIGN.md)",
                "chunk_table_bytes": tables,
                "avg_launch_ms": elem_ms, "node_kernel_ms": node_ms, "node_alg_bytes": node_bytes,
                "node_frac": (node_bytes / (node_ms / 1e3) / 1e9 / peak) if node_ms > 0 else None,
                "elem_share_of_step": (tim["element_ms"] / K) / (ms / K),
                "frac_survey_bytes": (elem_bytes_survey / elem_launches_per_step) / (elem_ms / 1e3) / 1e9 / peak,
                "step_frac_survey_bytes": step_bytes_survey / (ms / K / 1e3) / 1e9 / peak}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and not dry:
        T0 = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
        T0[:] = prob.T0
        out = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.set_temperature(T0)
        g.step(K)
        g.temperature(out)
        torch.cuda.synchronize()
        secs = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": E * K / secs, "unit": UNIT, "h2d_bytes_per_step": 8 * N / K,
               "d2h_bytes_per_step": 8 * N / K,
               "note": "per run: fed_set_temperature(T0 host) + fed_step(K) + fed_get_temperature(host), wall clock"}
    info_end = g.info()
    g.close()
    plans = [None] * world
    if world > 1:
        dist.all_gather_object(plans, {k: info[k] for k in ("n_elems_local", "n_interface", "n_chunks")})
    else:
        plans[0] = {k: info[k] for k in ("n_elems_local", "n_interface", "n_chunks")}

    # ---- N > 1: the other interface transport on the same workload (same line)
    transports = {args.transport: {"ms_per_step": ms / K, "value": value}}
    if world > 1 and not args.one_transport:
        other = "nccl" if args.transport == "peer" else "peer"
        if other not in transport_errors:
            g2, _, err2 = create_and_warm(other)
            if g2 is None:
                transport_errors[other] = err2
            else:
                ms2 = timed_steps(g2, K)
                g2.close()
                transports[other] = {"ms_per_step": ms2 / K, "value": E * K / (ms2 / 1e3) if ms2 > 0 else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not dry:
        model, ncpu = host_info()
        rate, Es, secs = oracle_sample_rate(60, 2, 128)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"cfg5 physics on 128^3 ({Es} elements), 60 steps, fp64, {secs:.1f} s on host "
                         f"{model} ({ncpu} logical cores, 1 used)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"cfg{args.config}" + ("" if args.n is None else f" n={args.n}"),
                       "grid": f"{prob.grid[0]}^3 hex8", "elements": E, "nodes": N,
                       "parallelism": f"z-slab x{world}", "scatter": args.scatter,
                       "exchange": args.transport if world > 1 else "none",
                       "mode": "resident" if info["resident"] else "stream",
                       "chunk_elems": info["chunk_elems"], "dt": info["dt"],
                       "l2": "inputs larger than L2 (per-step traffic >> 126 MB), no flush",
                       "create_s": round(t_create, 2)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "impl": "fed",
            "fail_step": info_end["fail_step"],
        }
        if world > 1:
            line["transports"] = transports
            if transport_errors:
                line["transport_errors"] = transport_errors
            line["ranks"] = plans
        if dry:
            line["dry_run"] = True
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
