# Round 2, after removing the folded step: GPU tests (incl. the checked build),
# smoke, bench, per-rank slab projection (alone method), ncu traffic capture of the
# element kernel (profiles/traffic file for bench.py), tables kernel profile.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_c.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -4 gpurun_out/pytest_gpu_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo smoke=$?
for i in 1 2; do
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$i.json 2> gpurun_out/bench_c$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_c$i.json'));r=d['roofline'];print('bench ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3),'node_frac',round(r['node_frac'],3))"
done
timeout 1200 python scripts/slab_projection.py --out gpurun_out/proj_c.jsonl > gpurun_out/proj_c.log 2>&1; echo proj=$?
timeout 1200 python scripts/slab_projection.py --transport nccl --ranks 2 4 8 --out gpurun_out/proj_c_nccl.jsonl > gpurun_out/proj_c_nccl.log 2>&1; echo projn=$?
python - <<'EOF'
import json
for f in ("proj_c", "proj_c_nccl"):
    try:
        for l in open(f"gpurun_out/{f}.jsonl"):
            d = json.loads(l)
            print(f, d["P"], "group", round(d["group_ms_per_step_1gpu"], 4), "events", round(d["projected_ms_per_step"], 4),
                  "alone", [round(x, 4) for x in d["alone_ms_per_step"]],
                  "eff_alone", round(d["projected_alone_efficiency_vs_P1"], 3))
    except Exception as e:
        print(f, "missing", e)
EOF
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c.csv python bench.py $ARGS2 > gpurun_out/ncu_launch_c.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/prof_c -f python bench.py $ARGS2 > gpurun_out/ncu_full_c.log 2>&1; echo ncufull=$?
python scripts/ncu_summary.py gpurun_out/prof_c.ncu-rep --out gpurun_out/ncu_c.json --traffic gpurun_out/traffic_cfg5_fp32.json; cat gpurun_out/traffic_cfg5_fp32.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 2 -c 1 -o gpurun_out/prof_tables -f python scripts/next_rows_perf.py --only tables --steps 5 > gpurun_out/ncu_tables.log 2>&1; echo ncutab=$?
python scripts/ncu_summary.py gpurun_out/prof_tables.ncu-rep --out gpurun_out/ncu_tables.json
timeout 900 python scripts/next_rows_perf.py --steps 100 > gpurun_out/next_rows_c.jsonl 2> gpurun_out/next_rows_c.err; echo next=$?; cat gpurun_out/next_rows_c.jsonl
