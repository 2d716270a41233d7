# Round 2: folded step -- GPU tests, bench A/B (folded vs node-kernel step), slab
# projection, ncu launch list + full capture of the element kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_b.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -5 gpurun_out/pytest_gpu_b.log
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
for f in 0 -1 0 -1; do
  timeout 600 python bench.py $ARGS --fold $f > gpurun_out/bench_fold$f.json 2> gpurun_out/bench_fold$f.err
  python -c "import json;d=json.load(open('gpurun_out/bench_fold$f.json'));r=d['roofline'];print('fold',$f,'ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3))"
done
timeout 900 python scripts/slab_projection.py --out gpurun_out/proj_fold0.jsonl > gpurun_out/proj_fold0.log 2>&1; echo proj0=$?
timeout 900 python scripts/slab_projection.py --fold -1 --out gpurun_out/proj_fold1.jsonl > gpurun_out/proj_fold1.log 2>&1; echo proj1=$?
python - <<'EOF'
import json
for f in ("proj_fold0", "proj_fold1"):
    try:
        for l in open(f"gpurun_out/{f}.jsonl"):
            d = json.loads(l)
            print(f, d["P"], "group", round(d["group_ms_per_step_1gpu"], 4), "events", round(d["projected_ms_per_step"], 4),
                  "eff", round(d["projected_efficiency_vs_P1"], 3), "alone", round(d["projected_alone_ms_per_step"], 4),
                  "eff_alone", round(d["projected_alone_efficiency_vs_P1"], 3))
    except Exception as e:
        print(f, "missing", e)
EOF
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_b.csv python bench.py $ARGS2 > gpurun_out/ncu_launch_b.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 5 -c 1 -o gpurun_out/prof_fold -f python bench.py $ARGS2 > gpurun_out/ncu_full_b.log 2>&1; echo ncufull=$?
python scripts/ncu_summary.py gpurun_out/prof_fold.ncu-rep --out gpurun_out/ncu_fold.json --traffic gpurun_out/traffic_fold.json > /dev/null 2>&1; cat gpurun_out/traffic_fold.json
timeout 900 python scripts/next_rows_perf.py --steps 100 > gpurun_out/next_rows_b.jsonl 2> gpurun_out/next_rows_b.err; echo next=$?; cat gpurun_out/next_rows_b.jsonl
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 25 -c 1 -o gpurun_out/prof_tables -f python scripts/next_rows_perf.py --only tables --steps 5 > gpurun_out/ncu_tables.log 2>&1; echo ncutab=$?
python scripts/ncu_summary.py gpurun_out/prof_tables.ncu-rep --out gpurun_out/ncu_tables.json > /dev/null 2>&1
