# PDL A/B: bench (cfg5 fp32, fp64), slab projection (alone method), GPU tests with PDL on.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
for i in 1 2; do for p in 1 0; do
  FED_PDL=$p timeout 600 python bench.py $ARGS > gpurun_out/bench_pdl$p.$i.json 2> gpurun_out/bench_pdl$p.$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_pdl$p.$i.json'));r=d['roofline'];print('pdl',$p,'ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3))"
done; done
for p in 1 0; do
  FED_PDL=$p timeout 600 python bench.py $ARGS --precision 64 > gpurun_out/bench64_pdl$p.json 2> gpurun_out/bench64_pdl$p.err
  python -c "import json;d=json.load(open('gpurun_out/bench64_pdl$p.json'));r=d['roofline'];print('fp64 pdl',$p,'ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3))"
done
for p in 1 0; do
  FED_PDL=$p timeout 1200 python scripts/slab_projection.py --out gpurun_out/proj_pdl$p.jsonl > gpurun_out/proj_pdl$p.log 2>&1; echo proj$p=$?
done
python - <<'PY'
import json
for f in ("proj_pdl1", "proj_pdl0"):
    try:
        for l in open(f"gpurun_out/{f}.jsonl"):
            d = json.loads(l)
            print(f, d["P"], "group", round(d["group_ms_per_step_1gpu"], 4), "events", round(d["projected_ms_per_step"], 4),
                  "alone", round(d["projected_alone_ms_per_step"], 4), "eff_alone", round(d["projected_alone_efficiency_vs_P1"], 3))
    except Exception as e:
        print(f, "missing", e)
PY
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu_d.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -4 gpurun_out/pytest_gpu_d.log
for p in 1 0; do FED_PDL=$p timeout 900 python scripts/next_rows_perf.py --steps 100 > gpurun_out/next_rows_d$p.jsonl 2> gpurun_out/next_rows_d$p.err; echo next$p=$?; cat gpurun_out/next_rows_d$p.jsonl; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 2 -c 1 -o gpurun_out/prof_tables_d -f python scripts/next_rows_perf.py --only tables --steps 5 > gpurun_out/ncu_tables_d.log 2>&1; echo ncutab=$?
python scripts/ncu_summary.py gpurun_out/prof_tables_d.ncu-rep --out gpurun_out/ncu_tables_d.json
