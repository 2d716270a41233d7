# PDL A/B with the restored node kernel; tables; full GPU tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
for i in 1 2; do for p in 1 0; do
  FED_PDL=$p timeout 600 python bench.py $ARGS > gpurun_out/bench_h_pdl$p.$i.json 2> gpurun_out/bench_h_pdl$p.$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_h_pdl$p.$i.json'));r=d['roofline'];print('pdl',$p,'ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3),'nfrac',round(r['node_frac'],3))"
done; done
for p in 1 0; do
  FED_PDL=$p timeout 1200 python scripts/slab_projection.py --out gpurun_out/proj_h_pdl$p.jsonl > gpurun_out/proj_h_pdl$p.log 2>&1; echo proj$p=$?
done
python - <<'PY'
import json
for f in ("proj_h_pdl1", "proj_h_pdl0"):
    try:
        for l in open(f"gpurun_out/{f}.jsonl"):
            d = json.loads(l)
            print(f, d["P"], "group", round(d["group_ms_per_step_1gpu"], 4), "events", round(d["projected_ms_per_step"], 4),
                  "alone", [round(x, 4) for x in d["alone_ms_per_step"]], "eff_alone", round(d["projected_alone_efficiency_vs_P1"], 3))
    except Exception as e:
        print(f, "missing", e)
PY
for p in 1 0; do FED_PDL=$p timeout 900 python scripts/next_rows_perf.py --steps 100 --only tables > gpurun_out/next_rows_h$p.jsonl 2> gpurun_out/next_rows_h$p.err; echo next$p=$?; cat gpurun_out/next_rows_h$p.jsonl; done
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_h.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -4 gpurun_out/pytest_gpu_h.log
