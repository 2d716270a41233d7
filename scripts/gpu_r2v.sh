# General tables: phi pass with four searches in flight (tree) vs HEAD (_ab/A); the new
# packed-record GPU tests; ncu traffic of the (unchanged) default kernels for this source hash.
mkdir -p gpurun_out/v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v/build.log 2>&1
for i in 1 2; do
  for v in tree A; do D=.; [ $v = A ] && D=_ab/A
    (cd $D && timeout 600 python scripts/next_rows_perf.py --only tables4 --steps 200 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$i', 'tables4', round(d['ms_per_step'],4))")
    (cd $D && timeout 600 python scripts/next_rows_perf.py --only base --steps 200 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$i', 'base', round(d['ms_per_step'],4))")
  done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed_record or table or clamped" > gpurun_out/v/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/v/pytest.log
ARGS="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/v/prof_fp32 -f python bench.py $ARGS > gpurun_out/v/ncu_full.log 2>&1; echo ncufull=$?
python scripts/ncu_summary.py gpurun_out/v/prof_fp32.ncu-rep --out gpurun_out/v/r2_ncu_full_cfg5_fp32.json --traffic gpurun_out/v/traffic_cfg5_fp32.json
timeout 900 ncu --set full --clock-control none --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/v/prof_fp64 -f python bench.py $ARGS --precision 64 > gpurun_out/v/ncu_full64.log 2>&1; echo ncufull64=$?
python scripts/ncu_summary.py gpurun_out/v/prof_fp64.ncu-rep --out gpurun_out/v/r2_ncu_full_cfg5_fp64.json --traffic gpurun_out/v/traffic_cfg5_fp64.json
