# TDK 3 (clamped-linear tables): GPU table tests, NEXT-row costs, bench (TDK 1 unchanged).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -k "table or clamped" > gpurun_out/pytest_j.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_j.log
timeout 900 python scripts/next_rows_perf.py --steps 100 > gpurun_out/next_rows_j.jsonl 2> gpurun_out/next_rows_j.err; echo next=$?; cat gpurun_out/next_rows_j.jsonl
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err
python -c "import json;d=json.load(open('gpurun_out/bench_j.json'));r=d['roofline'];print('ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3))"
