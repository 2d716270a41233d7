# Re-entry (session 3) baseline of HEAD: build, GPU test suite, smoke, default bench.
mkdir -p gpurun_out/w
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w/build.log 2>&1; echo build=$?
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/w/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/w/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/w/bench_fp32.json 2> gpurun_out/w/bench_fp32.err; echo bench=$?; cat gpurun_out/w/bench_fp32.json | cut -c1-400
