mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench=$?; cat gpurun_out/bench3.json
timeout 600 python bench.py --no-cpu-baseline --no-e2e --precision 64 > gpurun_out/bench3_fp64.json 2> gpurun_out/bench3_fp64.err; echo bench64=$?; cat gpurun_out/bench3_fp64.json
