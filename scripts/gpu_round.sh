mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest10.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest10.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke2.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_r1b.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_r1b.log
