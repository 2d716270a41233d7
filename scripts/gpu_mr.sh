mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_mr.log 2>&1; echo mr=$?; tail -25 gpurun_out/pytest_mr.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$?; tail -5 gpurun_out/pytest_gpu.log
