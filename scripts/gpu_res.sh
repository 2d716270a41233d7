mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/pytest_res.log 2>&1; echo res=$?; tail -30 gpurun_out/pytest_res.log
