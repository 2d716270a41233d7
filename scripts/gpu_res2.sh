mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/pytest_res.log 2>&1; echo res=$?; tail -3 gpurun_out/pytest_res.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/all_configs.py --max-steps 500 > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err; echo cfgs=$?; cut -c1-200 gpurun_out/all_configs.jsonl
