mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/pytest_res.log 2>&1; echo res=$?; tail -25 gpurun_out/pytest_res.log
timeout 900 python scripts/all_configs.py --configs paper_ti,paper_td,1,2 --max-steps 2000 > gpurun_out/tet_cfgs.jsonl 2> gpurun_out/tet_cfgs.err; echo cfgs=$?; cut -c1-220 gpurun_out/tet_cfgs.jsonl
