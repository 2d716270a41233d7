# Round-2 re-entry: A/B of chunk order x L2 policy (gpu_r2k.sh), then the GPU test suite on HEAD.
bash scripts/gpu_r2k.sh
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/pytest_gpu.log
