mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest11.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest11.log
timeout 900 python scripts/sweep.py --steps 50 --variants regc:1024,regc64:1024 > gpurun_out/sweep8.log 2>&1; grep variant gpurun_out/sweep8.log | cut -c1-200
