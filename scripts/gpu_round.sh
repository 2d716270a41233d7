mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest9.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest9.log
timeout 900 python scripts/sweep.py --steps 50 --variants regc:1024,regc:512,reg:1024,regc64:1024,regc64:512 > gpurun_out/sweep6.log 2>&1; cat gpurun_out/sweep6.log | grep variant
