mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "concentrated or steady or table or tet" > gpurun_out/pytest12.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest12.log
