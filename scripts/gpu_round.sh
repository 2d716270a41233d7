mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest5.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest5.log
timeout 900 python scripts/sweep.py --steps 50 --variants chunk:1024,cas:1024,reg:1024,reg:512,reg:256,cas:512,cas:256,reg64:512,cas64:512,chunk64:1024 > gpurun_out/sweep2.log 2>&1; cat gpurun_out/sweep2.log | grep variant
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --scatter reg --chunk 512"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"element_chunk|node_kernel" -s 4 -c 2 -o gpurun_out/prof3 $B > gpurun_out/ncu_full3.log 2>&1; echo ncu=$?
