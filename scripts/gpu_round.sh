mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpuinfo.txt
lscpu | head -20 > gpurun_out/hostinfo.txt
timeout 600 python bench.py > gpurun_out/bench_r1.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_r1.log
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"element_chunk|node_kernel" -s 4 -c 2 -o gpurun_out/prof_r1 $B > gpurun_out/ncu_full_r1.log 2>&1; echo ncu2=$?
