mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
python bench.py $ARGS > gpurun_out/ncu_pre.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/prof_r1c -f python bench.py $ARGS > gpurun_out/ncu_elem.log 2>&1; echo ncuelem=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1c.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncul=$?
