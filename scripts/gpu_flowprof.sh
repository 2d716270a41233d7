mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 10 --warmup 3 --n 192 --mode flow"
python bench.py $ARGS > gpurun_out/fp_pre.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:flow_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_flow -f python bench.py $ARGS > gpurun_out/ncu_flow.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_flow.log
