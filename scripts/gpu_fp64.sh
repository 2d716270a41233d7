# fp64 evidence after an fp64-only kernel change: full GPU suite, smoke, fp64 bench,
# fp64 ncu --set full capture of the element + node kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --precision 64 --no-cpu-baseline > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo bench64=$?
ARGS="--steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --precision 64"
python bench.py $ARGS > gpurun_out/ncu_pre64.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/prof_full64 -f python bench.py $ARGS > gpurun_out/ncu_full64.log 2>&1; echo ncufull64=$?
