# Operator words in 16-byte groups (tree: fp32 3 loads / fp64 4 loads per element) vs HEAD
# (_ab/A: fp32 6 loads, fp64 7): same-box A/B fp32 + fp64, ncu DRAM bytes, GPU tests.
mkdir -p gpurun_out/o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
BENCH_ARGS="--steps 100 --precision 64" bash scripts/gpu_abn.sh
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 4 -c 1 -o gpurun_out/o/prof_tree -f python bench.py $ARGS2 > gpurun_out/o/ncu_tree.log 2>&1; echo ncu $?
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/pytest_gpu.log
