# L2 evict_last, third pass: element-kernel-only hints (FED_L2_KEEP 1 headers, 8 shared-T
# gather, 16 shared-F reductions), builds under _ab/K*, tree = 0.
mkdir -p gpurun_out/s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
