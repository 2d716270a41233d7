# L2 evict_last policies, second pass (node-kernel hinted accesses as plain asm):
# FED_L2_KEEP bits 1 headers, 2 shared T, 4 shared F; builds under _ab/K*, tree = 0.
mkdir -p gpurun_out/r
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
