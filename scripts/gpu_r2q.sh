# L2 evict_last policies (FED_L2_KEEP bits: 1 headers, 2 shared T, 4 shared F) as
# separate builds under _ab/K*, vs the tree (0); read/write/copy HBM probes.
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/read_peak.py > gpurun_out/q/read_peak.json 2>&1; cat gpurun_out/q/read_peak.json
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
