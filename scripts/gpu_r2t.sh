# Clean bench lines (no concurrent host load) with the committed traffic files of these
# sources, and the slab projection on a quiet box.
mkdir -p gpurun_out/t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t/build.log 2>&1
for i in 1 2 3; do timeout 900 python bench.py > gpurun_out/t/bench_fp32_$i.json 2> gpurun_out/t/bench_fp32_$i.err; echo bench=$?; done
timeout 900 python bench.py --precision 64 --no-cpu-baseline > gpurun_out/t/bench_fp64.json 2> gpurun_out/t/bench_fp64.err; echo bench64=$?
timeout 1500 python scripts/slab_projection.py --out gpurun_out/t/r2_slab_projection_cfg5_fp32.jsonl > gpurun_out/t/proj.log 2>&1; echo proj=$?
