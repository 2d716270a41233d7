mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?; cat gpurun_out/bench2.json
timeout 1500 python scripts/slab_projection.py --out gpurun_out/slab_projection.jsonl > gpurun_out/proj.log 2>&1; echo proj=$?; cat gpurun_out/proj.log | cut -c1-600
