# Round evidence in one GPU call: tests, smoke, bench (fp32 headline + fp64),
# reference arm, ncu launch list + full captures (fp32 and fp64), per-rank slab
# projection.  Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
ARGS="--steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
python bench.py $ARGS > gpurun_out/ncu_pre.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/prof_full -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
python bench.py $ARGS --precision 64 > gpurun_out/ncu_pre64.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o gpurun_out/prof_full64 -f python bench.py $ARGS --precision 64 > gpurun_out/ncu_full64.log 2>&1; echo ncufull64=$?
timeout 900 python bench.py > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo bench=$?
timeout 900 python bench.py --precision 64 --no-cpu-baseline > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo bench64=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 1500 python scripts/slab_projection.py --out gpurun_out/slab_projection.jsonl > gpurun_out/proj.log 2>&1; echo proj=$?
timeout 1500 python scripts/all_configs.py --max-steps 1000 > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err; echo cfgs=$?
