# Round 2 evidence with the final kernels (session 4 re-run of the session-3 kernels for the current source hash; real-time capacity not repeated): full-size full-length parity (oracles on the
# host cores in the background), GPU tests, smoke, bench lines (fp32 headline, fp64,
# reference arm), ncu launch list + full captures (traffic file for bench.py), slab
# projection, all configs, NEXT-row costs, real-time capacity.  Outputs under gpurun_out/.
mkdir -p gpurun_out/final4
O=gpurun_out/final4
{ nvidia-smi; free -g; nproc; lscpu | grep -i "model name"; } > $O/gpuinfo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "from paper_1909_03355_b200.build import source_hash; print(source_hash())" > $O/source_hash.txt
( timeout 4200 python tests/full_parity_run.py --configs 1 2 3 4 5 --workdir /tmp/fed_fp \
    --out $O/r2_full_parity.jsonl > $O/full_parity.log 2>&1; echo "rc=$?" >> $O/full_parity.log ) &
FP=$!
sleep 240   # let the parity run's GPU part (all five configs) finish before timing anything
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
ARGS="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg5_fp32.csv python bench.py $ARGS > $O/ncu_launch.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o $O/prof_fp32 -f python bench.py $ARGS > $O/ncu_full.log 2>&1; echo ncufull=$?
python scripts/ncu_summary.py $O/prof_fp32.ncu-rep --out $O/r2_ncu_full_cfg5_fp32.json --traffic $O/traffic_cfg5_fp32.json
timeout 900 ncu --set full --clock-control none --kernel-name regex:"element_chunk|node_kernel" --launch-skip 6 -c 2 -o $O/prof_fp64 -f python bench.py $ARGS --precision 64 > $O/ncu_full64.log 2>&1; echo ncufull64=$?
python scripts/ncu_summary.py $O/prof_fp64.ncu-rep --out $O/r2_ncu_full_cfg5_fp64.json --traffic $O/traffic_cfg5_fp64.json
cp $O/traffic_cfg5_fp32.json $O/traffic_cfg5_fp64.json profiles/   # this box's bench reads them
timeout 900 python bench.py > $O/bench_fp32.json 2> $O/bench_fp32.err; echo bench=$?
timeout 900 python bench.py > $O/bench_fp32_b.json 2> $O/bench_fp32_b.err; echo bench_b=$?
timeout 900 python bench.py --precision 64 --no-cpu-baseline > $O/bench_fp64.json 2> $O/bench_fp64.err; echo bench64=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 1500 python scripts/slab_projection.py --out $O/r2_slab_projection_cfg5_fp32.jsonl > $O/proj.log 2>&1; echo proj=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/slab_launches.csv python scripts/slab_launches.py --steps 3 > $O/slab_launches.log 2>&1; echo slabl=$?
python scripts/slab_launches.py --summarize $O/slab_launches.csv --alone $O/r2_slab_projection_cfg5_fp32.jsonl > $O/r2_slab_launches.txt 2>&1
timeout 1500 python scripts/slab_projection.py --transport nccl --ranks 1 2 4 8 --out $O/r2_slab_projection_cfg5_fp32_nccl.jsonl > $O/proj_nccl.log 2>&1; echo projn=$?
timeout 1500 python scripts/all_configs.py --max-steps 1000 > $O/r2_all_configs.jsonl 2> $O/all_configs.err; echo cfgs=$?
timeout 900 python scripts/next_rows_perf.py --steps 200 > $O/r2_next_rows_perf.jsonl 2> $O/next_rows.err; echo next=$?
timeout 900 python scripts/all_configs.py --configs paper_ti,paper_td,tet160 --max-steps 500 > $O/r2_tet_perf.jsonl 2> $O/tet.err; echo tet=$?
python scripts/read_peak.py > $O/r2_read_peak.json 2>&1
wait $FP
tail -12 $O/full_parity.log
