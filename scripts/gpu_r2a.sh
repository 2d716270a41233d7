# Round 2, first GPU call: full-size full-length parity (oracles on the host
# cores in the background), the GPU test suite, smoke, bench, compute-sanitizer
# over every execution mode.  Outputs under gpurun_out/.
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | grep -i "model name"; } > gpurun_out/gpuinfo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
( timeout 5000 python tests/full_parity_run.py --configs 1 2 3 4 5 --workdir /tmp/fed_fp \
    --out gpurun_out/r2_full_parity.jsonl > gpurun_out/full_parity.log 2>&1; echo "rc=$?" >> gpurun_out/full_parity.log ) &
FP=$!
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo bench=$?
for tool in memcheck racecheck synccheck initcheck; do
  for c in stream stream64 resident peer nccl tables tet atomic; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py --case $c --steps 3 \
      > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "san $tool $c rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_${tool}_${c}.log | tail -1)"
  done
done
wait $FP
tail -40 gpurun_out/full_parity.log
