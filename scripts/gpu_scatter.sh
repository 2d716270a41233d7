# Parity of the scatter baselines + cfg5 fp32 step time of every scatter strategy.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "baseline or color_passes" > gpurun_out/pytest_sc.log 2>&1; echo sc=$?; tail -15 gpurun_out/pytest_sc.log
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 50 --warmup 3"
rm -f gpurun_out/scatter_cfg5.jsonl
for sc in regc reg cas chunk atomic atomic_warp color gather; do
 timeout 900 python bench.py $ARGS --scatter $sc > gpurun_out/sc.json 2>gpurun_out/sc_$sc.err; tail -1 gpurun_out/sc.json >> gpurun_out/scatter_cfg5.jsonl
 python -c "
import json,sys; d=json.loads(open('gpurun_out/sc.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$sc', 'ms/step %.4f elem %.4f node %.4f' % (d['ms_per_step'], r['avg_launch_ms']*r['alg_bytes_per_launch']/max(1,r['alg_bytes_per_launch']), r['node_kernel_ms']))"
done
