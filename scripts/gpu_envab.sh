# Same-box A/B of an environment switch: A = with $AB_ENV set, B = without.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -k "rich_trajectory or config_trajectory or one_step or group" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 100 $BENCH_ARGS"
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], 'ms/step %.4f elem %.4f node %.4f' % (d['ms_per_step'], r['avg_launch_ms'], r['node_kernel_ms']))" $1 $2; }
for i in 1 2; do
 env $AB_ENV python bench.py $ARGS > gpurun_out/abA.json 2>/dev/null; summ gpurun_out/abA.json A$i
 python bench.py $ARGS > gpurun_out/abB.json 2>/dev/null; summ gpurun_out/abB.json B$i
done
if [ -n "$PROJ" ]; then
 env $AB_ENV timeout 900 python scripts/slab_projection.py --ranks 1 8 --out gpurun_out/projA.jsonl > /dev/null 2>&1
 timeout 900 python scripts/slab_projection.py --ranks 1 8 --out gpurun_out/projB.jsonl > /dev/null 2>&1
 python -c "
import json
for t in 'AB':
  for l in open(f'gpurun_out/proj{t}.jsonl'):
    r=json.loads(l); print(t, r['P'], 'group %.4f'%r['group_ms_per_step_1gpu'])"
fi
