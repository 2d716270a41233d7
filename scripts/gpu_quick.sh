mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rich_trajectory or config_trajectory or one_step" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/bq.json 2> gpurun_out/bq.err; echo bench=$?; python -c "
import json; d=json.load(open('gpurun_out/bq.json')); r=d['roofline']; print('ms/step', d['ms_per_step'], 'elem', r['avg_launch_ms'], 'node', r['node_kernel_ms'], 'frac', r['frac'])"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 100 --precision 64 > gpurun_out/bq64.json 2> gpurun_out/bq64.err; echo bench=$?; python -c "
import json; d=json.load(open('gpurun_out/bq64.json')); r=d['roofline']; print('fp64 ms/step', d['ms_per_step'], 'elem', r['avg_launch_ms'], 'node', r['node_kernel_ms'], 'frac', r['frac'])"
