mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_flow.py -x -q -k "not full_size" > gpurun_out/pytest_flow.log 2>&1; echo flow=$?; tail -3 gpurun_out/pytest_flow.log
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step %.4f  G/s %.1f' % (d['ms_per_step'], d['value']/1e9))" $1 $2; }
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 100"
for n in 384 192; do
 timeout 600 python bench.py $ARGS --n $n --mode flow > gpurun_out/bf.json 2>gpurun_out/bf.err; summ gpurun_out/bf.json flow_n$n
done
