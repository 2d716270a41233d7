mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step %.4f  G/s %.1f' % (d['ms_per_step'], d['value']/1e9))" $1 $2; }
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 50"
for pr in 0 1 2; do
 FED_FLOW_PROBE=$pr timeout 600 python bench.py $ARGS --n 384 --mode flow > gpurun_out/bf.json 2>gpurun_out/bf.err; summ gpurun_out/bf.json probe$pr
done
