# Element/node kernel time vs chunk size and mesh size (streaming path, fp32).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], 'ms/step %.4f elem %.4f node %.4f' % (d['ms_per_step'], r['avg_launch_ms'], r['node_kernel_ms']))" $1 $2; }
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 100"
for n in 384 192 128; do
 for ch in 1024 512; do
  timeout 600 python bench.py $ARGS --n $n --chunk $ch > gpurun_out/cs.json 2>/dev/null; summ gpurun_out/cs.json n${n}_c$ch
 done
done
