# Same-box A/B of the working tree against every variant staged under _ab/<name>
# (each a copy of bench.py + package with its own in-tree libfed.so); 2 interleaved reps.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 100 $BENCH_ARGS"
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], 'ms/step %.4f elem %.4f node %.4f' % (d['ms_per_step'], r['avg_launch_ms'], r['node_kernel_ms']))" $1 $2; }
AB=${AB:-_ab}
for i in 1 2; do
 python bench.py $ARGS > gpurun_out/ab_tree.json 2>/dev/null; summ gpurun_out/ab_tree.json tree_r$i
 for v in $AB/*/; do n=$(basename $v)
  (cd $v && python bench.py $ARGS > ../../gpurun_out/ab_$n.json 2>/dev/null); summ gpurun_out/ab_$n.json ${n}_r$i
 done
done
