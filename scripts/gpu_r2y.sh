# Node kernel: boundary group first + grouped special-node operands (tree) vs HEAD (_ab/A),
# and the tree with the round-1 order (FED_BND_FIRST=0); P=1 bench and the 8-slab projection;
# then the GPU test suite on the tree.
mkdir -p gpurun_out/y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y/build.log 2>&1; echo build=$?
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 200"
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], 'ms/step %.4f elem %.4f node %.4f' % (d['ms_per_step'], r['avg_launch_ms'], r['node_kernel_ms']))" $1 $2; }
for i in 1 2; do
  python bench.py $ARGS > gpurun_out/y/t.json 2>/dev/null; summ gpurun_out/y/t.json tree_r$i
  FED_BND_FIRST=0 python bench.py $ARGS > gpurun_out/y/t0.json 2>/dev/null; summ gpurun_out/y/t0.json tree_bndlast_r$i
  (cd _ab/A && python bench.py $ARGS > ../../gpurun_out/y/a.json 2>/dev/null); summ gpurun_out/y/a.json A_r$i
done
timeout 900 python scripts/slab_projection.py --ranks 1 8 --out gpurun_out/y/proj8_tree.jsonl > gpurun_out/y/proj8_tree.log 2>&1; echo proj_tree=$?
(cd _ab/A && timeout 900 python scripts/slab_projection.py --ranks 1 8 --out ../../gpurun_out/y/proj8_A.jsonl > ../../gpurun_out/y/proj8_A.log 2>&1); echo proj_A=$?
for f in tree A; do python -c "
import json,sys; d=json.loads(open('gpurun_out/y/proj8_$f.jsonl').read().strip().splitlines()[-1])
print('$f', 'alone', round(max(d['alone_ms_per_step']),5), 'eff', round(d.get('projected_alone_efficiency_vs_P1',0),3), 'events', round(d['projected_ms_per_step'],5), 'group', round(d['group_ms_per_step_1gpu']/8,5), 'node', [round(r['node_ms'],4) for r in d['per_rank']])"; done
T0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/y/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/y/pytest_gpu.log
