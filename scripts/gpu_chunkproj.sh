# Per-rank kernel time of the 1- and 8-slab cfg5 partitions vs chunk size (one GPU, projection).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for ch in 1024 512 256; do
 timeout 900 python scripts/slab_projection.py --ranks 1 8 --chunk $ch --out gpurun_out/chunkproj_$ch.jsonl > gpurun_out/chunkproj_$ch.log 2>&1; echo chunk=$ch rc=$?
 python -c "
import json,sys
for l in open(sys.argv[1]):
    r=json.loads(l); e=max(x['element_ms'] for x in r['per_rank']); n=max(x['node_ms'] for x in r['per_rank'])
    print(sys.argv[2], 'P', r['P'], 'elem %.4f node %.4f proj %.4f group %.4f' % (e, n, r['projected_ms_per_step'], r['group_ms_per_step_1gpu']))" gpurun_out/chunkproj_$ch.jsonl $ch
done
