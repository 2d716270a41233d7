# Chunk launch order (layer-major vs Morton) x L2 evict_first policy on streamed-once loads.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e"
for i in 1 2; do for o in 0 1; do for h in 1 0; do
  FED_L2_STREAM=$h timeout 600 python bench.py $ARGS --chunk-order $o > gpurun_out/bench_k_o$o.h$h.$i.json 2> gpurun_out/bench_k_o$o.h$h.$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_k_o$o.h$h.$i.json'));r=d['roofline'];print('order',$o,'hint',$h,'ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4),'frac',round(r['frac'],3))" || tail -2 gpurun_out/bench_k_o$o.h$h.$i.err
done; done; done
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
for o in 0 1; do for h in 1 0; do
  FED_L2_STREAM=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 12 --csv --log-file gpurun_out/launch_k_o$o.h$h.csv python bench.py $ARGS2 --chunk-order $o > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/launch_k_o$o.h$h.csv")))
i=next(k for k,r in enumerate(rows) if r and r[0]=="ID"); h=rows[i]; d=rows[i+1:]
kn,mn,mv=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value")
agg={}
for r in d:
    if len(r)>mv: agg.setdefault((r[kn][:30],r[mn]),[]).append(float(r[mv].replace(",","")))
for k,v in sorted(agg.items()): print("order $o hint $h",k,round(sum(v[-3:])/3,1))
PY
done; done
