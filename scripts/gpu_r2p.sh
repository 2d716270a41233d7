# 16-bit shared-node lists (tree) vs HEAD (_ab/A, int32 lists): same-box A/B fp32 + fp64,
# ncu DRAM bytes of the element kernel, GPU tests on the tree.
mkdir -p gpurun_out/p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
BENCH_ARGS="--steps 100 --precision 64" bash scripts/gpu_abn.sh
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
for v in tree A; do
  D=.; [ $v = A ] && D=_ab/A
  (cd $D && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file /root/repo/gpurun_out/p/launch_$v.csv python bench.py $ARGS2 > /dev/null 2>&1)
  python scripts/ncu_lines.py --help > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/p/launch_$v.csv")))
i=next(k for k,r in enumerate(rows) if r and r[0]=="ID"); h=rows[i]; d=rows[i+1:]
kn,mn,mv=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value")
agg={}
for r in d:
    if len(r)>mv: agg.setdefault((r[kn][:30],r[mn]),[]).append(float(r[mv].replace(",","")))
for k,v in sorted(agg.items()): print("$v",k,round(sum(v[-3:])/3,1))
PY
done
T0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? $(( $(date +%s) - T0 ))s; tail -3 gpurun_out/pytest_gpu.log
