# Node-kernel regression hunt: library variants (PDL instructions off / plain launches) + ncu of the node kernel.
mkdir -p gpurun_out
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks"
for v in main v1 v2 v3; do
  if [ $v = main ]; then L=paper_1909_03355_b200/libfed.so; else L=paper_1909_03355_b200/libfed_$v.so; fi
  FED_PDL=0 FED_LIB=$PWD/$L timeout 600 python bench.py $ARGS > gpurun_out/bench_f_$v.json 2> gpurun_out/bench_f_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_f_$v.json'));r=d['roofline'];print('$v','ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4))" || tail -3 gpurun_out/bench_f_$v.err
done
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
FED_PDL=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"node_kernel" --launch-skip 3 -c 1 -o gpurun_out/prof_node_f -f python bench.py $ARGS2 > gpurun_out/ncu_node_f.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/prof_node_f.ncu-rep --out gpurun_out/ncu_node_f.json
