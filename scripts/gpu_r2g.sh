# Node-kernel regression hunt, part 2: the round-1 tree (its own bench.py and library) next to the
# current tree and the runtime-PEER node kernel variant, same box, interleaved.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pci.bus_id,serial,memory.total,clocks.max.mem --format=csv > gpurun_out/g_gpu.txt 2>&1
ARGS="--steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-clocks"
for i in 1 2; do
  (cd _oldtree && timeout 600 python bench.py $ARGS > ../gpurun_out/bench_g_old$i.json 2> ../gpurun_out/bench_g_old$i.err)
  python -c "import json;d=json.load(open('gpurun_out/bench_g_old$i.json'));r=d['roofline'];print('old','ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4))" || tail -3 gpurun_out/bench_g_old$i.err
  for v in main v4; do
    if [ $v = main ]; then L=paper_1909_03355_b200/libfed.so; else L=paper_1909_03355_b200/libfed_$v.so; fi
    FED_PDL=0 FED_LIB=$PWD/$L timeout 600 python bench.py $ARGS > gpurun_out/bench_g_$v$i.json 2> gpurun_out/bench_g_$v$i.err
    python -c "import json;d=json.load(open('gpurun_out/bench_g_$v$i.json'));r=d['roofline'];print('$v','ms',round(d['ms_per_step'],4),'elem',round(r['avg_launch_ms'],4),'node',round(r['node_kernel_ms'],4))" || tail -3 gpurun_out/bench_g_$v$i.err
  done
done
