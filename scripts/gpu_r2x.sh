# Diagnosis of the per-slab fixed costs at 8 slabs (cfg5 fp32, PEER rank group on one GPU):
# ncu full capture of one element and every node kernel launch of one eager step.
mkdir -p gpurun_out/x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x/build.log 2>&1; echo build=$?
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:"node_kernel|element_chunk" \
  --launch-skip 16 -c 16 -o gpurun_out/x/slab8 -f python scripts/slab_launches.py --ranks 8 --steps 2 > gpurun_out/x/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/x/ncu.log
ncu -i gpurun_out/x/slab8.ncu-rep --page raw --csv > gpurun_out/x/slab8_raw.csv 2>/dev/null; echo raw=$?
python scripts/ncu_lines.py gpurun_out/x/slab8.ncu-rep --kernel node_kernel --top 30 > gpurun_out/x/node_lines.txt 2>&1
