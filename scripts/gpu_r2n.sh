# Packed connectivity, two layouts: tree = 16-B record (12-bit positions + P_xx) + 5 planes,
# _ab/B = separate 8-B + 4-B connectivity planes + 6 planes, _ab/A = HEAD (16-bit offsets).
# Same-box A/B (fp32), then one ncu --set full launch of each element kernel.
mkdir -p gpurun_out/n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
BENCH_ARGS="--steps 100" bash scripts/gpu_abn.sh
ARGS2="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
for v in tree A B; do
  D=.; [ $v != tree ] && D=_ab/$v
  (cd $D && timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 4 -c 1 -o /root/repo/gpurun_out/n/prof_$v -f python bench.py $ARGS2 > /root/repo/gpurun_out/n/ncu_$v.log 2>&1); echo ncu $v $?
done
