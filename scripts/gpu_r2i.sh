# Tables kernel: 6 CTAs/SM (driver carveout) vs 7 CTAs/SM (max carveout), ncu of the default.
mkdir -p gpurun_out
for v in main v7; do
  if [ $v = main ]; then L=paper_1909_03355_b200/libfed.so; else L=paper_1909_03355_b200/libfed_$v.so; fi
  for i in 1 2; do FED_LIB=$PWD/$L timeout 900 python scripts/next_rows_perf.py --steps 100 --only tables > gpurun_out/tab_i_$v$i.jsonl 2> gpurun_out/tab_i_$v$i.err; echo "$v $(cat gpurun_out/tab_i_$v$i.jsonl)"; done
done
FED_LIB=$PWD/paper_1909_03355_b200/libfed.so timeout 600 python scripts/next_rows_perf.py --steps 100 --only base
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"element_chunk" --launch-skip 2 -c 1 -o gpurun_out/prof_tables_i -f python scripts/next_rows_perf.py --only tables --steps 5 > gpurun_out/ncu_tables_i.log 2>&1; echo ncutab=$?
python scripts/ncu_summary.py gpurun_out/prof_tables_i.ncu-rep --out gpurun_out/ncu_tables_i.json
