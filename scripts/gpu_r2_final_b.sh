# Round 2 evidence, part 2: real-time capacity (the paper's 5 ms criterion) and tet workloads.
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > $O/build_b.log 2>&1
timeout 2400 python scripts/realtime_capacity.py --sizes 384 512 640 768 > $O/r2_realtime_capacity.jsonl 2> $O/realtime.err; echo cap=$?; cat $O/r2_realtime_capacity.jsonl
timeout 900 python scripts/all_configs.py --configs paper_ti,paper_td,tet160 --max-steps 500 > $O/r2_tet_perf.jsonl 2> $O/tet.err; echo tet=$?; cat $O/r2_tet_perf.jsonl
