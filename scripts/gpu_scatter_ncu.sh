# ncu counters of every scatter strategy's kernels (cfg5 fp32, a few launches each).
mkdir -p gpurun_out/ncu_scatter
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS="--no-cpu-baseline --no-e2e --no-clocks --steps 2 --warmup 3"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for sc in regc reg chunk cas atomic atomic_warp color gather; do
 python bench.py $ARGS --scatter $sc > gpurun_out/ncu_scatter/pre_$sc.json 2>&1 && \
 timeout 600 ncu --metrics $M --clock-control none --launch-skip 8 -c 12 --csv --log-file gpurun_out/ncu_scatter/$sc.csv python bench.py $ARGS --scatter $sc > gpurun_out/ncu_scatter/log_$sc.txt 2>&1; echo $sc=$?
done
