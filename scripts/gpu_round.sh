mkdir -p gpurun_out
timeout 900 python scripts/all_configs.py --configs paper_ti,paper_td,tet160,tet160 --precisions 32,64 --scatter 4 > gpurun_out/tet_perf_reg.log 2>&1; grep cfg gpurun_out/tet_perf_reg.log | cut -c1-260
timeout 900 python scripts/all_configs.py --configs paper_ti,tet160 --precisions 32 --scatter 5 > gpurun_out/tet_perf_regc.log 2>&1; grep cfg gpurun_out/tet_perf_regc.log | cut -c1-260
