set -x
python bench.py > gpurun_out/final_bench_cfg5.json 2> gpurun_out/final_bench_cfg5.err
SBG_PCG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --tts-runs 1 --dl-grid 0 > gpurun_out/launches_cfg5.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
ncu --metrics $M --clock-control none -k regex:'k_far_tiles|k_near_leaves' --launch-skip 2 -c 2 --csv python tools/asm_once.py 5 > gpurun_out/asm5_metrics.csv 2> gpurun_out/asm5_metrics.err
ncu --set full --clock-control none --import-source on -k regex:'k_far_tiles|k_near_leaves|k_sauter_partial' --launch-skip 5 -c 5 -o gpurun_out/asm2_full python tools/asm_once.py 2 > gpurun_out/asm2_full.log 2>&1
echo done
