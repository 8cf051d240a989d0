CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_fss_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active --clock-control none -k regex:fss_eval_kernel -s 1 -c 1 --csv --log-file gpurun_out/ncu_fss_full.csv $CMD > gpurun_out/ncu_fss_full.log 2>&1
echo rc=$?
