CMD="python bench_configs.py c3p --steps 1 --warmup 0"
$CMD > gpurun_out/c3p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3p_launches.csv $CMD > gpurun_out/c3p_ncu.log 2>&1
echo rc=$?
