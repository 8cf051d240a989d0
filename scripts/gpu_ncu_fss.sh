# ncu evidence for the FSS eval kernel (run plain first; ncu only if it exits 0)
CMD="python bench.py --keys 4194304 --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fss.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fss_eval_kernel -s 2 -c 1 -o gpurun_out/prof_fss_eval $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full.log
