# ncu --set full captures of this session's new top kernels (outputs in gpurun_out/)
C4="python bench_configs.py c4 --steps 2 --warmup 1"
$C4 > gpurun_out/ncu_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:masked_parity_tma -s 1 -c 1 -o gpurun_out/prof_c4_parity_tma $C4 > gpurun_out/ncu_c4.log 2>&1
echo "c4 ncu rc=$?"
C5="python bench_configs.py c5 --min-log 24 --max-log 24 --steps 2 --warmup 1"
$C5 > gpurun_out/ncu_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:plan_partition_tma|plan_chain|win_gather_dual" -s 5 -c 5 -o gpurun_out/prof_c5_chain $C5 > gpurun_out/ncu_c5.log 2>&1
echo "c5 ncu rc=$?"
