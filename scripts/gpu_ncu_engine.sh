bash scripts/gpu_tests.sh
timeout 600 python bench_configs.py c4 --steps 5 > gpurun_out/c4.jsonl 2> gpurun_out/c4.err; tail -2 gpurun_out/c4.err; cat gpurun_out/c4.jsonl
C3="python bench_configs.py c3 --steps 2 --warmup 1"
$C3 > gpurun_out/ncu_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:masked_parity_v2 -s 1 -c 1 -o gpurun_out/prof_c3_parity $C3 > gpurun_out/ncu_c3.log 2>&1
echo "c3 ncu rc=$?"
C5="python bench_configs.py c5 --min-log 26 --max-log 26 --steps 2 --warmup 1"
$C5 > gpurun_out/ncu_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:shuffle_gather_kernel -s 12 -c 4 -o gpurun_out/prof_c5_gather $C5 > gpurun_out/ncu_c5.log 2>&1
echo "c5 ncu rc=$?"
tail -2 gpurun_out/ncu_c5.log
