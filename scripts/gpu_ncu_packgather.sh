# one --set full capture of the fused pack+gather and the wide gather (C3 online fetch)
CMD="python bench_configs.py c3p --steps 1 --warmup 0"
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"pack_gather_rows|shuffle_gather_kernel<0>" -c 2 \
    -o gpurun_out/c3p_fetch $CMD > gpurun_out/c3p_fetch_ncu.log 2>&1
echo rc=$?
