timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 900 python bench_configs.py c1 --steps 10 > gpurun_out/c1.jsonl 2> gpurun_out/c1.err; tail -3 gpurun_out/c1.err; cat gpurun_out/c1.jsonl
timeout 900 python bench_configs.py c3 > gpurun_out/c3.jsonl 2> gpurun_out/c3.err; tail -3 gpurun_out/c3.err; cat gpurun_out/c3.jsonl
timeout 1500 python bench_configs.py c5 --max-log ${MAXLOG:-28} > gpurun_out/c5.jsonl 2> gpurun_out/c5.err; tail -3 gpurun_out/c5.err; cat gpurun_out/c5.jsonl
