# Round-1 refresh of every measured number (run under gpurun; outputs in gpurun_out/)
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_dcf.json 2> $O/bench_dcf.err; tail -c 300 $O/bench_dcf.json
timeout 600 python bench.py --kind dpf --no-query > $O/bench_dpf.json 2> $O/bench_dpf.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 200 $O/bench_ref.json
timeout 900 python bench_configs.py c1 --steps 20 > $O/c1.jsonl 2> $O/c1.err
timeout 900 python bench_configs.py c3 > $O/c3.jsonl 2> $O/c3.err
timeout 900 python bench_configs.py c3p > $O/c3p.jsonl 2> $O/c3p.err
timeout 900 python bench_configs.py c4 > $O/c4.jsonl 2> $O/c4.err
timeout 1500 python bench_configs.py c5 --min-log 16 --max-log 28 > $O/c5.jsonl 2> $O/c5.err
timeout 600 python bench_configs.py funcs > $O/funcs.jsonl 2> $O/funcs.err
for f in c1 c3 c3p c4 c5; do echo "$f: $(wc -l < $O/$f.jsonl) lines; $(tail -1 $O/$f.err)"; done
# launch list of the headline command (cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-query --no-c4 > $O/bench_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench_configs.py access > $O/access.jsonl 2> $O/access.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:select_fold --csv \
  python bench_configs.py access --steps 2 --warmup 1 > $O/access_ncu.csv 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  python scripts/exp_trio_gpu.py > $O/trio_c1_launches.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "regex:plan_|win_gather" --csv python bench_configs.py c5 --min-log 24 --max-log 24 --steps 2 --warmup 1 > $O/c5_24_ncu.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "regex:masked_parity|zero_share" --csv python bench_configs.py c4 --steps 2 --warmup 1 > $O/c4_ncu.csv 2>&1
echo refresh-done
