# one GPU round: default bench (c5 + c3), c4 bench
python -m pytest tests -m gpu -x -q -k "stage and (4096 or 8192 or 128 or 512)" 2>&1 | tail -1
s=$(date +%s); python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench wall $(( $(date +%s) - s )) s"; tail -1 gpurun_out/bench_default.log | cut -c1-5000; tail -5 gpurun_out/bench_default.err
python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c4.log
