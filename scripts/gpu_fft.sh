timeout 900 python -m pytest tests -m gpu -x -q -k "stage or sweep_fp32 or config4" 2>&1 | tail -4
python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c4.log
