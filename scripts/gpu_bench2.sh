python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.log | cut -c1-600; tail -2 gpurun_out/bench_default.err
python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c4.log
python bench.py --workload c2 --steps 20 --warmup 5 --no-c3 > gpurun_out/bench_c2.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-400
