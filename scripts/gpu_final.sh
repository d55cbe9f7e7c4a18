# Round-end style validation on one B200: GPU tests, smoke, the default bench (config 5 + config 3),
# configs 4 and 2, the bench's ncu launch list, and a config-4 ncu capture.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
python __graft_entry__.py --smoke 2>&1 | tail -3
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.log | cut -c1-400; tail -2 gpurun_out/bench_default.err
python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c4.log
python bench.py --workload c2 --steps 20 --warmup 5 --no-c3 > gpurun_out/bench_c2.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*' gpurun_out/bench_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
bash scripts/gpu_profile.sh c4 "fwd4|inv4|absmax|gemm" > /dev/null 2>&1; echo c4prof done
