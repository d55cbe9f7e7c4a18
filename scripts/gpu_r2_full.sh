# Round-2 validation on one B200: GPU tests, smoke, default bench, the bench's ncu launch list, and
# ncu --set full captures of config 5 / 4 / 3 (per-kernel summaries for profiles/).
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$?; tail -c 300 gpurun_out/bench_default.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra c3 > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
for w in c5 c4 c3; do bash scripts/gpu_profile.sh $w > /dev/null 2>&1; echo prof $w done; done
