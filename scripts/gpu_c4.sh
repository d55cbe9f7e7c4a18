python -m pytest tests -m gpu -x -q -k "stage or config4 or sweep" > gpurun_out/pytest_fft.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_fft.log
tail -3 gpurun_out/pytest_fft.log
python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-300; grep -o '"stage_ms[^]]*' gpurun_out/bench_c4.log
timeout 600 ncu --set full --import-source on -k regex:"fft" -c 3 -o gpurun_out/c4_fft2 --force-overwrite python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo NCU=$?
