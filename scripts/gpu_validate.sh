# One-B200 validation of HEAD: GPU tests, smoke, the default bench line and configs 4 / 2.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$?; tail -c 400 gpurun_out/bench_default.log
