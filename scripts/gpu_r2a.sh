set -x
timeout 900 python -m pytest tests/test_bench_multirank_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_multirank.log 2>&1; tail -3 gpurun_out/pytest_multirank.log
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$?; tail -c 600 gpurun_out/bench_default.log
