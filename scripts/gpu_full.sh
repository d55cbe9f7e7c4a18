timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
python __graft_entry__.py --smoke 2>&1 | tail -3
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.log | cut -c1-1500; tail -3 gpurun_out/bench_default.err
