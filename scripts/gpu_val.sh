# Validation of HEAD on one B200: GPU tests, smoke, default bench (config 5 + extra keys c3/c4/c2).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/val_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/val_pytest.log
python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/val_bench.log 2> gpurun_out/val_bench.err; echo bench rc=$?; tail -1 gpurun_out/val_bench.log | cut -c1-300
