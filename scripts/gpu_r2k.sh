# fp64 FFT transforms + one-pass cluster transforms (n3 = 4096): targeted GPU tests, c4 bench, fp64 timings.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "fp64 or cluster or stage or fourstep or zero_rows or operand_scales or config4 or c4 or prepared" > gpurun_out/pytest_k.log 2>&1; tail -3 gpurun_out/pytest_k.log; grep -E "^FAILED|Error|error" gpurun_out/pytest_k.log | head -20
python bench.py --workload c4 --steps 20 --warmup 5 --extra "" --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*\|"parity_rel_err_sampled": [0-9.e-]*' gpurun_out/bench_c4.log | head -4
for w in c4 c3 c2; do timeout 300 python scripts/bench_f64.py $w 5; done
