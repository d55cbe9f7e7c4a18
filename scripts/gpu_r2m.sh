mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fp64 or cluster or fourstep or zero_rows or operand_scales or config4 or config1" > gpurun_out/pytest_m.log 2>&1; tail -2 gpurun_out/pytest_m.log; grep -E "^FAILED" gpurun_out/pytest_m.log | head -20
python bench.py --workload c4 --steps 20 --warmup 5 --extra "" --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"stage_ms[^]]*\|"parity_rel_err_sampled": [0-9.e-]*' gpurun_out/bench_c4.log | head -3
python scripts/diag_f64.py
for w in c4 c3 c2; do timeout 300 python scripts/bench_f64.py $w 5; done
bash scripts/gpu_profile.sh c4 "cl_" > /dev/null 2>&1; echo prof done
grep -E "cl_fwd_kernel<0>|cl_inv|Duration|Executed Ipc Active|Active Warps Per|Eligible Warps|Registers Per|Achieved Occupancy" gpurun_out/p_c4_details.txt | head -30
