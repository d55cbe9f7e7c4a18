# K2 -> K3 overlap: new parity test, neighbouring GEMM/transform tests, same-box stage A/B on c3/c2.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "k3_overlap or variants_bitwise or config2 or sweep_fp32 or prepared" 2>&1 | tail -5
for w in c3 c2; do
timeout 300 python scripts/stage_ab.py --workload $w --opt 9=0 --opt 9=1 --steps 30 2>&1 | tail -4
done
timeout 300 python bench.py --workload c3 --steps 20 --warmup 5 --no-c3 --extra "" > gpurun_out/ov_c3.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/ov_c3.log | head -2
