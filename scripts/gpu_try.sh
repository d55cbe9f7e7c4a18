timeout 900 python -m pytest tests -m gpu -x -q -k "variants or tube or sweep_fp32 or stage_forward" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
for s in "4096 4096 64 8192" "1024 1024 31 512" "1024 1024 128 512"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2; done
timeout 900 ncu --set full --clock-control none -k regex:"gemm" -c 1 -o /tmp/g5 --force-overwrite python scripts/profile_step.py c5 > gpurun_out/ncu_g5.log 2>&1; echo rc=$?
ncu -i /tmp/g5.ncu-rep --page raw --csv > gpurun_out/g5_raw.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/g5_raw.csv gpurun_out/g5_summary.json --gemm-traffic gpurun_out/r1_c5_gemm_ncu.json
