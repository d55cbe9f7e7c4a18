timeout 900 python -m pytest tests -m gpu -x -q -k "variants or sweep_fp32 or config2 or simt or determinism" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
for s in "4096 4096 64 8192" "1024 1024 31 512" "256 256 32 256" "64 64 4096 64"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2 | head -1; done
