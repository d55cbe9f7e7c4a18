timeout 900 python -m pytest tests -m gpu -x -q -k "sweep_fp32 or config4 or config2 or prepared" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head
for s in "64 64 4096 64" "1024 1024 31 512" "4096 4096 64 8192"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2 | head -1; done
