timeout 900 python -m pytest tests -m gpu -x -q -k "tube or sweep_fp32 or config2" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head
for rep in 1 2; do for s in "4096 4096 64 8192" "1024 1024 64 512" "1024 1024 128 512" "1024 1024 256 256"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2; done; done
