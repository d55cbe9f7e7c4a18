timeout 900 python -m pytest tests -m gpu -x -q -k "fourstep or config4 or stage_forward" 2>&1 | grep -E "FAIL|Error|assert|passed|failed|err" | head -20
for s in "64 64 4096 64" "256 256 4096 64" "64 64 8192 64"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2; done
