timeout 900 python -m pytest tests -m gpu -x -q -k "variants or sweep_fp32 or config3 or config2 or determinism or prepared" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head
for rep in 1 2; do
for lib in ab/libtprod_HEAD.so paper_1806_07247_b200/libtprod.so; do
  echo "== $lib"
  for s in "1024 1024 31 512" "1024 1024 64 512" "4096 4096 64 8192"; do TPROD_LIB=$PWD/$lib timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2 | head -1; done
done
done
