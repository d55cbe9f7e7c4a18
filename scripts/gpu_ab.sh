timeout 900 python -m pytest tests -m gpu -x -q -k "sweep_fp32 or config4 or config2 or prepared or config3" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head
for rep in 1 2; do
for lib in ab/libtprod_HEAD.so paper_1806_07247_b200/libtprod.so; do
  echo "== $lib"
  for s in "64 64 4096 64" "1024 1024 31 512" "256 256 32 256" "4096 4096 64 8192"; do TPROD_LIB=$PWD/$lib timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2 | head -1; done
done
done
