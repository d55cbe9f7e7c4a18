for o in -1 0 6; do
  TPROD_GEMM_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm" -c 1 python scripts/profile_step.py c5 2>&1 | grep -E "dram__|gpu__time|tensor|per_second" | sed "s/^/order $o /"
done
for o in -1 0; do TPROD_GEMM_ORDER=$o timeout 300 python scripts/gemm_variants.py 4096 4096 64 8192 --quick 2>&1 | tail -2 | head -1 | sed "s/^/order $o /"; done
