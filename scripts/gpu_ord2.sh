# Overlap counter variants on config 3 (TPROD_OV_ORDER bits: 1 = m,f,n order, 2 = one arrive per CTA
# after a named barrier, 4 = red.release instead of fence + atomic): stage A/B, GEMM alone under ncu.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "k3_overlap" 2>&1 | tail -1
for o in 2 6; do TPROD_OV_ORDER=$o timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "k3_overlap" 2>&1 | tail -1; done
for r in 1 2; do for o in 0 2 6 3; do
TPROD_OV_ORDER=$o timeout 300 python scripts/stage_ab.py --workload c3 --opt 9=1 --steps 40 2>&1 | tail -1 | sed "s/^/ord$o /"
done; done
for o in 0 2 6; do
TPROD_OV_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -c 8 --csv python scripts/stage_ab.py --workload c3 --opt 9=1 --steps 3 2>/dev/null | grep gemm_tc2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/ncu ord$o gemm ns: /"; echo
done
