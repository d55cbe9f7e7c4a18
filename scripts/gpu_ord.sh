# Overlap tile order A/B on config 3 (TPROD_OV_ORDER 0 = f fastest, 1 = m, f, n), plus the GEMM's own
# duration per order under ncu (kernels serialised there: no overlap, the GEMM alone).
mkdir -p gpurun_out
for r in 1 2; do for o in 0 1; do
TPROD_OV_ORDER=$o timeout 300 python scripts/stage_ab.py --workload c3 --opt 9=1 --steps 40 2>&1 | tail -1 | sed "s/^/ord$o /"
done; done
timeout 300 python scripts/stage_ab.py --workload c3 --opt 9=0 --steps 40 2>&1 | tail -1
for o in 0 1; do
TPROD_OV_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -c 12 --csv python scripts/stage_ab.py --workload c3 --opt 9=1 --steps 3 2>/dev/null | grep gemm_tc2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/ncu ord$o gemm ns: /"; echo
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -c 12 --csv python scripts/stage_ab.py --workload c3 --opt 9=0 --steps 3 2>/dev/null | grep gemm_tc2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/ncu serial gemm ns: /"; echo
