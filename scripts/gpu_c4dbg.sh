# Default overlap order (3) tests + config-4 GEMM per-role wait cycles (TPROD_GEMM_DEBUG).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "k3_overlap or variants_bitwise or fused_column" 2>&1 | tail -1
TPROD_GEMM_DEBUG=1 timeout 300 python scripts/stage_ab.py --workload c4 --opt 9=1 --steps 3 2>&1 | grep "tprod gemm" | tail -2
TPROD_GEMM_DEBUG=1 timeout 300 python scripts/stage_ab.py --workload c2 --opt 9=1 --steps 3 2>&1 | grep "tprod gemm" | tail -2
timeout 300 python scripts/stage_ab.py --workload c3 --opt 9=0 --opt 9=1 --steps 40 2>&1 | tail -2
