# Fused column scales of B (K0 of B inside K1 of B): tests + same-box stage A/B on c3 / c2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "fused_column or k3_overlap or operand_scales or zero_rows or extreme or config2 or sweep_fp32 or prepared or determinism" 2>&1 | tail -5
for w in c3 c2; do
timeout 300 python scripts/stage_ab.py --workload $w --opt 10=0 --opt 10=1 --opt 10=0 --opt 10=1 --steps 30 2>&1 | tail -4
done
