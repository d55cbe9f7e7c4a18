# Streaming K2 -> K3 overlap (n3 = 64, any number of GEMM tile rounds): bitwise tests, then same-box
# A/B of config 5 (option 9: 0 = serial, 2 = short-run overlap only, 1 = streaming) and a config-3 check.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "k3_stream or k3_overlap or config5 or graph_replay or prepared_operand" 2>&1 | tail -3
for r in 1 2; do
timeout 600 python scripts/stage_ab.py --workload c5 --opt 9=0 --opt 9=1 --opt 9=2 --steps 8
done
timeout 300 python scripts/stage_ab.py --workload c3 --opt 9=0 --opt 9=1 --steps 30
