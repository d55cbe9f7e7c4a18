# Streaming K2 -> K3 overlap (TPROD_OPT_OVERLAP = 2; n3 = 64, any number of GEMM tile rounds): same-box
# A/B of config 5, arms alternated (option 9: 1 = default, K3 after the GEMM for this shape; 2 = streaming).
mkdir -p gpurun_out
for r in 1 2 3; do
timeout 600 python scripts/stage_ab.py --workload c5 --opt 9=1 --opt 9=2 --steps 10
timeout 600 python scripts/stage_ab.py --workload c5 --opt 9=2 --opt 9=1 --steps 10
done 2>&1 | tee gpurun_out/stream_ab.jsonl
