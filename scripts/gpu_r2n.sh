mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "cluster or fp64_longer or fourstep" > gpurun_out/pytest_n.log 2>&1; tail -2 gpurun_out/pytest_n.log; grep -E "^FAILED|^E " gpurun_out/pytest_n.log | head -20
python scripts/stage_ab.py --workload c4 --opt 5=0 --opt 5=3 --opt 5=0 --opt 5=3 --steps 20
