rm -f gpurun_out/stage_ab.log; for w in c3 c5 c2; do python scripts/stage_ab.py --workload $w --opt 5=0 --opt 5=2 >> gpurun_out/stage_ab.log 2>&1; done; grep workload gpurun_out/stage_ab.log
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "tensor_core" 2>&1 | tail -2
