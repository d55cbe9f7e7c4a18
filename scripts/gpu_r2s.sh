mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_memory_safety_gpu.py -q -p no:cacheprovider -k "graph or capture or config2 or config4 or sweep_fp32 or prepared or host or poison or guard or determinism" > gpurun_out/pytest_s.log 2>&1; tail -2 gpurun_out/pytest_s.log; grep -E "^FAILED|^E " gpurun_out/pytest_s.log | head -10
for w in c2 c4 c3; do
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
done
python scripts/host_overhead.py 2>&1 | tail -4
