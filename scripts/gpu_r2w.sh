mkdir -p gpurun_out
TPROD_LIB=ab/libtprod_forkk0.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "config2 or config3 or config4 or graph or capture or sweep_fp32" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "config2 or config3 or config4 or graph or capture or sweep_fp32" 2>&1 | tail -1
for w in c2 c3 c4; do for r in 1 2; do
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
TPROD_LIB=ab/libtprod_forkk0.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
done; done
