mkdir -p gpurun_out
python scripts/stage_ab.py --workload c4 --opt 5=0 --opt 5=3 --steps 20
TPROD_LIB=ab/libtprod_tub16.so python scripts/stage_ab.py --workload c4 --opt 5=3 --opt 5=0 --opt 5=3 --steps 20
TPROD_LIB=ab/libtprod_tub16.so timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "cluster" > gpurun_out/pytest_o.log 2>&1; tail -2 gpurun_out/pytest_o.log; grep -E "^FAILED|^E " gpurun_out/pytest_o.log | head -10
