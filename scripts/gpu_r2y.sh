mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "config2 or config3 or sweep_fp32 or zero_rows or operand_scales" 2>&1 | tail -1
for r in 1 2; do for w in c3 c2; do
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 30
done; done
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload c5 --opt 5=0 --steps 6
python scripts/stage_ab.py --workload c5 --opt 5=0 --steps 6
