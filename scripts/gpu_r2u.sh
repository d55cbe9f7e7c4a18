mkdir -p gpurun_out
for L in ab/libtprod_inv32.so ab/libtprod_inv16.so; do
TPROD_LIB=$L timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fourstep or config4 or stage_inverse or zero_rows or operand_scales" 2>&1 | tail -1
done
for r in 1 2; do
python scripts/stage_ab.py --workload c4 --opt 5=0 --steps 30
TPROD_LIB=ab/libtprod_inv32.so python scripts/stage_ab.py --workload c4 --opt 5=0 --steps 30
TPROD_LIB=ab/libtprod_inv16.so python scripts/stage_ab.py --workload c4 --opt 5=0 --steps 30
done
