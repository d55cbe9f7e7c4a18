mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fourstep or config4 or config2 or zero_rows or operand_scales or stage_inverse or extreme or sweep_fp32" > gpurun_out/pytest_r.log 2>&1; tail -2 gpurun_out/pytest_r.log; grep -E "^FAILED|^E " gpurun_out/pytest_r.log | head -10
for w in c4 c2 c3; do
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 20
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 20
TPROD_LIB=ab/libtprod_HEAD.so python scripts/stage_ab.py --workload $w --opt 5=0 --steps 20
python scripts/stage_ab.py --workload $w --opt 5=0 --steps 20
done
