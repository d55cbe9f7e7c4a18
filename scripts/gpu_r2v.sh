mkdir -p gpurun_out
for r in 1 2; do
python scripts/stage_ab.py --workload c3 --opt 5=0 --steps 30
TPROD_LIB=ab/libtprod_forkall.so python scripts/stage_ab.py --workload c3 --opt 5=0 --steps 30
done
python scripts/stage_ab.py --workload c5 --opt 5=0 --steps 8
TPROD_LIB=ab/libtprod_forkall.so python scripts/stage_ab.py --workload c5 --opt 5=0 --steps 8
