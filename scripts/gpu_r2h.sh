rm -f gpurun_out/stage_ab.log
for mb in 0 40 24; do TPROD_4STEP_L2_MB=$mb python scripts/stage_ab.py --workload c4 --opt 5=0 --steps 20 >> gpurun_out/stage_ab.log 2>&1; done; grep workload gpurun_out/stage_ab.log
python scripts/bench_f64.py c3 5; python scripts/bench_f64.py c2 10
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fp64 or fourstep or config4 or prepared or operand_scales" 2>&1 | tail -2
