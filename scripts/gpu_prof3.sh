timeout 900 ncu --set full --clock-control none -k regex:"gemm" -c 1 -o /tmp/g5 --force-overwrite python scripts/profile_step.py c5 > gpurun_out/ncu_g5.log 2>&1; echo rc=$?
ncu -i /tmp/g5.ncu-rep --page raw --csv > gpurun_out/g5_raw.csv 2>/dev/null
ncu -i /tmp/g5.ncu-rep --page details > gpurun_out/g5_details.txt 2>/dev/null
python scripts/ncu_summary.py gpurun_out/g5_raw.csv gpurun_out/g5_summary.json --gemm-traffic gpurun_out/r1_c5_gemm_ncu.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
