timeout 600 python -m pytest tests -m gpu -x -q -k "argument_errors" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none -k regex:"tube|absmax|inv_|gemm" -c 6 -o /tmp/p5 --force-overwrite python scripts/profile_step.py c5 > gpurun_out/ncu_p5.log 2>&1; echo rc=$?
ncu -i /tmp/p5.ncu-rep --page raw --csv > gpurun_out/p5_raw.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/p5_raw.csv gpurun_out/p5_summary.json --gemm-traffic gpurun_out/r1_c5_gemm_ncu.json
