CMD="python scripts/stage_ab.py --workload c3 --opt 5=0 --steps 2"
$CMD > gpurun_out/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dft_tc -s 2 -c 2 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_tc.log
