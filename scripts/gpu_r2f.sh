rm -f gpurun_out/stage_ab.log; for w in c3 c5; do python scripts/stage_ab.py --workload $w --opt 5=0 --opt 5=2 >> gpurun_out/stage_ab.log 2>&1; done; grep workload gpurun_out/stage_ab.log
CMD="python scripts/stage_ab.py --workload c3 --opt 5=0 --steps 2"
$CMD > gpurun_out/plain_tc.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dft_tc -s 2 -c 2 -o gpurun_out/prof_tc4 $CMD > gpurun_out/ncu_tc.log 2>&1; echo ncu rc=$?
