w=${1:-c5}; k=${2:-"tube|absmax|inv_|fwd_"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 6 -o /tmp/p_$w --force-overwrite python scripts/profile_step.py $w > gpurun_out/ncu_p_$w.log 2>&1; echo rc=$?
ncu -i /tmp/p_$w.ncu-rep --page raw --csv > gpurun_out/p_${w}_raw.csv 2>/dev/null
ncu -i /tmp/p_$w.ncu-rep --page details > gpurun_out/p_${w}_details.txt 2>/dev/null
python scripts/ncu_summary.py gpurun_out/p_${w}_raw.csv gpurun_out/p_${w}_summary.json
