# ncu --set full capture of one step of a workload (default config 5), exported on the box to CSV +
# a per-kernel JSON summary (gpurun_out/ is capped at 64 MiB, so no .ncu-rep is brought back).
#   bash scripts/gpu_profile.sh [c5|c4|c3|c2] [kernel regex]
w=${1:-c5}; k=${2:-"tube|fwd|inv|absmax|gemm|fft"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 8 -o /tmp/p_$w --force-overwrite python scripts/profile_step.py $w > gpurun_out/ncu_p_$w.log 2>&1; echo rc=$?
ncu -i /tmp/p_$w.ncu-rep --page raw --csv > gpurun_out/p_${w}_raw.csv 2>/dev/null
ncu -i /tmp/p_$w.ncu-rep --page details > gpurun_out/p_${w}_details.txt 2>/dev/null
python scripts/ncu_summary.py gpurun_out/p_${w}_raw.csv gpurun_out/p_${w}_summary.json --gemm-traffic gpurun_out/r2_${w}_gemm_ncu.json
