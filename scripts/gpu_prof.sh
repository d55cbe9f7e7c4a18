# ncu evidence: launch list of the default bench command and full captures of each kernel class.
# Reports are exported to CSV/text on the box (gpurun_out is capped at 64 MiB).
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
for w in c5 c3 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -o /tmp/full_$w --force-overwrite -s 5 -c 5 python scripts/profile_step.py $w > gpurun_out/ncu_full_$w.log 2>&1; echo $w rc=$?
  ncu -i /tmp/full_$w.ncu-rep --page raw --csv > gpurun_out/full_${w}_raw.csv 2>/dev/null
  ncu -i /tmp/full_$w.ncu-rep --page details > gpurun_out/full_${w}_details.txt 2>/dev/null
  ncu -i /tmp/full_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/full_${w}_source.csv 2>/dev/null
  ls -la /tmp/full_$w.ncu-rep
done
du -sh gpurun_out; ls -la gpurun_out
