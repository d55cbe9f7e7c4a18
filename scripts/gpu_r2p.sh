mkdir -p gpurun_out
for w in c2 c4 c3; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launch_$w.csv python scripts/profile_step.py $w > /dev/null 2>&1
done
python - <<'PY'
import csv
for w in ("c2", "c4", "c3"):
    rows = list(csv.reader(open(f"gpurun_out/launch_{w}.csv")))
    hdr = None; seen = []
    for r in rows:
        if "Kernel Name" in r: hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r)); seen.append((d["ID"], d["Kernel Name"][:50], d["Metric Name"], d["Metric Value"]))
    print(w)
    for s in seen[len(seen)//2:]: print("  ", s)
PY
