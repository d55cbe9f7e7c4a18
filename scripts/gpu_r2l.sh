mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag_f64_launches.csv python scripts/diag_f64.py > gpurun_out/diag_f64.log 2>&1; tail -3 gpurun_out/diag_f64.log
python scripts/diag_f64.py
bash scripts/gpu_profile.sh c4 "cl_|fwd4|inv4" > /dev/null 2>&1; echo prof done
python - <<'PY'
import json
d = json.load(open("gpurun_out/p_c4_summary.json"))
for k in (d if isinstance(d, list) else d.get("kernels", d)):
    print(k if isinstance(k, str) else json.dumps(k)[:400])
PY
