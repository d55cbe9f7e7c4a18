# checkpoint validation: GPU suite, smoke, default bench line (c5 + c3, c4, c2), launch list of c2
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.log").read().strip().splitlines()[-1])
print("c5", round(d["value"], 1), round(d["ms_per_step"], 2), round(d["roofline"]["frac"], 3), round(d["roofline"]["call_frac"], 3), d["clocks"], d["e2e"]["value"])
for k in ("c3", "c4", "c2"):
    x = d.get(k)
    if x: print(k, x.get("ms_per_step"), x.get("value"), x.get("roofline", {}).get("call_frac"), x.get("roofline", {}).get("stage_ms"))
PY
