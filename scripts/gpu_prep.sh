timeout 900 python -m pytest tests -m gpu -x -q -k "prepared or variants or config2 or errors or host_entry" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['prepared_a'], d['gpu_launches'])"
