timeout 900 python -m pytest tests -m gpu -x -q -k "host_entry or prepared or fourstep or config4" 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['e2e'])"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['e2e'])"
