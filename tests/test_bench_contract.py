"""bench.py contract checks that need no GPU: the reference arm (the fp64 oracle timed on the host
cores) prints one JSON line with the keys the driver reads, and the metric flop count follows
BASELINE.json's formula."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_metric_flops_formula():
    sys.path.insert(0, ROOT)
    import bench
    n1, n2, n3, n4 = 1024, 1024, 31, 512
    h = math.ceil((n3 + 1) / 2)
    want = 8 * n1 * n2 * n4 * h + 2.5 * n3 * math.log2(n3) * (n1 * n2 + n2 * n4 + n1 * n4)
    assert bench.metric_flops(n1, n2, n3, n4) == want
    assert bench.h_slices(n3) == h == 16
    assert bench.h_slices(64) == 33 and bench.h_slices(4096) == 2049


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "c2", "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "c2"
