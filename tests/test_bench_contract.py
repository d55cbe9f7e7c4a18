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


def test_roofline_call_frac_and_stage_rates():
    """The bench line's roofline: GEMM fraction against bf16/3, SURVEY 8(d)'s whole-call fraction
    T_roof / T with T_roof = max(F / P, B / BW), and the memory-bound stages' algorithmic GB/s."""
    sys.path.insert(0, ROOT)
    import bench
    n1, n2, n3, n4 = 1024, 1024, 31, 512
    peaks = {"hbm_gbs": 6000.0, "bf16_tflops": 1500.0, "bf16_tflops_sustained": 1200.0}
    meas = {"gemm_flops_local": bench.gemm_flops(n1, n2, n3, n4), "gemm_ms": 0.2,
            "metric_flops_local": bench.metric_flops(n1, n2, n3, n4),
            "compulsory_bytes_local": 4.0 * n3 * (n1 * n2 + n2 * n4 + n1 * n4),
            "stage_bytes_local": bench.stage_bytes(n1, n2, n3, n4),
            "stage_ms": [0.05, 0.1, 0.2, 0.05], "ms": 0.5}
    r = bench.roofline(meas, peaks, "test", "c3", sustained=False)
    P = 1500.0 / 3
    assert abs(r["peak"] - P) < 1e-9
    assert abs(r["achieved"] - bench.gemm_flops(n1, n2, n3, n4) / 0.2e-3 / 1e12) < 1e-9
    t_roof = max(bench.metric_flops(n1, n2, n3, n4) / (P * 1e12),
                 4.0 * n3 * (n1 * n2 + n2 * n4 + n1 * n4) / 6000e9)
    assert abs(r["call_frac"] - t_roof * 1e3 / 0.5) < 1e-12
    h = n3 // 2 + 1
    k1 = (4 * n3 + 8 * h) * (n1 * n2 + n2 * n4) / 0.1e-3 / 1e9
    assert abs(r["stages"]["K1 forward DFT (A, B)"]["GB/s"] - k1) < 1e-6
    assert abs(r["stages"]["K3 fill + inverse DFT"]["frac"] - (8 * h + 4 * n3) * n1 * n4 / 0.05e-3 / 1e9 / 6000) < 1e-9
    rs = bench.roofline(meas, peaks, "test", "c3", sustained=True)
    assert abs(rs["peak"] - 400.0) < 1e-9
    # concurrent A / B chains: the library reports K0 + K1 as stage 0 and 0 for stage 1
    meas2 = dict(meas, stage_ms=[0.12, 0.0, 0.2, 0.05])
    r2 = bench.roofline(meas2, peaks, "test", "c3", sustained=False)
    comb = r2["stages"]["K0 + K1 scales and forward DFTs (A, B chains concurrent)"]
    sb = bench.stage_bytes(n1, n2, n3, n4)
    assert abs(comb["GB/s"] - (sb["K0"] + sb["K1"]) / 0.12e-3 / 1e9) < 1e-6
    assert "K1 forward DFT (A, B)" not in r2["stages"] and "K2 GEMM" in r2["stages"]
