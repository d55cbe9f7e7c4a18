"""The multi-rank branch of bench.py, run for real without an 8-GPU node: two ranks (torchrun,
world size 2) on the one GPU gpurun provides, torch collectives over gloo, A replicated by the
host broadcast (replicate(handle=None)).  The ranks' kernels never wait on one another (the
lateral-slice partition has no exchange, Eq. (9)), so sharing one GPU changes only
the timings, not what is tested: the shard split, the max-over-ranks timing and every rank's
shard vs the fp64 oracle (bench.py's parity sample, reduced over ranks)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload", ["c2", "c3"])
def test_bench_two_ranks_gloo_one_gpu(workload):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", workload, "--dist-backend", "gloo",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    n4 = d["config"]["n4"]
    assert d["n_gpus"] == 2 and d["config"]["n4_per_gpu"] == (n4 + 1) // 2
    assert d["parity_rel_err_sampled"] <= 1e-5                    # every rank's shard vs the oracle
    assert "max over ranks" in d["parity_sample"]
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] >= 3 * 4
    assert d["roofline"]["call_frac"] > 0
