"""Host-side issue cost of one t-product call vs its device time (is a small problem launch-bound?).

    python scripts/host_overhead.py [n1 n2 n3 n4]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402


def main():
    args = [int(a) for a in sys.argv[1:5]] if len(sys.argv) >= 5 else [256, 256, 32, 256]
    n1, n2, n3, n4 = args
    g = torch.Generator(device="cuda").manual_seed(0)
    A = tp.to_matlab(torch.randn(n1, n2, n3, device="cuda", generator=g))
    B = tp.to_matlab(torch.randn(n2, n4, n3, device="cuda", generator=g))
    h = tp.Handle()
    C = tp.tprod(A, B, handle=h)
    torch.cuda.synchronize()
    reps = 200
    for trial in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            tp.tprod(A, B, out=C, handle=h)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"{n1}x{n2}x{n3}x{n4}: host issue {1e6 * (t1 - t0) / reps:.1f} us/call, device "
              f"{1e3 * e0.elapsed_time(e1) / reps:.1f} us/call (back to back, L2 warm)", flush=True)
    # a single call bracketed by a sync on both sides (what the bench step sees, minus its L2 flush)
    ts = []
    for _ in range(50):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tp.tprod(A, B, out=C, handle=h)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"single call (synced): median {1e3 * ts[len(ts) // 2]:.1f} us", flush=True)


if __name__ == "__main__":
    main()
