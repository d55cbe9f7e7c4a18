"""Host<->device link probe and the pipelined host entry point at several chunk counts.

    python scripts/e2e_probe.py [n1 n2 n3 n4]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402


def ev_time(fn, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n1, n2, n3, n4 = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (4096, 4096, 64, 8192)
    nb = 2 << 30
    hsrc = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    hdst = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    d2 = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    h2d = ev_time(lambda: d.copy_(hsrc, non_blocking=True))
    d2h = ev_time(lambda: hdst.copy_(d, non_blocking=True))
    s2 = torch.cuda.Stream()

    def both():
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(s2):
            s2.wait_event(ev)
            hdst.copy_(d2, non_blocking=True)
        d.copy_(hsrc, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)
    bo = ev_time(both)
    print(f"H2D {nb / h2d / 1e6:.1f} GB/s, D2H {nb / d2h / 1e6:.1f} GB/s, both concurrently {2 * nb / bo / 1e6:.1f} GB/s "
          f"total ({bo:.1f} ms for 2 x {nb >> 30} GiB)", flush=True)
    del hsrc, hdst, d, d2
    g = torch.Generator().manual_seed(0)
    A = tp.to_matlab(torch.randn(n1, n2, n3, generator=g)).pin_memory()
    B = tp.to_matlab(torch.randn(n2, n4, n3, generator=g)).pin_memory()
    A, B = (x if tp.is_matlab_layout(x) else tp.to_matlab(x) for x in (A, B))
    C = tp.matlab_empty(n1, n4, n3, torch.float32, "cpu").pin_memory()
    F = 8.0 * n1 * n2 * n4 * (n3 // 2 + 1)
    h = tp.Handle()
    for chunks in (0, 16, 32, 64):
        if chunks:
            os.environ["TPROD_HOST_CHUNKS"] = str(chunks)
        tp.tprod_f32_host(A, B, out=C, handle=h)
        ms = ev_time(lambda: tp.tprod_f32_host(A, B, out=C, handle=h), reps=2)
        print(f"{n1}x{n2}x{n3}x{n4} e2e chunks={chunks}: {ms:.1f} ms = {F / ms / 1e9:.1f} TFLOP/s "
              f"(H2D {4 * (n1 * n2 + n2 * n4) * n3 / 1e9:.2f} GB, D2H {4 * n1 * n4 * n3 / 1e9:.2f} GB)", flush=True)


if __name__ == "__main__":
    main()
