"""Timing of the SURVEY 8(f) NEXT rows on one B200 (CUDA events, warm-up, L2 flushed between reps):
prepared-operand t-product (NEXT-1), t-SVT (NEXT-2), t-SVD factors and scalars (NEXT-3), tinv,
tran, teye (NEXT-4).  Each line: ms per call (median), algorithmic HBM bytes (inputs read + outputs
written) and that rate against the measured HBM peak; for the t-product also TFLOP/s.

    python scripts/bench_next.py [--reps R] > profiles/r1_next_rows.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402


def timed(fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 10
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    bw = peaks["hbm_gbs"]
    g = torch.Generator(device="cuda").manual_seed(0)
    rnd = lambda *s: tp.to_matlab(torch.randn(*s, device="cuda", generator=g))
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fl = torch.empty(2 * l2 // 4, device="cuda")
    flush = lambda: fl.zero_()
    h = tp.Handle()
    rows = []

    def row(name, shape, ms, nbytes, flops=None):
        d = {"op": name, "shape": shape, "ms": ms, "bytes": nbytes, "gbs": nbytes / ms / 1e6,
             "hbm_frac": nbytes / ms / 1e6 / bw}
        if flops:
            d["tflops"] = flops / ms / 1e9
        rows.append(d)
        print(json.dumps(d), flush=True)

    # NEXT-1: prepared operand, config 3 shape
    n1, n2, n3, n4 = 1024, 1024, 31, 512
    A, B = rnd(n1, n2, n3), rnd(n2, n4, n3)
    C = tp.tprod(A, B, handle=h)
    full = timed(lambda: tp.tprod(A, B, out=C, handle=h), reps, flush)
    h.prepare_a(A)
    prep = timed(lambda: tp.tprod_prepared(B, out=C, handle=h), reps, flush)
    F = 8.0 * n1 * n2 * n4 * (n3 // 2 + 1)
    row("tprod (config 3)", [n1, n2, n3, n4], full, 4 * n3 * (n1 * n2 + n2 * n4 + n1 * n4), F)
    row("tprod_prepared (config 3, A prepared)", [n1, n2, n3, n4], prep, 4 * n3 * (n2 * n4 + n1 * n4), F)
    h.release_a()
    # NEXT-2 / NEXT-3 / NEXT-4
    for (m, n, k) in ((64, 64, 64), (64, 64, 1024), (32, 48, 255)):
        Y = rnd(m, n, k)
        X = torch.empty_like(Y)
        row("tsvt", [m, n, k], timed(lambda: tp.tsvt(Y, 5.0, out=X, handle=h), reps, flush), 2 * 4 * m * n * k)
        row("tsvd_values", [m, n, k], timed(lambda: tp.tsvd_values(Y, handle=h), reps, flush), 4 * m * n * k)
        r = min(m, n)
        row("tsvd (skinny)", [m, n, k], timed(lambda: tp.tsvd(Y, handle=h), reps, flush),
            4 * k * (m * n + m * r + r * r + n * r))
    for (n, k) in ((64, 64), (96, 31), (32, 4096)):
        Ai = rnd(n, n, k)
        Ai[:, :, 0] += 3.0 * torch.eye(n, device="cuda") * (n ** 0.5)
        Xi = torch.empty_like(Ai)
        row("tinv (synchronous)", [n, n, k], timed(lambda: tp.tinv(Ai, out=Xi, handle=h), reps, flush),
            2 * 4 * n * n * k)
    for (a, b, k) in ((4096, 4096, 16), (1024, 512, 31)):
        At = rnd(a, b, k)
        Ot = tp.matlab_empty(b, a, k, torch.float32, "cuda")
        row("tran", [a, b, k], timed(lambda: tp.tran(At, out=Ot, handle=h), reps, flush), 2 * 4 * a * b * k)
    row("teye", [4096, 64], timed(lambda: tp.teye(4096, 64, handle=h), reps, flush), 4 * 4096 * 4096 * 64)
    print(json.dumps({"next_rows": rows, "hbm_peak_gbs": bw, "device": torch.cuda.get_device_name(0)}))


if __name__ == "__main__":
    main()
