"""Time the K2 GEMM stage of the production path for each GEMM variant (TPROD_OPT_GEMM_CLUSTER /
TPROD_OPT_GEMM_BN) on a given shape and check that all variants are bitwise identical.

    python scripts/gemm_variants.py [n1 n2 n3 n4] [--reps R]

Inputs are torch.randn on the device (timing only; parity is covered by tests/).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n1, n2, n3, n4 = (int(x) for x in args[:4]) if len(args) >= 4 else (1024, 1024, 31, 512)
    reps = 10
    g = torch.Generator(device="cuda").manual_seed(0)
    A = tp.to_matlab(torch.randn(n1, n2, n3, device="cuda", generator=g))
    B = tp.to_matlab(torch.randn(n2, n4, n3, device="cuda", generator=g))
    flops = 8.0 * n1 * n2 * n4 * (n3 // 2 + 1)
    ref = None
    variants = ((128, 1, 0), (128, 2, 0), (128, 3, 0), (0, 0, 0), (0, 0, 1))
    if "--quick" in sys.argv:
        variants = ((0, 0, 0), (0, 0, 1))
    for bn, cn, tr in variants:
        h = tp.Handle()
        h.set_option(tp._lib.TPROD_OPT_GEMM_BN, bn)
        h.set_option(tp._lib.TPROD_OPT_GEMM_CLUSTER, cn)
        h.set_option(tp._lib.TPROD_OPT_TRANSFORM, tr)
        C = tp.tprod(A, B, handle=h)
        torch.cuda.synchronize()
        h.set_option(tp._lib.TPROD_OPT_TIMING, 1)
        ks = []
        for _ in range(reps):
            tp.tprod(A, B, out=C, handle=h)
            ks.append(h.last_stage_ms())
        torch.cuda.synchronize()
        k2 = sorted(k[2] for k in ks)[reps // 2]
        same = "ref" if ref is None else ("bitwise-equal" if torch.equal(C, ref) else
                                          f"differs: max rel {((C - ref).abs().max() / ref.abs().max()).item():.2e}")
        if ref is None:
            ref = C.clone()
        stages = [round(sorted(k[i] for k in ks)[reps // 2], 4) for i in range(4)]
        print(f"{n1}x{n2}x{n3} * {n2}x{n4}x{n3}  bn={bn} cn={cn} transform={tr}: K2 {k2:.4f} ms = "
              f"{flops / k2 / 1e9:.1f} TFLOP/s  stages {stages}  {same}", flush=True)
        h.close()


if __name__ == "__main__":
    main()
