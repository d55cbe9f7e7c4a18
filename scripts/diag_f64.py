"""fp64 path: one t-product per shape, CUDA-event timed (run under an ncu launch list to see which
transform kernels ran).  python scripts/diag_f64.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1806_07247_b200 as tp
from synth import normal

for (n1, n2, n3, n4) in [(16, 16, 4096, 16), (64, 64, 4096, 64)]:
    A = tp.to_matlab(torch.from_numpy(normal((n1, n2, n3), 1, np.float64)).cuda())
    B = tp.to_matlab(torch.from_numpy(normal((n2, n4, n3), 2, np.float64)).cuda())
    h = tp.Handle()
    C = tp.tprod(A, B, handle=h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tp.tprod(A, B, out=C, handle=h)
    e1.record()
    torch.cuda.synchronize()
    print((n1, n2, n3, n4), "ms", e0.elapsed_time(e1), flush=True)
