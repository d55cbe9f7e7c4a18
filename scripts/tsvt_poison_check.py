import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O
import paper_1806_07247_b200 as T
from synth import normal
for dims in [(24, 20, 9), (33, 17, 64), (8, 12, 4096)]:
    n1, n2, n3 = dims
    Y = normal((n1, n2, n3), 61 + n3)
    ref = O.tsvt(Y.astype(np.float64), 2.0)
    for poison in (0, 1):
        h = T.Handle()
        h.set_option(T._lib.TPROD_OPT_POISON, poison)
        dY = torch.from_numpy(np.asfortranarray(Y)).cuda()
        X = T.tsvt(dY, 2.0, handle=h)
        torch.cuda.synchronize()
        print(dims, "poison", poison, "rel_err", O.rel_err(X.cpu().numpy(), ref), flush=True)
