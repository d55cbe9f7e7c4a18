"""Memory-safety checks of the CUDA path without compute-sanitizer (the GPU pool has it closed):

* TPROD_OPT_POISON fills every byte of workspace a call uses with 0xFF (NaN in fp16 / fp32 / fp64)
  before the call: a kernel that reads workspace it did not write first (the initcheck class of
  bug) turns the result into NaN;
* outputs are views into larger buffers whose guard zones before and after hold a sentinel: a
  kernel writing outside its output (the memcheck class, for the outputs) changes a guard;
* inputs are views into guarded buffers too, and must be bitwise unchanged afterwards;
* every case is compared with the fp64 oracle.
The shapes reach every kernel family of libtprod.so (tensor-core DFT, tube / four-step /
mixed-radix / generic / register transforms, single-CTA and CTA-pair GEMMs, fp64, the NEXT rows)
with ragged tiles."""
import numpy as np
import pytest

import oracle as O
from synth import normal

pytestmark = pytest.mark.gpu
GUARD = 4096
SENT = 1.2345e30


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_07247_b200 import build
    build.build()
    import paper_1806_07247_b200 as tp
    return tp


def guarded(shape, dtype, fill=None):
    """A Matlab-layout CUDA tensor of `shape` inside a buffer with GUARD sentinel elements before
    and after; returns (tensor, buffer)."""
    import torch
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), SENT, dtype=dtype, device="cuda")
    t = buf[GUARD:GUARD + n].view(tuple(shape[::-1])).permute(2, 1, 0)
    if fill is not None:
        t.copy_(torch.from_numpy(np.ascontiguousarray(fill)))
    return t, buf


def guards_intact(buf):
    import torch
    torch.cuda.synchronize()
    g = torch.cat([buf[:GUARD], buf[-GUARD:]]).cpu().numpy()
    return bool(np.all(g == np.asarray(SENT, dtype=g.dtype)))


CASES = [
    (20, 30, 10, 15, np.float64), (33, 17, 100, 9, np.float64), (6, 5, 4096, 4, np.float64),
    (20, 30, 10, 15, np.float32), (256, 256, 32, 256, np.float32), (512, 96, 64, 256, np.float32),
    (300, 64, 31, 130, np.float32), (260, 40, 45, 20, np.float32), (64, 40, 45, 20, np.float32),
    (36, 20, 128, 12, np.float32), (33, 17, 100, 9, np.float32), (16, 12, 4096, 8, np.float32),
    (12, 10, 67, 6, np.float32), (1, 1, 1, 1, np.float32), (129, 65, 8, 130, np.float32),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:4])) + "-" + np.dtype(c[4]).name)
def test_poisoned_workspace_and_guarded_buffers(T, case):
    import torch
    n1, n2, n3, n4, dt = case
    tdt = torch.float64 if dt == np.float64 else torch.float32
    A = normal((n1, n2, n3), 3 + n3, dt)
    B = normal((n2, n4, n3), 4 + n3, dt)
    h = T.Handle()
    h.set_option(T._lib.TPROD_OPT_POISON, 1)
    h.set_option(T._lib.TPROD_OPT_GRAPHS, 0)
    dA, bufA = guarded((n1, n2, n3), tdt, A)
    dB, bufB = guarded((n2, n4, n3), tdt, B)
    dC, bufC = guarded((n1, n4, n3), tdt)
    assert T.is_matlab_layout(dA) and T.is_matlab_layout(dC)
    for _ in range(2):                                 # second call: workspace reused, poisoned again
        T.tprod(dA, dB, out=dC, handle=h)
    torch.cuda.synchronize()
    C = dC.cpu().numpy()
    assert np.isfinite(C).all()
    assert guards_intact(bufC) and guards_intact(bufA) and guards_intact(bufB)
    assert np.array_equal(dA.cpu().numpy(), A) and np.array_equal(dB.cpu().numpy(), B)
    cols = np.arange(min(n4, 6))
    ref = O.tprod_columns(A.astype(np.float64), B.astype(np.float64), cols)
    assert O.rel_err(C[:, cols], ref) <= (1e-12 if dt == np.float64 else 1e-5)
    if dt == np.float32 and n4 > 1:                    # prepared operand, poisoned
        h.prepare_a(dA)
        dC2, bufC2 = guarded((n1, n4, n3), tdt)
        T.tprod_prepared(dB, out=dC2, handle=h)
        torch.cuda.synchronize()
        assert guards_intact(bufC2)
        assert np.array_equal(dC2.cpu().numpy(), C)
        h.release_a()


@pytest.mark.parametrize("dims", [(24, 20, 9), (33, 17, 64), (8, 12, 4096), (100, 72, 5), (130, 130, 3)],
                         ids=lambda d: "x".join(map(str, d)))
def test_poisoned_next_rows(T, dims):
    """t-SVT, t-SVD scalars and factors, tinv and the forward stage entry with a poisoned workspace
    and guarded outputs (the last two shapes take the blocked Jacobi and the global-memory
    Gauss-Jordan)."""
    import torch
    n1, n2, n3 = dims
    h = T.Handle()
    h.set_option(T._lib.TPROD_OPT_POISON, 1)
    Y = normal((n1, n2, n3), 61 + n3)
    dY, bufY = guarded((n1, n2, n3), torch.float32, Y)
    dX, bufX = guarded((n1, n2, n3), torch.float32)
    T.tsvt(dY, 2.0, out=dX, handle=h)
    torch.cuda.synchronize()
    assert guards_intact(bufX) and guards_intact(bufY)
    assert O.rel_err(dX.cpu().numpy(), O.tsvt(Y.astype(np.float64), 2.0)) <= 1e-5
    out = T.tsvd_values(dY, rtol=1e-6, handle=h).cpu().numpy()
    assert np.isfinite(out).all()
    U, S, V = (x.cpu().numpy() for x in T.tsvd(dY, handle=h))
    _, S_ref, _ = O.tsvd(Y.astype(np.float64))
    assert O.rel_err(S, S_ref) <= 1e-5 and np.isfinite(U).all() and np.isfinite(V).all()
    n = min(n1, n2)
    Z = normal((n, n, n3), 71 + n3, np.float64) * (0.2 / np.sqrt(n3))   # spectral slices 2 I + O(0.2)
    Z[:, :, 0] += 2.0 * np.eye(n)
    Z = Z.astype(np.float32)
    dZ, bufZ = guarded((n, n, n3), torch.float32, Z)
    dI, bufI = guarded((n, n, n3), torch.float32)
    T.tinv(dZ, out=dI, handle=h)
    assert guards_intact(bufI) and guards_intact(bufZ)
    assert O.rel_err(dI.cpu().numpy(), O.tinv(Z.astype(np.float64))) <= 1e-5
    spec = T.dft_f32(dY, role=0, handle=h).cpu().numpy()
    ref = np.fft.rfft(Y.astype(np.float64), axis=2)
    assert np.linalg.norm(spec - ref) <= 2e-6 * np.linalg.norm(ref)
