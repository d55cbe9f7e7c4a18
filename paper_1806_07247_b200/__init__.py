"""B200-native t-product (Lu, Tensor-Tensor Product Toolbox, arXiv 1806.07247).

    C = A * B = fold(bcirc(A) . unfold(B))          (Definition 2.1, Eq. (9))

computed by Algorithm 1 in hand-written sm_100a CUDA kernels behind the C ABI
of include/tprod.h.  This module is the thin Python binding: it checks shapes and strides,
allocates outputs with torch, and passes raw device pointers plus the current CUDA stream to
libtprod.so.  torch is used for device memory, streams and process groups only.

Tensors use the Matlab layout of the ABI: a torch tensor of shape (n1, n2, n3) whose element
(i, j, k) lives at offset i + n1*j + n1*n2*k, i.e. strides (1, n1, n1*n2).  ``matlab_empty`` and
``to_matlab`` produce such tensors.
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import TprodError, check, lib, strerror, workspace_bytes  # noqa: F401

__all__ = ["Handle", "tprod", "tprod_f32", "tprod_f64", "tprod_prepared", "tran", "teye", "tinv", "tsvt", "tsvd_values", "tsvd", "tsvd_full", "tprod_f32_host", "tprod_f64_host",
           "matlab_empty", "to_matlab", "is_matlab_layout", "dft_f32", "idft_f32",
           "nccl_unique_id", "workspace_bytes", "TprodError", "h_slices"]


def h_slices(n3: int) -> int:
    """ceil((n3+1)/2): frequency slices multiplied by Algorithm 1."""
    return n3 // 2 + 1


def is_matlab_layout(t) -> bool:
    """True if element (i,j,k) of the 3-D tensor t is at i + n1*j + n1*n2*k (contiguous).
    Stride test (what permute(2, 1, 0).is_contiguous() decides, without building a view: this
    runs on every call)."""
    if t.dim() != 3:
        return False
    n1, n2, n3 = t.shape
    if n1 == 0 or n2 == 0 or n3 == 0:
        return True
    s0, s1, s2 = t.stride()
    return (n1 == 1 or s0 == 1) and (n2 == 1 or s1 == n1) and (n3 == 1 or s2 == n1 * n2)


def matlab_empty(n1: int, n2: int, n3: int, dtype=None, device="cuda"):
    import torch
    return torch.empty((n3, n2, n1), dtype=dtype or torch.float32, device=device).permute(2, 1, 0)


def to_matlab(t):
    """Copy a 3-D tensor into the Matlab layout (no-op if it already has it)."""
    return t if is_matlab_layout(t) else t.permute(2, 1, 0).contiguous().permute(2, 1, 0)


class Handle:
    """Owns a tprod_handle: device binding, plan/DFT tables, workspace, optional NCCL world."""

    def __init__(self, device: int | None = None):
        import torch
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        h = C.c_void_p()
        check(lib().tprod_create(self.device, C.byref(h)), f"tprod_create(device={self.device})")
        self._h = h

    @property
    def ptr(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().tprod_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option: int, value: int):
        check(lib().tprod_set_option(self._h, option, value), "tprod_set_option")

    def last_launch_count(self) -> int:
        out = C.c_int64()
        check(lib().tprod_last_launch_count(self._h, C.byref(out)), "tprod_last_launch_count")
        return out.value

    def status(self, stream=None) -> int:
        """TPROD_STATUS_* bits the handle's kernels raised since the last query (SINGULAR from an
        asynchronous tinv, NOCONVERGE from an SVD slice that hit its sweep cap); synchronises
        `stream` (default: the current stream) and clears the word (tprod_status)."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        out = C.c_int()
        check(lib().tprod_status(self._h, C.c_void_p(s.cuda_stream), C.byref(out)), "tprod_status")
        return out.value

    def last_stage_ms(self):
        """[K0 scales, K1 forward, K2 GEMM, K3 inverse] durations (ms) of the last fp32 call
        (requires set_option(TPROD_OPT_TIMING, 1) before the call)."""
        out = (C.c_float * 4)()
        check(lib().tprod_last_stage_ms(self._h, out), "tprod_last_stage_ms")
        return [float(x) for x in out]

    def prepare_a(self, A, stream=None):
        """Prepared left operand (NEXT-1): run A's scales + forward DFT once (tprod_prepare_a_f32);
        later tprod_prepared(B) calls on this handle reuse it.  A: float32 CUDA, Matlab layout."""
        import torch
        if A.dim() != 3 or A.dtype != torch.float32 or not A.is_cuda:
            raise ValueError("prepare_a needs a 3-D float32 CUDA tensor")
        if not is_matlab_layout(A):
            raise ValueError("A must have the Matlab layout (strides (1, n1, n1*n2)); use to_matlab()")
        n1, n2, n3 = (int(x) for x in A.shape)
        s = stream if stream is not None else torch.cuda.current_stream(A.device)
        check(lib().tprod_prepare_a_f32(A.data_ptr(), n1, n2, n3, C.c_void_p(s.cuda_stream), self._h),
              "tprod_prepare_a_f32")
        self.prepared = (n1, n2, n3)
        return self

    def release_a(self):
        check(lib().tprod_release_a(self._h), "tprod_release_a")
        self.prepared = None

    def set_world(self, rank: int, world: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = C.create_string_buffer(uid, 128)
        check(lib().tprod_set_world(self._h, rank, world, buf), "tprod_set_world")

    def bcast_(self, t, root: int = 0, stream=None):
        """In-place ncclBroadcast of a contiguous CUDA tensor from `root` (setup-time only)."""
        import torch
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("bcast_ needs a contiguous CUDA tensor")
        fn = {torch.float32: lib().tprod_bcast_f32, torch.float64: lib().tprod_bcast_f64}.get(t.dtype)
        if fn is None:
            raise TypeError(f"bcast_: unsupported dtype {t.dtype}")
        s = stream if stream is not None else torch.cuda.current_stream(t.device)
        check(fn(self._h, t.data_ptr(), t.numel(), root, C.c_void_p(s.cuda_stream)), "tprod_bcast")
        return t


_handles: dict[int, Handle] = {}


def _default_handle(device: int) -> Handle:
    h = _handles.get(device)
    if h is None:
        h = _handles[device] = Handle(device)
    return h


def _shapes(A, B):
    if A.dim() != 3 or B.dim() != 3 or A.shape[1] != B.shape[0] or A.shape[2] != B.shape[2]:
        raise ValueError(f"t-product shape mismatch: A {tuple(A.shape)} vs B {tuple(B.shape)} "
                         "(need A n1 x n2 x n3 and B n2 x n4 x n3)")
    n1, n2, n3 = A.shape
    return int(n1), int(n2), int(n3), int(B.shape[1])


def _check_out(out, shape, dtype, device, name="out"):
    """A caller-supplied output must match exactly what the kernels will write: shape, dtype,
    device (CUDA index or CPU) and the Matlab layout -- anything else would be an out-of-bounds
    or wrong-device write inside the library."""
    if tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != device:
        raise ValueError(f"{name} must be a {tuple(shape)} {dtype} tensor on {device}, got "
                         f"{tuple(out.shape)} {out.dtype} on {out.device}")
    if not is_matlab_layout(out):
        raise ValueError(f"{name} must have the Matlab layout (strides (1, n1, n1*n2)); use matlab_empty()")
    return out


def _call(fn_name, A, B, out=None, handle=None, stream=None):
    import torch
    n1, n2, n3, n4 = _shapes(A, B)
    if not (A.is_cuda and B.is_cuda) or A.device != B.device:
        raise ValueError("A and B must be CUDA tensors on the same device")
    if A.dtype != B.dtype:
        raise TypeError(f"dtype mismatch {A.dtype} vs {B.dtype}")
    if not (is_matlab_layout(A) and is_matlab_layout(B)):
        raise ValueError("A and B must have the Matlab layout (strides (1, n1, n1*n2)); use to_matlab()")
    dev = A.device.index
    if out is None:
        out = matlab_empty(n1, n4, n3, A.dtype, A.device)
    else:
        _check_out(out, (n1, n4, n3), A.dtype, A.device)
    h = handle or _default_handle(dev)
    s = stream if stream is not None else torch.cuda.current_stream(A.device)
    st = getattr(lib(), fn_name)(A.data_ptr(), B.data_ptr(), out.data_ptr(), n1, n2, n3, n4,
                                 C.c_void_p(s.cuda_stream), h.ptr)
    check(st, fn_name)
    return out


def tprod_prepared(B, out=None, handle=None, stream=None):
    """C = A * B for the A prepared on `handle` (Handle.prepare_a); bitwise equal to tprod_f32(A, B)."""
    import torch
    h = handle
    if h is None or getattr(h, "prepared", None) is None:
        raise ValueError("tprod_prepared needs a handle with a prepared A (Handle.prepare_a)")
    n1, n2, n3 = h.prepared
    if B.dim() != 3 or B.shape[0] != n2 or B.shape[2] != n3:
        raise ValueError(f"t-product shape mismatch: prepared A ({n1}, {n2}, {n3}) vs B {tuple(B.shape)}")
    if B.dtype != torch.float32 or not B.is_cuda or not is_matlab_layout(B):
        raise ValueError("B must be a float32 CUDA tensor in the Matlab layout")
    n4 = int(B.shape[1])
    if out is None:
        out = matlab_empty(n1, n4, n3, torch.float32, B.device)
    else:
        _check_out(out, (n1, n4, n3), torch.float32, B.device)
    s = stream if stream is not None else torch.cuda.current_stream(B.device)
    check(lib().tprod_f32_prepared(B.data_ptr(), out.data_ptr(), n4, C.c_void_p(s.cuda_stream), h.ptr),
          "tprod_f32_prepared")
    return out


def _h_s(t, handle, stream):
    import torch
    h = handle or _default_handle(t.device.index)
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    return h, C.c_void_p(s.cuda_stream)


def tran(A, out=None, handle=None, stream=None):
    """A^* (Definition 2.2): n2 x n1 x n3, slice 0 transposed, slices 1.. reversed and transposed."""
    import torch
    if A.dim() != 3 or not A.is_cuda or not is_matlab_layout(A):
        raise ValueError("tran needs a 3-D CUDA tensor in the Matlab layout")
    n1, n2, n3 = (int(x) for x in A.shape)
    if out is None:
        out = matlab_empty(n2, n1, n3, A.dtype, A.device)
    else:
        _check_out(out, (n2, n1, n3), A.dtype, A.device)
    fn = {torch.float32: lib().tprod_tran_f32, torch.float64: lib().tprod_tran_f64}.get(A.dtype)
    if fn is None:
        raise TypeError(f"tran: unsupported dtype {A.dtype}")
    h, s = _h_s(A, handle, stream)
    check(fn(A.data_ptr(), out.data_ptr(), n1, n2, n3, s, h.ptr), "tprod_tran")
    return out


def teye(n: int, n3: int, dtype=None, device="cuda", handle=None, stream=None):
    """The n x n x n3 identity tensor (Definition 2.3), written by the library."""
    import torch
    dtype = dtype or torch.float32
    out = matlab_empty(n, n, n3, dtype, device)
    fn = {torch.float32: lib().tprod_teye_f32, torch.float64: lib().tprod_teye_f64}.get(dtype)
    if fn is None:
        raise TypeError(f"teye: unsupported dtype {dtype}")
    h, s = _h_s(out, handle, stream)
    check(fn(out.data_ptr(), n, n3, s, h.ptr), "tprod_teye")
    return out


def tinv(A, out=None, handle=None, stream=None):
    """A^-1 (Definition 2.4, Eq. (11)) for a float32 n x n x n3 CUDA tensor (n <= 8192).  By default
    synchronous, raising TprodError (status TPROD_ESINGULAR) if a spectral slice is singular to
    working precision; with handle.set_option(TPROD_OPT_SYNC_CHECKS, 0) asynchronous, singularity
    then reported by handle.status()."""
    import torch
    if A.dim() != 3 or A.shape[0] != A.shape[1] or A.dtype != torch.float32 or not A.is_cuda:
        raise ValueError("tinv needs a float32 n x n x n3 CUDA tensor")
    if not is_matlab_layout(A):
        raise ValueError("A must have the Matlab layout (strides (1, n1, n1*n2)); use to_matlab()")
    n, _, n3 = (int(x) for x in A.shape)
    if out is None:
        out = matlab_empty(n, n, n3, torch.float32, A.device)
    else:
        _check_out(out, (n, n, n3), torch.float32, A.device)
    h, s = _h_s(A, handle, stream)
    check(lib().tprod_tinv_f32(A.data_ptr(), out.data_ptr(), n, n3, s, h.ptr), "tprod_tinv_f32")
    return out


def tsvt(Y, tau: float, out=None, handle=None, stream=None):
    """Prox of tau * TNN (Algorithm 3, t-SVT) for a float32 n1 x n2 x n3 CUDA tensor (any slice
    size: one CTA per spectral slice up to 64 x 64, a blocked Jacobi beyond)."""
    import torch
    if Y.dim() != 3 or Y.dtype != torch.float32 or not Y.is_cuda or not is_matlab_layout(Y):
        raise ValueError("tsvt needs a float32 3-D CUDA tensor in the Matlab layout")
    n1, n2, n3 = (int(x) for x in Y.shape)
    if out is None:
        out = matlab_empty(n1, n2, n3, torch.float32, Y.device)
    else:
        _check_out(out, (n1, n2, n3), torch.float32, Y.device)
    h, s = _h_s(Y, handle, stream)
    check(lib().tprod_tsvt_f32(Y.data_ptr(), out.data_ptr(), n1, n2, n3, C.c_float(tau), s, h.ptr),
          "tprod_tsvt_f32")
    return out


def tsvd_values(A, rtol: float = 1e-6, handle=None, stream=None):
    """t-SVD scalars of a float32 n1 x n2 x n3 CUDA tensor (any slice size): returns a CUDA float32
    vector [S(1,1,1) .. S(r,r,1), TNN, TSN, tubal rank] (Eq. (14), Def. 2.9, Def. 2.8, Eq. (16))."""
    import torch
    if A.dim() != 3 or A.dtype != torch.float32 or not A.is_cuda or not is_matlab_layout(A):
        raise ValueError("tsvd_values needs a float32 3-D CUDA tensor in the Matlab layout")
    n1, n2, n3 = (int(x) for x in A.shape)
    out = torch.empty(min(n1, n2) + 3, dtype=torch.float32, device=A.device)
    h, s = _h_s(A, handle, stream)
    check(lib().tprod_tsvd_values_f32(A.data_ptr(), n1, n2, n3, C.c_float(rtol), out.data_ptr(), s, h.ptr),
          "tprod_tsvd_values_f32")
    return out


def tsvd(A, handle=None, stream=None):
    """Skinny t-SVD (Algorithm 2) of a float32 n1 x n2 x n3 CUDA tensor (any slice size):
    returns (U n1 x r x n3, S r x r x n3, V n2 x r x n3) with A = U * S * V^*."""
    import torch
    if A.dim() != 3 or A.dtype != torch.float32 or not A.is_cuda or not is_matlab_layout(A):
        raise ValueError("tsvd needs a float32 3-D CUDA tensor in the Matlab layout")
    n1, n2, n3 = (int(x) for x in A.shape)
    r = min(n1, n2)
    U = matlab_empty(n1, r, n3, torch.float32, A.device)
    S = matlab_empty(r, r, n3, torch.float32, A.device)
    V = matlab_empty(n2, r, n3, torch.float32, A.device)
    h, s = _h_s(A, handle, stream)
    check(lib().tprod_tsvd_f32(A.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), n1, n2, n3, s, h.ptr),
          "tprod_tsvd_f32")
    return U, S, V


def tsvd_full(A, handle=None, stream=None):
    """Full t-SVD (Theorem 2.2) of a float32 n1 x n2 x n3 CUDA tensor: returns (U n1 x n1 x n3,
    S n1 x n2 x n3, V n2 x n2 x n3) with A = U * S * V^*, U and V orthogonal."""
    import torch
    if A.dim() != 3 or A.dtype != torch.float32 or not A.is_cuda or not is_matlab_layout(A):
        raise ValueError("tsvd_full needs a float32 3-D CUDA tensor in the Matlab layout")
    n1, n2, n3 = (int(x) for x in A.shape)
    U = matlab_empty(n1, n1, n3, torch.float32, A.device)
    S = matlab_empty(n1, n2, n3, torch.float32, A.device)
    V = matlab_empty(n2, n2, n3, torch.float32, A.device)
    h, s = _h_s(A, handle, stream)
    check(lib().tprod_tsvd_full_f32(A.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), n1, n2, n3, s, h.ptr),
          "tprod_tsvd_full_f32")
    return U, S, V


def tprod_f32(A, B, out=None, handle=None, stream=None):
    """C = A * B for float32 CUDA tensors (asynchronous on the current stream)."""
    import torch
    if A.dtype != torch.float32:
        raise TypeError("tprod_f32 needs float32 tensors")
    return _call("tprod_f32", A, B, out, handle, stream)


def tprod_f64(A, B, out=None, handle=None, stream=None):
    """C = A * B for float64 CUDA tensors."""
    import torch
    if A.dtype != torch.float64:
        raise TypeError("tprod_f64 needs float64 tensors")
    return _call("tprod_f64", A, B, out, handle, stream)


def tprod(A, B, out=None, handle=None, stream=None):
    """C = A * B (Definition 2.1) for float32 or float64 CUDA tensors in the Matlab layout."""
    import torch
    if A.dtype == torch.float32:
        return tprod_f32(A, B, out, handle, stream)
    if A.dtype == torch.float64:
        return tprod_f64(A, B, out, handle, stream)
    raise TypeError(f"unsupported dtype {A.dtype}")


def _host_call(fn_name, dtype, A, B, out, handle, stream, device):
    """End-to-end call on HOST tensors (pinned recommended): H2D, t-product, D2H, synchronise.
    The library copies sizeof(dtype) bytes per element from A, B and into out, so all three are
    checked for exactly that dtype, shape and layout (a mismatch would be a host over-read /
    overflow inside the library)."""
    import torch
    n1, n2, n3, n4 = _shapes(A, B)
    if A.is_cuda or B.is_cuda:
        raise ValueError("*_host entry points take CPU tensors")
    if A.dtype != dtype or B.dtype != dtype:
        raise TypeError(f"{fn_name} needs {dtype} tensors, got {A.dtype} and {B.dtype}")
    if not (is_matlab_layout(A) and is_matlab_layout(B)):
        raise ValueError("A and B must have the Matlab layout")
    if out is None:
        out = matlab_empty(n1, n4, n3, dtype, "cpu")
    else:
        _check_out(out, (n1, n4, n3), dtype, torch.device("cpu"))
    h = handle or _default_handle(device if device is not None else torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(h.device)
    check(getattr(lib(), fn_name)(A.data_ptr(), B.data_ptr(), out.data_ptr(), n1, n2, n3, n4,
                                  C.c_void_p(s.cuda_stream), h.ptr), fn_name)
    return out


def tprod_f32_host(A, B, out=None, handle=None, stream=None, device=None):
    import torch
    return _host_call("tprod_f32_host", torch.float32, A, B, out, handle, stream, device)


def tprod_f64_host(A, B, out=None, handle=None, stream=None, device=None):
    import torch
    return _host_call("tprod_f64_host", torch.float64, A, B, out, handle, stream, device)


def dft_f32(X, role: int = 0, handle=None):
    """Stage entry: Hermitian-half mode-3 DFT of a float32 Matlab-layout CUDA tensor through the
    production kernels (split operand format decoded back to fp32).  Returns complex (p, q, h)."""
    import torch
    p, q, n3 = (int(x) for x in X.shape)
    hh = h_slices(n3)
    re = torch.empty((hh, q, p), dtype=torch.float32, device=X.device)
    im = torch.empty_like(re)
    h = handle or _default_handle(X.device.index)
    s = torch.cuda.current_stream(X.device)
    check(lib().tprod_dft_f32(to_matlab(X).data_ptr(), re.data_ptr(), im.data_ptr(), p, q, n3, role,
                              C.c_void_p(s.cuda_stream), h.ptr), "tprod_dft_f32")
    return torch.complex(re, im).permute(2, 1, 0)


def idft_f32(Xbar, n3: int, handle=None):
    """Stage entry: inverse of dft_f32 with the fused conjugate fill.  Xbar: complex (p, q, h)."""
    import torch
    p, q, hh = (int(x) for x in Xbar.shape)
    if hh != h_slices(n3):
        raise ValueError("Xbar must hold the h = n3//2+1 Hermitian-half slices")
    re = Xbar.real.permute(2, 1, 0).contiguous().float()
    im = Xbar.imag.permute(2, 1, 0).contiguous().float()
    out = matlab_empty(p, q, n3, torch.float32, Xbar.device)
    h = handle or _default_handle(Xbar.device.index)
    s = torch.cuda.current_stream(Xbar.device)
    check(lib().tprod_idft_f32(re.data_ptr(), im.data_ptr(), out.data_ptr(), p, q, n3,
                               C.c_void_p(s.cuda_stream), h.ptr), "tprod_idft_f32")
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().tprod_nccl_unique_id(buf), "tprod_nccl_unique_id")
    return buf.raw
