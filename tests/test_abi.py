"""CPU-side checks of the C-ABI boundary (-m "not gpu"): the library builds/loads, exports every
symbol include/tprod.h declares, and its pure host functions behave.  No compute calls."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "tprod.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tprod_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    from paper_1806_07247_b200 import build, _lib
    build.build()
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    syms = _declared_symbols()
    assert len(syms) >= 16
    from paper_1806_07247_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == syms, "binding must cover exactly the header's entry points"
    for s in syms:
        assert hasattr(L, s), f"libtprod.so does not export {s}"


def test_strerror(L):
    from paper_1806_07247_b200 import _lib
    for code in range(8):
        assert L.tprod_strerror(code)
    assert b"overlap" in L.tprod_strerror(_lib.TPROD_EALIAS)
    assert L.tprod_strerror(999) == b"unknown tprod status"


def test_workspace_bytes(L):
    from paper_1806_07247_b200 import workspace_bytes, _lib
    # fp32: h * (4 planes fp16 * (n2*lda + n4*ldb)) + fp32 re/im C-bar + scale vectors
    n1, n2, n3, n4 = 1024, 1024, 31, 512
    h = n3 // 2 + 1
    exp_min = h * 8 * (n2 * n1 + n4 * n2) + h * 8 * n4 * n1
    got = workspace_bytes(n1, n2, n3, n4)
    assert exp_min <= got <= exp_min + 1 << 16
    got64 = workspace_bytes(20, 30, 10, 15, _lib.TPROD_DTYPE_F64)
    assert got64 >= 6 * 16 * (20 * 30 + 30 * 15 + 20 * 15)
    with pytest.raises(_lib.TprodError) as e:
        workspace_bytes(0, 1, 1, 1)
    assert e.value.status == _lib.TPROD_EINVAL
    with pytest.raises(_lib.TprodError):
        workspace_bytes(1, 1, 1, 1, 7)
    with pytest.raises(_lib.TprodError):
        workspace_bytes(1 << 20, 1 << 20, 1 << 20, 1)   # element-count overflow


def test_argument_errors_before_any_device_work(L):
    from paper_1806_07247_b200 import _lib
    # NULL handle / pointers are rejected synchronously (no GPU needed)
    assert L.tprod_f32(None, None, None, 1, 1, 1, 1, None, None) == _lib.TPROD_EINVAL
    assert L.tprod_f64(None, None, None, 1, 1, 1, 1, None, None) == _lib.TPROD_EINVAL
    h = C.c_void_p()
    assert L.tprod_create(0, C.byref(h)) != _lib.TPROD_OK or h.value  # no GPU here: error, not crash
    assert L.tprod_set_option(None, 1, 0) == _lib.TPROD_EINVAL
    assert L.tprod_destroy(None) == _lib.TPROD_EINVAL
    assert L.tprod_bcast_f32(None, None, 1, 0, None) == _lib.TPROD_EINVAL


def test_sass_is_sm100a():
    """The built library carries sm_100a SASS (the only target compiled)."""
    import shutil
    import subprocess
    lib = os.path.join(ROOT, "paper_1806_07247_b200", "libtprod.so")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
