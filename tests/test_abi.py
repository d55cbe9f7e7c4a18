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


def test_sass_summary_matches_build(L):
    """Per-kernel SASS evidence of the tcgen05 / TMEM / TMA path, recomputed from the built library
    (scripts/sass_summary.py) and compared with the committed profiles/sass_summary.json: the GEMM
    kernels issue UTCHMMA (2-CTA in the pair kernel), load operands with UTMALDG and read TMEM
    with LDTM; the tube / four-step transforms move tiles with UTMALDG / UTMASTG."""
    import json
    import shutil
    import sys
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import sass_summary
    got = sass_summary.summary(os.path.join(ROOT, "paper_1806_07247_b200", "libtprod.so"))
    assert got["arch"] == ["sm_100a"]

    def fam(name, d):
        return {k: v for k, v in d["kernels"].items() if name in k}
    pair = fam("gemm_tc2_kernel", got)
    assert pair and all(v.get("UTCHMMA.2CTA", 0) > 0 and v.get("LDTM.x16", 0) > 0 and
                        v.get("UTMALDG.3D.2CTA", 0) > 0 for v in pair.values())
    single = fam("gemm_tc_kernel", got)
    assert single and all(v.get("UTCHMMA", 0) > 0 and v.get("LDTM.x16", 0) > 0 for v in single.values())
    for name in ("fwd_dft_tc_kernel", "inv_dft_tc_kernel"):       # DFT-matrix contraction on tcgen05
        ks = fam(name, got)
        assert ks and all(v.get("UTCHMMA", 0) > 0 and v.get("UTMALDG.3D", 0) > 0 and v.get("LDTM.x8", 0) > 0
                          for v in ks.values()), name
    for name in ("fwd_tube_kernel", "inv_tube_kernel"):
        ks = fam(name, got)
        assert ks and all(v.get("UTMALDG.3D", 0) > 0 and v.get("UTMASTG.3D", 0) > 0 for v in ks.values()), name
    for name in ("fwd4_pass1_kernel", "inv4_pass2_kernel"):
        ks = fam(name, got)
        assert ks and all(v.get("UTMALDG.4D", 0) > 0 and v.get("UTMASTG.4D", 0) > 0 for v in ks.values()), name
    with open(os.path.join(ROOT, "profiles", "sass_summary.json")) as f:
        committed = json.load(f)
    assert committed["kernels"] == got["kernels"], "profiles/sass_summary.json is stale: rerun scripts/sass_summary.py"


def test_binding_rejects_mismatched_host_and_out_arguments():
    """The host entry points copy sizeof(dtype) bytes per element from A and B and into out: the
    binding rejects any dtype / shape / device / layout mismatch before the library is reached
    (a float32 tensor passed to tprod_f64_host was a host over-read / overflow)."""
    import torch
    import paper_1806_07247_b200 as T
    A32 = T.matlab_empty(4, 3, 5, torch.float32, "cpu").zero_()
    B32 = T.matlab_empty(3, 2, 5, torch.float32, "cpu").zero_()
    with pytest.raises(TypeError):
        T.tprod_f64_host(A32, B32)
    with pytest.raises(TypeError):
        T.tprod_f32_host(A32.double(), B32.double())
    with pytest.raises(TypeError):
        T.tprod_f32_host(A32, B32.double())
    with pytest.raises(ValueError):                    # wrong shape
        T.tprod_f32_host(A32, B32, out=T.matlab_empty(4, 3, 5, torch.float32, "cpu"))
    with pytest.raises(ValueError):                    # wrong dtype
        T.tprod_f32_host(A32, B32, out=T.matlab_empty(4, 2, 5, torch.float64, "cpu"))
    with pytest.raises(ValueError):                    # not the Matlab layout
        T.tprod_f32_host(A32, B32, out=torch.empty((4, 2, 5), dtype=torch.float32))
    with pytest.raises(ValueError):                    # shape mismatch of the operands
        T.tprod_f32_host(A32, T.matlab_empty(4, 2, 5, torch.float32, "cpu"))
