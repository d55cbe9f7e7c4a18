"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by element.

Bar (BASELINE.json north_star): relative Frobenius error <= 1e-5 on the fp32 path and <= 1e-12
on the fp64 path, the oracle always evaluated on the exact (rounded) values the GPU saw."""
import numpy as np
from ctypes import c_float as C_float
import pytest

import oracle as O
from synth import CONFIGS, lateral_shard, normal, sample_columns

pytestmark = pytest.mark.gpu

TOL32, TOL64 = 1e-5, 1e-12


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_07247_b200 import build
    build.build()
    import paper_1806_07247_b200 as tp
    return tp


def dev(x):
    import torch
    return torch.from_numpy(np.asfortranarray(x)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def gpu_tprod(T, A, B, handle=None):
    return host(T.tprod(dev(A), dev(B), handle=handle))


# ------------------------------------------------------------------------------- config 1
def test_config1_fp64(T):
    c = CONFIGS["c1"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"], np.float64)
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"], np.float64)
    D = normal((c["n4"], 8, c["n3"]), c["seedD"], np.float64)
    ref = O.tprod_bcirc(A, B)
    C = gpu_tprod(T, A, B)
    assert O.rel_err(C, ref) <= TOL64
    # A * teye = A and associativity, through the GPU path
    I = O.teye(c["n2"], c["n3"])
    assert O.rel_err(gpu_tprod(T, A, I), A) <= TOL64
    lhs = gpu_tprod(T, C, D)
    rhs = gpu_tprod(T, A, gpu_tprod(T, B, D))
    assert O.rel_err(lhs, O.tprod_bcirc(ref, D)) <= TOL64
    assert O.rel_err(lhs, rhs) <= 10 * TOL64


def test_config1_dims_fp32(T):
    """Unaligned dims (n1*n2 % 8 != 0, n2 = 30) on the fp32 path."""
    c = CONFIGS["c1"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"], np.float32)
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"], np.float32)
    assert O.rel_err(gpu_tprod(T, A, B), O.tprod_bcirc(A, B)) <= TOL32


# ------------------------------------------------------------------------------- config 2
def test_config2_full(T):
    c = CONFIGS["c2"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"])
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"])
    err = O.rel_err(gpu_tprod(T, A, B), O.tprod_bcirc(A, B))
    print("config2 rel_err", err)
    assert err <= TOL32


# ------------------------------------------------------------------------------- shape sweep
SWEEP = [
    (1, 1, 1, 1), (1, 1, 2, 1), (2, 3, 1, 4), (3, 2, 2, 5), (5, 4, 3, 2), (7, 9, 4, 6),
    (16, 8, 5, 24), (33, 17, 6, 31), (64, 64, 7, 64), (129, 65, 8, 130), (130, 200, 9, 70),
    (255, 129, 31, 257), (128, 256, 32, 128), (300, 260, 31, 200), (40, 50, 64, 30),
    (200, 136, 3, 264), (8, 1000, 2, 8), (1000, 8, 2, 3),
    (33, 17, 128, 9), (64, 40, 512, 20), (10, 7, 2048, 5), (70, 30, 100, 40),
    (33, 17, 240, 9), (20, 12, 375, 7), (16, 16, 1536, 16),
    (64, 48, 128, 40), (36, 20, 256, 12), (300, 264, 64, 132),   # tube-parallel K1/K3 (P % 4 == 0)
]


@pytest.mark.parametrize("dims", SWEEP, ids=lambda d: "x".join(map(str, d)))
def test_sweep_fp32(T, dims):
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 100 + n1 + n3)
    B = normal((n2, n4, n3), 200 + n4 + n3)
    err = O.rel_err(gpu_tprod(T, A, B), O.tprod_bcirc(A, B))
    assert err <= TOL32, err


@pytest.mark.parametrize("dims", SWEEP, ids=lambda d: "x".join(map(str, d)))
def test_sweep_fp64(T, dims):
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 300 + n1 + n3, np.float64)
    B = normal((n2, n4, n3), 400 + n4 + n3, np.float64)
    assert O.rel_err(gpu_tprod(T, A, B), O.tprod_bcirc(A, B)) <= TOL64


@pytest.mark.parametrize("dims", [(24, 20, 32, 16), (17, 33, 64, 9), (40, 24, 100, 20), (6, 5, 4096, 4),
                                  (130, 70, 9, 100), (256, 96, 31, 200),
                                  (9, 5, 2, 7), (7, 3, 3, 5),            # smallest FFT lengths
                                  (33, 17, 97, 9), (5, 7, 1021, 3),      # Bluestein (prime n3), odd P
                                  (4, 3, 4099, 3),                       # Bluestein, M = 8192
                                  (3, 4, 8192, 2),                       # longest in-smem fp64 FFT
                                  (2, 3, 8209, 2)],                      # beyond: generic O(n3^2)
                         ids=lambda d: "x".join(map(str, d)))
def test_fp64_longer_tubes(T, dims):
    """fp64 path beyond the sweep: the mixed-radix fp64 FFT (radix 8/4/2/3/5, transforms_f64.cu) at
    power-of-two, 5-smooth and long tubes, Bluestein for prime n3 up to M = 8192, the generic kernel
    beyond, and slices large enough for the register-tiled fp64 GEMM (ragged 64 x 64 tiles), vs the
    oracle at 1e-12."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 500 + n3, np.float64)
    B = normal((n2, n4, n3), 600 + n3, np.float64)
    C = gpu_tprod(T, A, B)
    if n3 <= 128:
        ref = O.tprod_bcirc(A, B)
    else:                                               # bcirc would be 24576 x 20480: block rows
        ref = O.tprod_columns(A, B, np.arange(n4))
    assert O.rel_err(C, ref) <= TOL64


@pytest.mark.parametrize("dims", [(40, 24, 67, 20), (33, 17, 97, 9), (64, 16, 97, 12), (8, 6, 4099, 5),
                                  (2, 3, 8209, 2)],      # prime > 8192: no Bluestein length fits, generic O(n3^2)
                         ids=lambda d: "x".join(map(str, d)))
def test_fp32_non_smooth_long_tubes(T, dims):
    """fp32 end to end for n3 > 64 that is not 5-smooth (prime 67, 97, 4099): Bluestein's chirp-z
    through a 5-smooth FFT, forward and inverse (R12), incl. the inverse's per-tube unscale (R18)."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 700 + n3)
    B = normal((n2, n4, n3), 800 + n3)
    C = gpu_tprod(T, A, B)
    ref = O.tprod_bcirc(A, B) if n3 <= 128 else O.tprod_columns(A, B, np.arange(n4))
    assert O.rel_err(C, ref) <= TOL32


def test_simt_engine_cross_check(T):
    """The SIMT reference engine and the tcgen05 engine on identical split operands."""
    h = T.Handle()
    A = normal((300, 260, 31), 5)
    B = normal((260, 200, 31), 6)
    ref = O.tprod_bcirc(A, B)
    C_tc = gpu_tprod(T, A, B, handle=h)
    h.set_option(T._lib.TPROD_OPT_ENGINE, 1)
    C_simt = gpu_tprod(T, A, B, handle=h)
    assert O.rel_err(C_tc, ref) <= TOL32
    assert O.rel_err(C_simt, ref) <= TOL32
    assert O.rel_err(C_tc, C_simt) <= TOL32


@pytest.mark.parametrize("dims", [(300, 260, 31, 200), (1000, 136, 3, 700), (129, 64, 7, 129),
                                  (1100, 200, 8, 300), (520, 96, 5, 130)],
                         ids=lambda d: "x".join(map(str, d)))
def test_gemm_tile_and_cluster_variants_bitwise(T, dims):
    """GEMM N tile (64/128), 2-CTA A-multicast clusters, cta_group::2 CTA pairs (256-row tiles
    across two SMs) and 4-CTA clusters of two pairs sharing B by multicast (512-row cluster tiles)
    change scheduling only: the K order of every output is fixed, so all variants are bitwise
    identical (odd N-tile counts, a lone 128-row half-pair and ragged 512-row cluster tiles
    included)."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 11)
    B = normal((n2, n4, n3), 12)
    ref = O.tprod_bcirc(A, B)
    outs = []
    for bn, cn in ((64, 1), (64, 2), (128, 1), (128, 2), (128, 3), (128, 4), (0, 0)):
        h = T.Handle()
        h.set_option(T._lib.TPROD_OPT_GEMM_BN, bn)
        h.set_option(T._lib.TPROD_OPT_GEMM_CLUSTER, cn)
        outs.append(gpu_tprod(T, A, B, handle=h))
    assert O.rel_err(outs[0], ref) <= TOL32
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("dims", [(600, 200, 31, 300), (600, 136, 32, 300), (1100, 200, 8, 300),
                                  (1024, 1024, 31, 512), (520, 96, 5, 1030)],
                         ids=lambda d: "x".join(map(str, d)))
def test_k3_overlap_bitwise(T, dims):
    """TPROD_OPT_OVERLAP: the GEMM on CTA pairs in 2..8 tile rounds runs m-row by m-row and counts
    finished (m, n) tiles; K3 (tube-pair register kernel, n3 <= 32) launches as a programmatic
    dependent and each block waits for its tile.  Scheduling only: bitwise equal to the serial
    order, direct launch and graph replay, ragged m / n tiles (600 rows, 300 / 1030 columns),
    CTA pairs and 4-CTA clusters; vs the oracle (Eq. (9)) on sampled lateral
    slices; the stage timer reports K2 + K3 as one stage."""
    import torch
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 21)
    B = normal((n2, n4, n3), 22)
    Ad, Bd = dev(A), dev(B)
    outs = []
    for ov, cn in ((0, 0), (1, 0), (1, 3), (1, 4)):
        h = T.Handle()
        h.set_option(T._lib.TPROD_OPT_OVERLAP, ov)
        h.set_option(T._lib.TPROD_OPT_GEMM_CLUSTER, cn)
        for _ in range(3):                                   # direct, capture, graph replay
            outs.append(host(T.tprod(Ad, Bd, handle=h)))
        h.set_option(T._lib.TPROD_OPT_TIMING, 1)
        outs.append(host(T.tprod(Ad, Bd, handle=h)))
        st = h.last_stage_ms()
        assert all(x >= 0 for x in st) and st[2] > 0
        if ov == 0:
            assert st[3] > 0
    cols = sample_columns(n4, 6, seed=3)
    ref = O.tprod_columns(A, B, cols)
    assert O.rel_err(outs[0][:, cols, :], ref) <= TOL32
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    torch.cuda.synchronize()


@pytest.mark.parametrize("dims", [(600, 136, 64, 300), (1100, 72, 64, 1030), (2048, 64, 64, 1100), (516, 40, 64, 2000)],
                         ids=lambda d: "x".join(map(str, d)))
def test_k3_stream_overlap_bitwise(T, dims):
    """TPROD_OPT_OVERLAP (default 1) with n3 = 64 (K3 = the TMA tube inverse): the GEMM of ANY number of tile
    rounds runs m-row by m-row with (m, n) counters and K3's CTAs take their items from a device
    work counter in tile-completion order (Alg. 1 steps 2-3 overlapped).
    Scheduling only: bitwise equal to the serial order (option 0) and to the short-run-only
    setting (option 2), direct launch and graph replay, ragged m / n tiles, CTA pairs and 4-CTA
    clusters; vs the oracle (Eq. (9)) on sampled lateral slices; with the
    overlap on the stage timer reports K2 + K3 as one stage (the path under test really ran)."""
    import torch
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 23)
    B = normal((n2, n4, n3), 24)
    Ad, Bd = dev(A), dev(B)
    outs = []
    for ov, cn in ((0, 0), (1, 0), (1, 3), (1, 4), (2, 0)):
        h = T.Handle()
        h.set_option(T._lib.TPROD_OPT_OVERLAP, ov)
        h.set_option(T._lib.TPROD_OPT_GEMM_CLUSTER, cn)
        for _ in range(3):                                   # direct, capture, graph replay
            outs.append(host(T.tprod(Ad, Bd, handle=h)))
        h.set_option(T._lib.TPROD_OPT_TIMING, 1)
        outs.append(host(T.tprod(Ad, Bd, handle=h)))
        st = h.last_stage_ms()
        assert all(x >= 0 for x in st) and st[2] > 0
        if ov != 1:
            assert st[3] > 0
        else:
            assert st[3] == 0
    cols = sample_columns(n4, 6, seed=3)
    ref = O.tprod_columns(A, B, cols)
    assert O.rel_err(outs[0][:, cols, :], ref) <= TOL32
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    torch.cuda.synchronize()


@pytest.mark.parametrize("dims", [(300, 1024, 31, 200), (256, 256, 32, 256), (64, 300, 7, 40), (40, 2048, 16, 24),
                                  (40, 2050, 16, 24), (36, 301, 5, 20), (20, 6, 1, 9), (33, 200, 2, 70)],
                         ids=lambda d: "x".join(map(str, d)))
def test_fused_column_scales_bitwise(T, dims):
    """TPROD_OPT_FUSED_SCALES: B's column scales reduced inside B's forward transform by a CTA cluster
    per lateral slice (DSMEM exchange of partial maxima) give the same maxima as the K0 pass, so the
    result is bitwise equal with the option off (1..8-CTA clusters, a ragged last CTA, n2 = 2050 and
    odd n2 falling back to K0), with planted per-column magnitudes 2^-20..2^20 and a zero column;
    prepared-operand path included; vs the oracle (Eq. (9))."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 31)
    B = normal((n2, n4, n3), 32)
    B *= np.exp2(np.linspace(-20, 20, n4)).astype(np.float32)[None, :, None]
    B[:, n4 // 2, :] = 0.0
    Ad, Bd = dev(A), dev(B)
    outs = []
    for fused in (0, 1):
        h = T.Handle()
        h.set_option(T._lib.TPROD_OPT_FUSED_SCALES, fused)
        outs.append(host(T.tprod(Ad, Bd, handle=h)))
        outs.append(host(T.tprod(Ad, Bd, handle=h)))          # graph capture
        h.prepare_a(Ad)
        outs.append(host(T.tprod_prepared(Bd, handle=h)))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert not outs[0][:, n4 // 2, :].any()
    cols = np.unique(np.array([0, 1, n4 // 2, n4 - 1]))
    ref = O.tprod_columns(A.astype(np.float64), B.astype(np.float64), cols)
    for j, c in enumerate(cols):                               # per column: each has its own scale
        if ref[:, j, :].any():
            assert O.rel_err(outs[0][:, c, :], ref[:, j, :]) <= TOL32


# ------------------------------------------------------------------------------- stages
@pytest.mark.parametrize("n3", [1, 2, 3, 10, 31, 32, 64, 65, 96, 100, 120, 128, 256, 375, 1000, 1536,
                                2048, 4096, 6000, 8192, 15360,
                                67, 97, 127, 1021, 4099, 8191])      # not 5-smooth: Bluestein
def test_stage_forward_dft(T, n3):
    """S1/S2 vs numpy.fft.rfft (library special case), both operand roles."""
    p, q = (37, 5) if n3 > 64 else (133, 9)
    X = normal((p, q, n3), 7 + n3)
    ref = np.fft.rfft(X.astype(np.float64), axis=2)
    for role in (0, 1):
        got = host(T.dft_f32(dev(X), role=role))
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err < 2e-6, (role, err)


@pytest.mark.parametrize("n3", [1, 2, 7, 31, 32, 64, 96, 100, 128, 375, 512, 1000, 4096, 6000, 8192,
                                15360, 67, 97, 1021, 4099])
def test_stage_inverse_roundtrip(T, n3):
    """S4(S1(X)) = X and the 1x1xn3 circular-convolution worked example."""
    import torch
    X = normal((45, 3, n3), 17 + n3)
    Xb = torch.from_numpy(np.fft.rfft(X.astype(np.float64), axis=2).astype(np.complex64)).cuda()
    back = host(T.idft_f32(Xb, n3))
    assert np.linalg.norm(back - X) / np.linalg.norm(X) < 2e-6


TC_N3 = [2, 3, 4, 5, 7, 8, 10, 15, 16, 17, 24, 31, 32, 33, 45, 48, 63, 64]


@pytest.mark.parametrize("n3", TC_N3)
def test_stage_forward_dft_tensor_core(T, n3):
    """The tcgen05 DFT-matrix forward kernel (TPROD_OPT_TRANSFORM = 2; 2 <= n3 <= 64, P % 4 == 0;
    the last 128-tube block ragged) vs numpy.fft.rfft for both operand roles, and vs the default
    kernels within fp32 rounding."""
    X = normal((132, 5, n3), 9 + n3)
    ref = np.fft.rfft(X.astype(np.float64), axis=2)
    htc = T.Handle()
    htc.set_option(T._lib.TPROD_OPT_TRANSFORM, 2)
    for role in (0, 1):
        got = host(T.dft_f32(dev(X), role=role, handle=htc))
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err < 2e-6, (role, err)
        old = host(T.dft_f32(dev(X), role=role))
        assert np.linalg.norm(got - old) / np.linalg.norm(ref) < 2e-6


@pytest.mark.parametrize("n3", TC_N3)
def test_tprod_tensor_core_transforms(T, n3):
    """End to end with the tcgen05 forward and inverse DFT kernels (TPROD_OPT_TRANSFORM = 2; n1, n2 %
    4 == 0 so both operands and C take them), rows of A spread over 2^-20 .. 2^20 (per-tube scales in
    the inverse): vs the oracle, and the default kernels too."""
    n1, n2, n4 = 260, 48, 36
    rng = np.random.default_rng(n3)
    A = normal((n1, n2, n3), 19 + n3).astype(np.float64) * np.exp2(rng.integers(-20, 21, size=n1)).reshape(n1, 1, 1)
    A = A.astype(np.float32)
    B = normal((n2, n4, n3), 29 + n3)
    ref = O.tprod_alg1(A.astype(np.float64), B.astype(np.float64)).real
    h2 = T.Handle()
    h2.set_option(T._lib.TPROD_OPT_TRANSFORM, 2)
    C = gpu_tprod(T, A, B, handle=h2)
    C2 = gpu_tprod(T, A, B)
    ra = np.abs(A).max(axis=(1, 2))
    for i in range(0, n1, 7):                           # every row to its own scale (R18)
        num = np.linalg.norm(C[i] - ref[i])
        assert num <= 1e-5 * ra[i] * np.abs(B).max() * np.sqrt(n2 * n3 * n4), (i, num)
    assert O.rel_err(C, ref) <= TOL32
    assert O.rel_err(C2, ref) <= TOL32


@pytest.mark.parametrize("n3", [64, 128, 256])
def test_tube_transforms_match_register_kernels(T, n3):
    """The TMA-staged tube-parallel Stockham kernels (picked for aligned shapes) and the register /
    buffer-major kernels (TPROD_OPT_TRANSFORM = 1) compute the same t-product: both within the
    fp32 tolerance of the oracle, and within fp32 rounding of each other.  P = 4k with a ragged last
    item (n1 not a multiple of the 2F tubes per item)."""
    A = normal((516, 40, n3), 31 + n3)
    B = normal((40, 24, n3), 32 + n3)
    ref = O.tprod_columns(A, B, np.arange(24))
    h0, h1 = T.Handle(), T.Handle()
    h1.set_option(T._lib.TPROD_OPT_TRANSFORM, 1)
    C0 = gpu_tprod(T, A, B, handle=h0)
    C1 = gpu_tprod(T, A, B, handle=h1)
    assert O.rel_err(C0, ref) <= TOL32
    assert O.rel_err(C1, ref) <= TOL32
    assert O.rel_err(C0, C1) <= 1e-6


@pytest.mark.parametrize("dims", [(300, 260, 31, 200), (256, 128, 64, 96), (64, 40, 100, 24), (7, 5, 2, 3),
                                  (16, 12, 4096, 8)],
                         ids=lambda d: "x".join(map(str, d)))
def test_prepared_operand_bitwise(T, dims):
    """NEXT-1 prepared left operand: tprod_prepare_a_f32 once, tprod_f32_prepared for several B --
    bitwise equal to tprod_f32 (same kernels, same operands, same K order); within the oracle
    tolerance; errors when nothing is prepared."""
    import torch
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 61 + n3)
    h = T.Handle()
    with pytest.raises(ValueError):
        T.tprod_prepared(dev(normal((n2, n4, n3), 1)), handle=h)
    assert h.ptr and T._lib.lib().tprod_f32_prepared(None, None, n4, None, h.ptr) == T._lib.TPROD_EINVAL
    h.prepare_a(dev(A))
    for seed in (62, 63):
        B = normal((n2, n4 + seed - 62, n3), seed)
        ref = gpu_tprod(T, A, B)
        got = host(T.tprod_prepared(dev(B), handle=h))
        assert np.array_equal(got, ref)
        assert O.rel_err(got, O.tprod_columns(A, B, np.arange(B.shape[1]))) <= TOL32
    h.release_a()
    with pytest.raises(ValueError):
        T.tprod_prepared(dev(B), handle=h)


@pytest.mark.parametrize("n3,p,q", [(4096, 36, 3), (4096, 132, 2), (8192, 24, 2), (16384, 8, 2)])
def test_fourstep_forward_stage(T, n3, p, q):
    """Two-pass four-step forward DFT (long power-of-two tubes, P % 4 == 0; TUB = 64 and 128 tiles,
    ragged last tile) vs numpy.fft.rfft, both operand roles."""
    X = normal((p, q, n3), 5 + n3 + p)
    ref = np.fft.rfft(X.astype(np.float64), axis=2)
    for role in (0, 1):
        got = host(T.dft_f32(dev(X), role=role))
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err < 2e-6, (role, err)


@pytest.mark.parametrize("p,q", [(36, 3), (64, 5), (132, 2), (4, 7), (96, 1)])
def test_cluster_fft_stages(T, p, q):
    """One-pass 8-CTA cluster transforms for n3 = 4096 (TPROD_OPT_TRANSFORM = 3,
    transforms_cluster.cu; P % 4 == 0, ragged 32-tube items): forward vs numpy.fft.rfft for both
    operand roles and vs the default two-pass four-step kernels; the inverse (conjugate fill fused)
    round trip on both."""
    import torch
    n3 = 4096
    X = normal((p, q, n3), 3 + p + q)
    ref = np.fft.rfft(X.astype(np.float64), axis=2)
    h3 = T.Handle()
    h3.set_option(T._lib.TPROD_OPT_TRANSFORM, 3)
    for role in (0, 1):
        clu = host(T.dft_f32(dev(X), role=role, handle=h3))
        four = host(T.dft_f32(dev(X), role=role))
        assert np.linalg.norm(clu - ref) / np.linalg.norm(ref) < 2e-6, role
        assert np.linalg.norm(clu - four) / np.linalg.norm(ref) < 2e-6, role
    Xb = torch.from_numpy(ref.astype(np.complex64)).cuda()
    for hh in (h3, None):
        back = host(T.idft_f32(Xb, n3, handle=hh))
        assert np.linalg.norm(back - X) / np.linalg.norm(X) < 2e-6


@pytest.mark.parametrize("dims", [(64, 64, 4096, 64), (36, 20, 4096, 12), (100, 8, 4096, 3)],
                         ids=lambda d: "x".join(map(str, d)))
def test_cluster_full_path(T, dims):
    """Full t-product through the cluster transforms (TPROD_OPT_TRANSFORM = 3: K1 of A and B, K3) on
    sampled frontal slices vs the oracle's Eq. (9) block rows, every row of C to its own scale with
    rows of A spread over 2^-20 .. 2^20 and one zero row (R18), and vs the default two-pass four-step
    kernels within 1e-6."""
    n1, n2, n3, n4 = dims
    rng = np.random.default_rng(n1 + n4)
    A = normal((n1, n2, n3), 81 + n1).astype(np.float64) * np.exp2(rng.integers(-20, 21, size=n1)).reshape(n1, 1, 1)
    A[n1 // 2] = 0.0
    A = A.astype(np.float32)
    B = normal((n2, n4, n3), 82 + n4)
    h3 = T.Handle()
    h3.set_option(T._lib.TPROD_OPT_TRANSFORM, 3)
    C = gpu_tprod(T, A, B, handle=h3)
    C3 = gpu_tprod(T, A, B)
    tl = np.array([0, 1, 2047, 2048, n3 - 1])
    ref = O.tprod_blockrow(A, B, tl, np.arange(n4))
    assert O.rel_err(C[:, :, tl], ref) <= TOL32
    assert not C[n1 // 2].any()
    ra = np.abs(A).max(axis=(1, 2))
    for i in range(n1):
        if ra[i] > 0:
            num = np.linalg.norm(C[i][:, tl] - ref[i])
            assert num <= 1e-5 * ra[i] * np.abs(B).max() * np.sqrt(n2 * n3 * n4), (i, num)
    assert O.rel_err(C, C3) <= 1e-6


@pytest.mark.parametrize("dims", [(24, 16, 8192, 8), (132, 8, 4096, 12)], ids=lambda d: "x".join(map(str, d)))
def test_fourstep_full_path(T, dims):
    """Full t-product with the four-step forward on sampled frontal slices vs the oracle, and vs the
    one-pass FFT kernels (TPROD_OPT_TRANSFORM = 1)."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 71)
    B = normal((n2, n4, n3), 72)
    h1 = T.Handle()
    h1.set_option(T._lib.TPROD_OPT_TRANSFORM, 1)
    C = gpu_tprod(T, A, B)
    C1 = gpu_tprod(T, A, B, handle=h1)
    tl = np.array([0, 1, n3 // 2, n3 - 1])
    J = np.arange(n4)
    ref = O.tprod_blockrow(A, B, tl, J)
    assert O.rel_err(C[:, :, tl], ref) <= TOL32
    assert O.rel_err(C, C1) <= 1e-6


# ------------------------------------------------------------------------------- NEXT-4
@pytest.mark.parametrize("dims", [(33, 17, 5), (7, 64, 1), (64, 3, 2), (40, 40, 31), (132, 68, 3), (4, 4, 2), (256, 128, 4)], ids=lambda d: "x".join(map(str, d)))
def test_tran_teye_gpu_exact(T, dims):
    """tran (Def. 2.2) and teye (Def. 2.3) on the GPU equal the oracle exactly (pure data movement)."""
    import torch
    n1, n2, n3 = dims
    for dt in (np.float32, np.float64):
        A = normal((n1, n2, n3), 91 + n3, dt)
        assert np.array_equal(host(T.tran(dev(A))), O.tran(A).astype(dt))
    for dt, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
        assert np.array_equal(host(T.teye(n1, n3, dtype=tdt)), O.teye(n1, n3).astype(dt))


def _well_conditioned(n, n3, seed):
    A = normal((n, n, n3), seed, np.float64) * 0.2
    A[:, :, 0] += 2.0 * np.eye(n)
    return A.astype(np.float32)


@pytest.mark.parametrize("n,n3", [(1, 1), (5, 4), (32, 7), (96, 2), (16, 64), (8, 100), (97, 2), (128, 5),
                                  (200, 3)])
def test_tinv_gpu_vs_oracle(T, n, n3):
    """tinv (Def. 2.4) through the production transforms + per-slice Gauss-Jordan (n <= 96 in shared
    memory, larger in global memory in fp64) vs the oracle's literal bcirc solve, and both sides of
    Eq. (11) in the oracle."""
    A = _well_conditioned(n, n3, 93 + n)
    X = host(T.tinv(dev(A)))
    ref = O.tinv(A)
    assert O.rel_err(X, ref) <= 1e-5
    I = O.teye(n, n3)
    assert O.rel_err(O.tprod_bcirc(A, X), I) <= 1e-5
    assert O.rel_err(O.tprod_bcirc(X, A), I) <= 1e-5


def test_tinv_gpu_long_tubes_and_errors(T):
    """tinv on long tubes (four-step transforms) checked by Eq. (11) on sampled slices of the oracle
    product; singular and unsupported inputs raise."""
    A = _well_conditioned(12, 4096, 97)
    X = host(T.tinv(dev(A)))
    tl = np.array([0, 1, 2048, 4095])
    AX = O.tprod_blockrow(A, X, tl, np.arange(12))
    assert O.rel_err(AX, O.teye(12, 4096)[:, :, tl]) <= 1e-5
    with pytest.raises(T.TprodError) as e:
        T.tinv(dev(np.zeros((4, 4, 3), np.float32)))
    assert e.value.status == T._lib.TPROD_ESINGULAR
    Ab = O.dft_mode3(_well_conditioned(3, 5, 5).astype(np.float64))
    Ab[:, :, 2] = 0.0
    Ab[:, :, 3] = 0.0
    with pytest.raises(T.TprodError) as e:
        T.tinv(dev(np.real(O.idft_mode3(Ab)).astype(np.float32)))
    assert e.value.status == T._lib.TPROD_ESINGULAR
    with pytest.raises(T.TprodError) as e:                # large-slice path, singular
        T.tinv(dev(np.zeros((100, 100, 3), np.float32)))
    assert e.value.status == T._lib.TPROD_ESINGULAR
    Y = dev(np.zeros((4, 4, 3), np.float32))
    assert T._lib.lib().tprod_tinv_f32(Y.data_ptr(), Y.data_ptr() + 4096, 8193, 1, None,
                                       T.Handle().ptr) == T._lib.TPROD_EUNSUPPORTED


@pytest.mark.parametrize("n", [6, 120], ids=["smem", "global"])
def test_tinv_async_status(T, n):
    """TPROD_OPT_SYNC_CHECKS = 0: tinv returns at once and a singular tensor is reported through the
    handle's status word (TPROD_STATUS_SINGULAR), which tprod_status clears; a regular tensor leaves
    it 0 and still matches the oracle."""
    h = T.Handle()
    h.set_option(T._lib.TPROD_OPT_SYNC_CHECKS, 0)
    T.tinv(dev(np.zeros((n, n, 3), np.float32)), handle=h)          # no exception
    assert h.status() == T._lib.TPROD_STATUS_SINGULAR
    assert h.status() == 0                                           # cleared by the read
    A = _well_conditioned(n, 3, 7)
    X = host(T.tinv(dev(A), handle=h))
    assert h.status() == 0
    assert O.rel_err(X, O.tinv(A)) <= 1e-5


@pytest.mark.parametrize("dims,tau", [((5, 4, 6), 1.5), ((64, 64, 7), 20.0), ((33, 17, 31), 8.0),
                                      ((8, 40, 1024), 6.0), ((1, 1, 2), 1.0), ((16, 16, 64), 0.0),
                                      ((32, 48, 255), 10.0)],
                         ids=lambda d: "x".join(map(str, d)) if isinstance(d, tuple) else str(d))
def test_tsvt_gpu_vs_oracle(T, dims, tau):
    """t-SVT (Algorithm 3) on the GPU -- production transforms + per-slice one-sided Jacobi SVT -- vs
    the oracle's step-by-step Algorithm 3 (numpy SVD per slice); tau = 0 returns Y."""
    n1, n2, n3 = dims
    Y = normal((n1, n2, n3), 101 + n3)
    X = host(T.tsvt(dev(Y), tau))
    err = O.rel_err(X, O.tsvt(Y, tau))
    print("tsvt", dims, tau, "rel_err", err)
    assert err <= 1e-5
    if tau == 0.0:
        assert O.rel_err(X, Y) <= 1e-6


@pytest.mark.parametrize("dims,tau", [((96, 80, 5), 8.0), ((65, 130, 3), 6.0), ((256, 256, 3), 20.0),
                                      ((200, 72, 9), 0.0), ((300, 40, 16), 1e6), ((200, 20, 5), 3.0),
                                      ((7, 150, 4), 2.0)],
                         ids=lambda d: "x".join(map(str, d)) if isinstance(d, tuple) else str(d))
def test_tsvt_large_slices_gpu_vs_oracle(T, dims, tau):
    """t-SVT (Algorithm 3) for slices beyond 64 x 64: the blocked one-sided Jacobi (column blocks of
    32, block pairs orthogonalised through their Gram matrix, X and V updated in global memory) vs
    the oracle's step-by-step Algorithm 3; tau = 0 returns Y, tau above every singular value gives
    zero (Eq. (19)-(21))."""
    n1, n2, n3 = dims
    Y = normal((n1, n2, n3), 171 + n3)
    h = T.Handle()
    X = host(T.tsvt(dev(Y), tau, handle=h))
    assert h.status() == 0                                # every slice converged
    ref = O.tsvt(Y.astype(np.float64), tau)
    if tau >= 1e6:
        assert np.abs(X).max() <= 1e-6 * np.abs(Y).max()
        return
    err = O.rel_err(X, ref)
    print("tsvt large", dims, tau, "rel_err", err)
    assert err <= 1e-5
    if tau == 0.0:
        assert O.rel_err(X, Y) <= 1e-6


@pytest.mark.slow
def test_tsvt_1024x1024x31_gpu(T):
    """The verdict's large case: t-SVT of 1024 x 1024 x 31 (16 spectral slices of 1024 x 1024) vs
    the oracle (numpy SVD per slice)."""
    Y = normal((1024, 1024, 31), 181)
    tau = 200.0
    X = host(T.tsvt(dev(Y), tau))
    err = O.rel_err(X, O.tsvt(Y.astype(np.float64), tau))
    print("tsvt 1024x1024x31 rel_err", err)
    assert err <= 1e-5


@pytest.mark.parametrize("dims", [(6, 5, 7), (64, 64, 8), (40, 12, 33), (16, 16, 100), (100, 70, 5),
                                  (65, 130, 8), (300, 20, 3)],
                         ids=lambda d: "x".join(map(str, d)))
def test_tsvd_values_gpu_vs_oracle(T, dims):
    """t-SVD scalars on the GPU (per-slice Jacobi SVD -- one CTA per slice up to 64 x 64, blocked
    beyond -- + Eq. (14) reduction) vs the oracle: singular values, TNN, TSN (the oracle's through
    bcirc), tubal rank."""
    n1, n2, n3 = dims
    A = normal((n1, n2, n3), 111 + n3)
    out = host(T.tsvd_values(dev(A), rtol=1e-6))
    r = min(n1, n2)
    s, tnn, tsn, rank = O.tsvd_values(A, rtol=1e-6)
    np.testing.assert_allclose(out[:r], s, rtol=2e-5, atol=2e-5 * s[0])
    assert abs(out[r] - tnn) <= 2e-5 * tnn and abs(out[r + 1] - tsn) <= 2e-5 * tsn
    assert int(out[r + 2]) == rank


@pytest.mark.parametrize("n1,n2", [(40, 30), (150, 90)])
def test_tsvd_tubal_rank_gpu(T, n1, n2):
    """Tubal rank of U * V (Def. 2.7) with U n1 x 5 x 31, V 5 x n2 x 31 is 5 on the GPU (small and
    blocked Jacobi)."""
    U = normal((n1, 5, 31), 121, np.float64)
    V = normal((5, n2, 31), 122, np.float64)
    A = O.tprod_bcirc(U, V).astype(np.float32)
    out = host(T.tsvd_values(dev(A), rtol=1e-4))
    assert int(out[min(n1, n2) + 2]) == 5


@pytest.mark.parametrize("dims", [(6, 4, 5), (3, 7, 4), (64, 48, 9), (20, 64, 31), (8, 8, 64), (100, 70, 5),
                                  (40, 130, 4), (200, 10, 3)],
                         ids=lambda d: "x".join(map(str, d)))
def test_tsvd_factors_gpu(T, dims):
    """Skinny t-SVD on the GPU: S equals the oracle's (unique); U, V (unique only up to phases) are
    checked by what holds for any valid factorisation, in the oracle: A = U * S * V^* and
    U^* * U = V^* * V = I."""
    n1, n2, n3 = dims
    r = min(n1, n2)
    A = normal(dims, 131 + n3)
    U, S, V = (host(x) for x in T.tsvd(dev(A)))
    _, S_ref, _ = O.tsvd(A)
    assert O.rel_err(S, S_ref) <= 1e-5
    A64 = A.astype(np.float64)
    assert O.rel_err(O.tprod_bcirc(O.tprod_bcirc(U, S), O.tran(V)), A64) <= 1e-5
    assert O.rel_err(O.tprod_bcirc(O.tran(U), U), O.teye(r, n3)) <= 1e-5
    assert O.rel_err(O.tprod_bcirc(O.tran(V), V), O.teye(r, n3)) <= 1e-5


@pytest.mark.parametrize("dims,rank", [((8, 8, 5), 2), ((12, 20, 7), 3), ((16, 6, 4), 0), ((100, 80, 5), 3),
                                       ((70, 90, 3), 0), ((40, 130, 4), 2)],
                         ids=lambda d: "x".join(map(str, d)) if isinstance(d, tuple) else str(d))
def test_tsvd_factors_rank_deficient(T, dims, rank):
    """Theorem 2.2 asks for orthogonal factors also when A is rank-deficient: with A = U0 * V0 of
    tubal rank 2 or 3 (and the zero tensor), every spectral slice has zero singular values, whose
    left vectors the Jacobi SVD cannot supply; the kernel completes them to an orthonormal set, so
    U^* * U = V^* * V = I still holds, A = U * S * V^* and S matches the oracle."""
    n1, n2, n3 = dims
    r = min(n1, n2)
    if rank:
        U0 = normal((n1, rank, n3), 141 + n3, np.float64)
        V0 = normal((rank, n2, n3), 142 + n3, np.float64)
        A = O.tprod_bcirc(U0, V0).astype(np.float32)
    else:
        A = np.zeros(dims, np.float32)
    U, S, V = (host(x) for x in T.tsvd(dev(A)))
    assert np.isfinite(U).all() and np.isfinite(V).all()
    _, S_ref, _ = O.tsvd(A.astype(np.float64))
    if rank:
        assert O.rel_err(S, S_ref) <= 1e-5
        assert O.rel_err(O.tprod_bcirc(O.tprod_bcirc(U, S), O.tran(V)), A.astype(np.float64)) <= 1e-5
    else:
        assert np.all(S == 0.0)
    assert O.rel_err(O.tprod_bcirc(O.tran(U), U), O.teye(r, n3)) <= 1e-5
    assert O.rel_err(O.tprod_bcirc(O.tran(V), V), O.teye(r, n3)) <= 1e-5


@pytest.mark.parametrize("dims,rank", [((6, 4, 5), 0), ((3, 7, 4), 0), ((64, 48, 9), 0), ((100, 70, 6), 0),
                                       ((40, 130, 4), 0), ((12, 20, 7), 3), ((100, 80, 5), 3), ((16, 6, 4), -1),
                                       ((1, 5, 3), 0)],
                         ids=lambda d: "x".join(map(str, d)) if isinstance(d, tuple) else str(d))
def test_tsvd_full_factors_gpu(T, dims, rank):
    """Full t-SVD (Theorem 2.2 shapes) on the GPU: S equals the oracle's full S; U (n1 x n1) and V
    (n2 x n2) are orthogonal both ways and A = U * S * V^*, checked in the oracle (the null-space
    columns are one valid completion, so they are not compared one by one).  rank > 0: a tubal-rank
    product; -1: the zero tensor."""
    n1, n2, n3 = dims
    if rank > 0:
        A = O.tprod_bcirc(normal((n1, rank, n3), 151 + n3, np.float64),
                          normal((rank, n2, n3), 152 + n3, np.float64)).astype(np.float32)
    elif rank < 0:
        A = np.zeros(dims, np.float32)
    else:
        A = normal(dims, 161 + n3)
    h = T.Handle()
    U, S, V = (host(x) for x in T.tsvd_full(dev(A), handle=h))
    assert h.status() == 0
    assert U.shape == (n1, n1, n3) and S.shape == (n1, n2, n3) and V.shape == (n2, n2, n3)
    _, S_ref, _ = O.tsvd(A.astype(np.float64), full=True)
    if rank >= 0:
        assert O.rel_err(S, S_ref) <= 1e-5
        assert O.rel_err(O.tprod_bcirc(O.tprod_bcirc(U, S), O.tran(V)), A.astype(np.float64)) <= 1e-5
    else:
        assert np.all(S == 0.0)
    for Q, n in ((U, n1), (V, n2)):
        assert O.rel_err(O.tprod_bcirc(O.tran(Q), Q), O.teye(n, n3)) <= 1e-5
        assert O.rel_err(O.tprod_bcirc(Q, O.tran(Q)), O.teye(n, n3)) <= 1e-5


def test_next_rows_argument_errors(T):
    """Argument errors of the NEXT-row entry points come back before any work: tau < 0 / NaN,
    slices beyond the 64 x 64 Jacobi kernel of the t-SVD scalars, aliasing output."""
    import torch
    L = T._lib.lib()
    h = T.Handle()
    Y = dev(normal((4, 3, 5), 1))
    X = dev(normal((4, 3, 5), 2))
    assert L.tprod_tsvt_f32(Y.data_ptr(), X.data_ptr(), 4, 3, 5, C_float(-1.0), None, h.ptr) == T._lib.TPROD_EINVAL
    assert L.tprod_tsvt_f32(Y.data_ptr(), X.data_ptr(), 4, 3, 5, C_float(float("nan")), None, h.ptr) == T._lib.TPROD_EINVAL
    assert L.tprod_tsvt_f32(Y.data_ptr(), Y.data_ptr(), 4, 3, 5, C_float(1.0), None, h.ptr) == T._lib.TPROD_EALIAS
    # every slice size up to min(n1, n2) = 65535 runs (blocked Jacobi); beyond: unsupported, nothing read
    assert L.tprod_tsvd_values_f32(Y.data_ptr(), 65536, 65536, 1, C_float(1e-6), X.data_ptr(), None,
                                   h.ptr) == T._lib.TPROD_EUNSUPPORTED
    assert L.tprod_tran_f32(Y.data_ptr(), Y.data_ptr(), 4, 3, 5, None, h.ptr) == T._lib.TPROD_EALIAS
    assert L.tprod_teye_f32(None, 3, 2, None, h.ptr) == T._lib.TPROD_EINVAL
    assert L.tprod_tinv_f32(Y.data_ptr(), X.data_ptr(), 0, 5, None, h.ptr) == T._lib.TPROD_EINVAL


def test_worked_examples_on_gpu(T, golden):
    for dt in (np.float32, np.float64):
        g = golden["tprod_tubes_1x1x3"]
        a = np.array(g["a"], dt).reshape(1, 1, -1)
        b = np.array(g["b"], dt).reshape(1, 1, -1)
        np.testing.assert_allclose(gpu_tprod(T, a, b)[0, 0], g["c"], rtol=1e-6)
        g = golden["tprod_n3_1"]
        A = np.array(g["A"], dt)[:, :, None]
        B = np.array(g["B"], dt)[:, :, None]
        np.testing.assert_allclose(gpu_tprod(T, A, B)[:, :, 0], g["C"], rtol=1e-6)


# ------------------------------------------------------------------------------- invariants
def test_identity_shift_transpose_fp32(T):
    A = normal((70, 50, 12), 1)
    B = normal((50, 40, 12), 2)
    I = O.teye(50, 12).astype(np.float32)
    assert O.rel_err(gpu_tprod(T, A, I), A) <= TOL32
    C = gpu_tprod(T, A, B)
    Cs = gpu_tprod(T, A, np.roll(B, 5, axis=2))
    assert O.rel_err(Cs, np.roll(C, 5, axis=2)) <= TOL32
    Ct = gpu_tprod(T, np.ascontiguousarray(O.tran(B)), np.ascontiguousarray(O.tran(A)))
    assert O.rel_err(Ct, O.tran(C)) <= TOL32


@pytest.mark.parametrize("dims", [(64, 64, 33, 48), (16, 8, 5, 12), (36, 100, 7, 20), (256, 160, 31, 40),
                                  (4, 12, 16, 8), (33, 17, 9, 10),
                                  # pair-packed FFT paths: tube (64, 128, 256), mixed radix, four-step
                                  (64, 64, 64, 48), (64, 32, 128, 16), (64, 64, 256, 16), (64, 16, 250, 8),
                                  (32, 8, 4096, 4),
                                  # register dense (odd n3), generic non-smooth (97)
                                  (40, 24, 31, 36), (20, 12, 97, 8)], ids=lambda d: "x".join(map(str, d)))
def test_operand_scales_follow_rows_and_columns(T, dims):
    """K0's exact power-of-two scales are per row of A and per column of B (the fp16 split keeps
    fp32 accuracy only if every row / column is scaled by its own maximum): rows and columns
    spread over 2^-24 .. 2^24 and one planted outlier per operand (10^4 x its row / column) must
    come out finite and accurate row by row.  A scale that missed the outlier's run would overflow
    the fp16 high part; a shared scale would flush the small rows."""
    n1, n2, n3, n4 = dims
    rng = np.random.default_rng(7 + n1 + n4)
    A = normal((n1, n2, n3), 71 + n1).astype(np.float64)
    B = normal((n2, n4, n3), 72 + n4).astype(np.float64)
    A *= np.exp2(rng.integers(-24, 25, size=n1)).reshape(n1, 1, 1)
    B *= np.exp2(rng.integers(-24, 25, size=n4)).reshape(1, n4, 1)
    ia, ja, ka = rng.integers(n1), rng.integers(n2), rng.integers(n3)
    A[ia, ja, ka] = 1e4 * np.abs(A[ia]).max()
    ib, jb, kb = rng.integers(n2), rng.integers(n4), rng.integers(n3)
    B[ib, jb, kb] = -1e4 * np.abs(B[:, jb]).max()
    A, B = A.astype(np.float32), B.astype(np.float32)
    C = gpu_tprod(T, A, B)
    assert np.isfinite(C).all()
    js = list(range(0, n4, max(1, n4 // 4)))
    if n3 <= 256:
        ref = O.tprod_alg1(A.astype(np.float64), B.astype(np.float64)).real
    else:                                               # long tubes: the sampled columns only
        ref = np.zeros((n1, n4, n3))
        ref[:, js] = O.tprod_columns(A.astype(np.float64), B.astype(np.float64), js)
    # C(i, j, :) scales with row i of A and column j of B: every output tube is accurate relative
    # to its OWN row's and column's scale, including on the inverse kernels that share one complex
    # FFT between output tubes i and i ^ 1 (R18: C-bar stays at the operands' scales through the
    # inverse FFT and each tube is unscaled afterwards)
    ra = np.abs(A).max(axis=(1, 2))
    for i in range(n1):
        for j in js:
            num = np.linalg.norm(C[i, j] - ref[i, j])
            den = ra[i] * np.abs(B[:, j]).max() * np.sqrt(n2 * n3)
            assert num <= 1e-5 * den, (i, j, num / den)


@pytest.mark.parametrize("dims", [(40, 24, 31, 36), (64, 64, 64, 64), (20, 12, 2048, 8), (36, 8, 4096, 8)],
                         ids=lambda d: "x".join(map(str, d)))
def test_zero_rows_columns_and_tensors(T, dims):
    """Degenerate operands: a zero row of A and a zero lateral slice of B take the max = 0 scale
    path (2^0, no division by zero) and give exactly zero rows / lateral slices of C, as Eq. (9)
    does (the oracle's are exactly zero too), also where the inverse shares one complex FFT
    between output tubes 3 and 2 (R18); an all-zero A gives an exactly zero C; the rest matches
    the oracle."""
    n1, n2, n3, n4 = dims
    A = normal((n1, n2, n3), 81 + n3)
    B = normal((n2, n4, n3), 82 + n3)
    A[3] = 0.0
    B[:, 5] = 0.0
    C = gpu_tprod(T, A, B)
    assert np.all(C[:, 5] == 0.0)
    assert np.all(C[3] == 0.0)
    ref = O.tprod_alg1(A.astype(np.float64), B.astype(np.float64)).real if n3 <= 64 else None
    if ref is not None:
        assert O.rel_err(C, ref) <= TOL32
    else:                                               # long tubes: sampled columns (Eq. (9))
        cols = [0, n4 - 1]
        assert O.rel_err(C[:, cols], O.tprod_columns(A, B, cols)) <= TOL32
    Z = gpu_tprod(T, np.zeros_like(A), B)
    assert np.all(Z == 0.0) and np.isfinite(Z).all()


@pytest.mark.parametrize("dims", [(64, 32, 31, 16), (64, 32, 64, 16), (32, 16, 4096, 4)],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("sa,sb", [(1e30, 1e-30), (1e-33, 1e28), (1e-20, 1e-15)], ids=str)
def test_extreme_operand_magnitudes(T, dims, sa, sb):
    """Operands at the ends of the fp32 range whose product is representable: the exact operand
    scales are undone by one combined exponent after the inverse (R18), so neither a huge A row
    times a tiny B column nor tiny operands overflow / flush an intermediate."""
    n1, n2, n3, n4 = dims
    A = (normal((n1, n2, n3), 91 + n3).astype(np.float64) * sa).astype(np.float32)
    B = (normal((n2, n4, n3), 92 + n3).astype(np.float64) * sb).astype(np.float32)
    C = gpu_tprod(T, A, B)
    assert np.isfinite(C).all()
    if n3 <= 64:
        ref = O.tprod_alg1(A.astype(np.float64), B.astype(np.float64)).real
        assert O.rel_err(C, ref) <= TOL32
    else:
        cols = [0, n4 - 1]
        assert O.rel_err(C[:, cols], O.tprod_columns(A.astype(np.float64), B.astype(np.float64), cols)) <= TOL32


def test_determinism_and_w_invariance(T):
    """Bitwise-repeatable, and lateral-slice shards equal the matching columns of the full
    result bitwise (no split-K; K order independent of n4) -- the multi-GPU partition run
    sequentially on one GPU."""
    A = normal((256, 192, 31), 3)
    B = normal((192, 300, 31), 4)
    C1 = gpu_tprod(T, A, B)
    C2 = gpu_tprod(T, A, B)
    assert np.array_equal(C1, C2)
    for W in (2, 3, 4):
        for r in range(W):
            s, e = lateral_shard(300, W, r)
            Cr = gpu_tprod(T, A, np.asfortranarray(B[:, s:e, :]))
            assert np.array_equal(Cr, C1[:, s:e, :]), (W, r)


def test_graph_replay_matches_direct(T):
    """TPROD_OPT_GRAPHS: from the second call with the same pointers / shapes / options the launch
    sequence replays as one CUDA graph.  Replays equal kernel-by-kernel launches bitwise, read the
    buffers' current contents (new data in the same tensors), keep the launch count, survive a
    workspace reallocation, cover the prepared-operand and fp64 paths, and still match the oracle."""
    import torch
    hg, hd = T.Handle(), T.Handle()
    hd.set_option(T._lib.TPROD_OPT_GRAPHS, 0)
    for dims in ((96, 80, 31, 72), (33, 17, 64, 40), (24, 16, 8192, 8)):
        n1, n2, n3, n4 = dims
        A = normal((n1, n2, n3), 31 + n3)
        B = normal((n2, n4, n3), 32 + n3)
        dA, dB = dev(A), dev(B)
        Cg = T.matlab_empty(n1, n4, n3, torch.float32, "cuda")
        Cd = T.matlab_empty(n1, n4, n3, torch.float32, "cuda")
        T.tprod(dA, dB, out=Cd, handle=hd)
        ref = host(Cd)
        if n3 <= 64:                                    # (the long-tube oracle check: test_fourstep_full_path)
            assert O.rel_err(ref, O.tprod_alg1(A.astype(np.float64), B.astype(np.float64)).real) <= TOL32
        counts = []
        for _ in range(3):                              # direct, capture + replay, replay
            Cg.zero_()
            T.tprod(dA, dB, out=Cg, handle=hg)
            assert np.array_equal(host(Cg), ref), dims
            counts.append(hg.last_launch_count())
        assert counts[0] == counts[1] == counts[2] == hd.last_launch_count()
        # new contents, same tensors: the replay reads them
        A2 = normal((n1, n2, n3), 41 + n3)
        dA.copy_(dev(A2))
        T.tprod(dA, dB, out=Cg, handle=hg)
        T.tprod(dA, dB, out=Cd, handle=hd)
        assert np.array_equal(host(Cg), host(Cd)), dims
    # workspace growth drops the cached graphs; the small shape captured before still runs right
    A = normal((40, 24, 7), 51)
    B = normal((24, 16, 7), 52)
    dA, dB = dev(A), dev(B)
    Cg = T.matlab_empty(40, 16, 7, torch.float32, "cuda")
    for _ in range(2):
        T.tprod(dA, dB, out=Cg, handle=hg)
    big_A, big_B = dev(normal((512, 512, 17), 53)), dev(normal((512, 512, 17), 54))
    T.tprod(big_A, big_B, handle=hg)
    for _ in range(3):
        T.tprod(dA, dB, out=Cg, handle=hg)
        assert np.array_equal(host(Cg), host(T.tprod(dA, dB, handle=hd)))
    # prepared operand
    A = normal((128, 96, 31), 55)
    dA = dev(A)
    hg.prepare_a(dA)
    hd.prepare_a(dA)
    dB = dev(normal((96, 40, 31), 56))
    Cg = T.matlab_empty(128, 40, 31, torch.float32, "cuda")
    for _ in range(3):
        T.tprod_prepared(dB, out=Cg, handle=hg)
        assert np.array_equal(host(Cg), host(T.tprod_prepared(dB, handle=hd)))
    # stage timing (TPROD_OPT_TIMING) bypasses the graphs: stage events between direct launches
    hg.set_option(T._lib.TPROD_OPT_TIMING, 1)
    dA, dB = dev(normal((96, 80, 31), 59)), dev(normal((80, 72, 31), 60))
    Cg = T.matlab_empty(96, 72, 31, torch.float32, "cuda")
    for _ in range(3):
        T.tprod(dA, dB, out=Cg, handle=hg)
        ms = hg.last_stage_ms()
        # small operands: the A and B chains run concurrently, stage 0 = K0 + K1 and stage 1 = 0 (tprod.h)
        assert len(ms) == 4 and ms[0] > 0 and ms[1] == 0.0 and ms[2] > 0 and ms[3] > 0, ms
        assert np.array_equal(host(Cg), host(T.tprod(dA, dB, handle=hd)))
    hg.set_option(T._lib.TPROD_OPT_TIMING, 0)
    # fp64
    A64, B64 = normal((20, 12, 9), 57, np.float64), normal((12, 8, 9), 58, np.float64)
    dA64, dB64 = dev(A64), dev(B64)
    C64 = T.matlab_empty(20, 8, 9, torch.float64, "cuda")
    for _ in range(3):
        T.tprod(dA64, dB64, out=C64, handle=hg)
        assert O.rel_err(host(C64), O.tprod_bcirc(A64, B64)) <= TOL64


def test_inside_caller_graph_capture(T):
    """A call made while the caller captures its stream joins the caller's graph (no nested
    capture); replaying that graph recomputes the product from the buffers' current contents."""
    import torch
    A, B = normal((64, 48, 16), 61), normal((48, 32, 16), 62)
    dA, dB = dev(A), dev(B)
    h = T.Handle()
    C = T.tprod(dA, dB, handle=h)                       # warm-up: workspace and tables exist
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            T.tprod(dA, dB, out=C, handle=h)
    A2 = normal((64, 48, 16), 63)
    dA.copy_(dev(A2))
    C.zero_()
    g.replay()
    assert O.rel_err(host(C), O.tprod_alg1(A2.astype(np.float64), B.astype(np.float64)).real) <= TOL32


def test_nccl_world_of_one(T):
    """The multi-GPU plumbing through the C ABI on one GPU: NCCL unique id, communicator init
    (world size 1) and the in-place broadcast used to replicate A; then a t-product on the
    broadcast tensor.  (World sizes > 1 need more GPUs than gpurun provides; the host logic is
    covered by tests/test_dist_gloo.py.)"""
    import torch
    uid = T.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    h = T.Handle()
    h.set_world(0, 1, uid)
    A = normal((40, 30, 9), 8)
    Ad = dev(A)
    before = host(Ad).copy()
    h.bcast_(Ad.permute(2, 1, 0), root=0)
    assert np.array_equal(host(Ad), before)
    B = normal((30, 20, 9), 9)
    assert O.rel_err(gpu_tprod(T, host(Ad), B, handle=h), O.tprod_bcirc(A, B)) <= TOL32
    with pytest.raises(T.TprodError):
        h.bcast_(Ad.permute(2, 1, 0), root=1)     # root out of range
    h2 = T.Handle()
    with pytest.raises(T.TprodError) as e:
        h2.bcast_(torch.zeros(4, device="cuda"))  # no world
    assert e.value.status == T._lib.TPROD_ENOWORLD


def test_host_entry_e2e(T):
    """tprod_f32_host / tprod_f64_host: host buffers in, host result out."""
    import torch
    for dt, tol in ((np.float32, TOL32), (np.float64, TOL64)):
        A = normal((50, 40, 7), 21, dt)
        B = normal((40, 30, 7), 22, dt)
        At, Bt = torch.from_numpy(A), torch.from_numpy(B)      # Fortran order = Matlab layout
        fn = T.tprod_f32_host if dt == np.float32 else T.tprod_f64_host
        C = fn(At, Bt).numpy()
        assert O.rel_err(C, O.tprod_bcirc(A, B)) <= tol


def test_host_entry_pipelined_bitwise(T):
    """tprod_f32_host above the pipelining threshold (B >= 32 MB: A prepared once, lateral-slice
    chunks of B / C double-buffered across copy and compute streams, ragged last chunk) returns
    exactly the one-shot device result."""
    import torch
    n1, n2, n3, n4 = 256, 1024, 32, 1003
    A = normal((n1, n2, n3), 81)
    B = normal((n2, n4, n3), 82)
    ref = gpu_tprod(T, A, B)
    At, Bt = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
    At, Bt = (x if T.is_matlab_layout(x) else T.to_matlab(x) for x in (At, Bt))
    out = T.matlab_empty(n1, n4, n3, torch.float32, "cpu").pin_memory()
    out = out if T.is_matlab_layout(out) else T.to_matlab(out)
    for _ in range(2):                                       # second call reuses the handle's buffers
        C = T.tprod_f32_host(At, Bt, out=out).numpy()
        assert np.array_equal(C, ref)
    J = np.array([0, 125, 126, 1002])
    assert O.rel_err(C[:, J, :], O.tprod_columns(A, B, J)) <= TOL32


def test_errors(T):
    import torch
    A = T.to_matlab(torch.randn(4, 5, 6, device="cuda"))
    B = T.to_matlab(torch.randn(5, 3, 6, device="cuda"))
    with pytest.raises(ValueError, match="shape mismatch"):
        T.tprod(A, T.to_matlab(torch.randn(4, 3, 6, device="cuda")))
    with pytest.raises(ValueError, match="Matlab layout"):
        T.tprod(torch.randn(4, 5, 6, device="cuda"), B)
    # aliasing output with an input -> TPROD_EALIAS from the C ABI
    X = T.to_matlab(torch.randn(4, 4, 6, device="cuda"))
    with pytest.raises(T.TprodError) as e:
        T.tprod(X, T.to_matlab(torch.randn(4, 4, 6, device="cuda")), out=X)
    assert e.value.status == T._lib.TPROD_EALIAS


# ------------------------------------------------------------------------------- full sizes
def _c3_inputs(rank5=False):
    c = CONFIGS["c3"]
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"])
    if rank5:
        U = normal((c["n1"], c["rank"], c["n3"]), c["seedU"], np.float64)
        V = normal((c["rank"], c["n2"], c["n3"]), c["seedV"], np.float64)
        A = O.tprod_bcirc(U, V).astype(np.float32)     # A' = U*V by the oracle, rounded to fp32
    else:
        A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"])
    return A, B


@pytest.mark.parametrize("rank5", [False, True], ids=["iid", "rank5"])
def test_config3_sampled(T, rank5):
    A, B = _c3_inputs(rank5)
    C = gpu_tprod(T, A, B)
    J = sample_columns(B.shape[1], 48)
    ref = O.tprod_columns(A, B, J)
    err = O.rel_err(C[:, J, :], ref)
    print("config3", "rank5" if rank5 else "iid", "sampled rel_err", err)
    assert err <= TOL32
    if rank5:
        # tubal rank <= 5 (Def. 2.7): every Fourier slice of C has sigma_6 / sigma_1 at fp32 noise
        Cb = np.fft.rfft(C[:, :64, :].astype(np.float64), axis=2)
        for f in range(0, Cb.shape[2], 5):
            s = np.linalg.svd(Cb[:, :, f], compute_uv=False)
            assert s[5] / s[0] < 1e-4


def test_config4_sampled(T):
    c = CONFIGS["c4"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"])
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"])
    C = gpu_tprod(T, A, B)
    J = np.array([0, 17, 63])
    tl = np.array([0, 1, 2, 1000, 2048, 4095])
    ref = O.tprod_blockrow(A, B, tl, J)
    err = O.rel_err(C[:, J][:, :, tl], ref)
    print("config4 sampled rel_err", err)
    assert err <= TOL32


@pytest.mark.slow
def test_config5_sampled(T):
    import torch
    c = CONFIGS["c5"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"])
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"])
    J = sample_columns(c["n4"], 32)
    ref = O.tprod_columns(A, B, J)
    Ad, Bd = dev(A), dev(B)
    C = T.tprod(Ad, Bd)
    Cj = host(C[:, torch.from_numpy(J).cuda(), :])
    err = O.rel_err(Cj, ref)
    print("config5 sampled rel_err", err)
    assert err <= TOL32
