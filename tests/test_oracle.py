"""Pins for the fp64 oracle (CPU only, -m "not gpu").

Each test ties an oracle function to something other than itself: the paper's printed
structural examples and SPEC's hand-derived worked examples (tests/golden/), closed forms,
numpy.fft as a library special case, and brute-force loops on tiny inputs.  Chosen so that a
dropped term, a wrong sign or index, or a transposed operand anywhere fails at least one."""
import itertools

import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, normal

RNG = np.random.default_rng(12345)


def rand(*shape):
    return RNG.standard_normal(shape)


def tube(v):
    return np.asarray(v, dtype=np.float64).reshape(1, 1, -1)


# ---------------------------------------------------------------- worked examples (golden)
def test_dft_worked_examples(golden):
    for key in ("dft_1x1x2", "dft_delta_1x1x4", "dft_1x1x1"):
        g = golden[key]
        got = O.dft_mode3(tube(g["tube"]))[0, 0]
        np.testing.assert_allclose(got.real, g["dft_re"], atol=1e-14)
        np.testing.assert_allclose(got.imag, g["dft_im"], atol=1e-14)


def test_idft_worked_example(golden):
    g = golden["idft_1x1x2"]
    got = O.idft_mode3(np.asarray(g["spec_re"], dtype=np.complex128).reshape(1, 1, -1))[0, 0]
    np.testing.assert_allclose(got.real, g["tube"], atol=1e-14)
    np.testing.assert_allclose(got.imag, 0, atol=1e-14)


def test_circ_display(golden):
    g = golden["circ_3"]
    np.testing.assert_array_equal(O.circ(np.array(g["v"])), np.array(g["circ"]))
    # bcirc of a 1x1xn3 tensor is circ of its tube (Eq. (6) reduces to the circ display)
    np.testing.assert_array_equal(O.bcirc(tube(g["v"])), np.array(g["circ"]))


def test_bcirc_block_pattern(golden):
    g = golden["bcirc_blocks_n3_4"]
    n3 = g["n3"]
    # tensor whose slice k (0-based) is filled with the value k+1 -> each block reveals its slice
    A = np.zeros((2, 3, n3))
    for k in range(n3):
        A[:, :, k] = k + 1
    M = O.bcirc(A)
    got = [[int(M[r * 2, c * 3]) for c in range(n3)] for r in range(n3)]
    assert got == g["slice_index"]


def test_tprod_worked_examples(golden):
    g = golden["tprod_n3_1"]
    A = np.array(g["A"], float)[:, :, None]
    B = np.array(g["B"], float)[:, :, None]
    np.testing.assert_array_equal(O.tprod_bcirc(A, B)[:, :, 0], np.array(g["C"], float))
    for key in ("tprod_tubes_1x1x2", "tprod_tubes_1x1x3"):
        g = golden[key]
        c = O.tprod_bcirc(tube(g["a"]), tube(g["b"]))[0, 0]
        np.testing.assert_array_equal(c, g["c"])
        c1 = O.tprod_alg1(tube(g["a"]), tube(g["b"]))[0, 0]
        np.testing.assert_allclose(c1.real, g["c"], atol=1e-13)
        cb = O.tprod_blockrow(tube(g["a"]), tube(g["b"]))[0, 0]
        np.testing.assert_array_equal(cb, g["c"])


def test_tran_example(golden):
    g = golden["tran_n3_4"]
    A = rand(3, 2, g["n3"]) + 1j * rand(3, 2, g["n3"])
    T = O.tran(A)
    for k, src in enumerate(g["source_slice_of_output"]):
        np.testing.assert_array_equal(T[:, :, k], A[:, :, src - 1].conj().T)


def test_teye_and_frobenius(golden):
    g = golden["teye_2_1"]
    np.testing.assert_array_equal(O.teye(g["n"], g["n3"]).transpose(2, 0, 1), np.array(g["slices"]))
    g = golden["frobenius_3_4"]
    assert O.frobenius(tube(g["tube"])) == pytest.approx(g["norm"], abs=0)


def test_rel_err_hand_values():
    """The parity gate itself (BASELINE.json north_star: ||X - Ref||_F / ||Ref||_F), pinned to
    values worked by hand: a mutation that returned 0, dropped the square root, used the max
    norm, normalised by ||X|| or ignored trailing dimensions fails one of these."""
    assert O.rel_err([4.0, 4.0], [3.0, 4.0]) == pytest.approx(0.2, abs=1e-15)          # |(1,0)| / 5
    assert O.rel_err([4.0, 5.0], [3.0, 4.0]) == pytest.approx(np.sqrt(2.0) / 5.0, abs=1e-15)  # not max norm 1/4
    assert O.rel_err([3.0, 4.0], [4.0, 5.0]) == pytest.approx(np.sqrt(2.0) / np.sqrt(41.0), abs=1e-15)
    assert O.rel_err([3.0, 4.0], [3.0, 4.0]) == 0.0
    assert O.rel_err([3.0, 4.0], [0.0, 0.0]) == pytest.approx(5.0, abs=0)                # zero reference: absolute
    X = np.zeros((2, 2, 2))
    R = np.ones((2, 2, 2))
    X[1, 1, 1] = 1.0                                   # 7 entries off by 1 out of ||R|| = sqrt(8)
    assert O.rel_err(X, R) == pytest.approx(np.sqrt(7.0 / 8.0), abs=1e-15)
    with pytest.raises(TypeError):                     # complex results must be reduced explicitly
        O.rel_err(np.array([1.0 + 1e-3j]), np.array([1.0]))
    with pytest.raises(ValueError):
        O.rel_err(np.zeros(3), np.zeros(4))


def test_inner_hand_values():
    """<A, B> = sum_k Tr(A^(k)* B^(k)), worked by hand on a complex tube pair
    (checks the conjugate sits on the first argument) and on a 2 x 2 x 1 pair (checks the trace
    pairs equal indices, not a transposed product)."""
    A = np.array([1 + 2j, 3.0]).reshape(1, 1, 2)
    B = np.array([2.0, 1 - 1j]).reshape(1, 1, 2)
    # conj(1+2i)*2 + conj(3)*(1-i) = (2-4i) + (3-3i)
    assert O.inner(A, B) == pytest.approx(5 - 7j, abs=1e-15)
    assert O.inner(B, A) == pytest.approx(5 + 7j, abs=1e-15)
    M = np.array([[1.0, 2.0], [3.0, 4.0]]).reshape(2, 2, 1)
    N = np.array([[5.0, 6.0], [7.0, 8.0]]).reshape(2, 2, 1)
    assert O.inner(M, N) == pytest.approx(1 * 5 + 2 * 6 + 3 * 7 + 4 * 8, abs=0)   # 70, not Tr(MN) = 69
    assert O.inner(M, M) == pytest.approx(O.frobenius(M) ** 2, abs=1e-12)


# ---------------------------------------------------------------- DFT machinery
@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 10, 31, 32, 64])
def test_dft_matrix_vs_library_and_eq1(n):
    F = O.dft_matrix(n)
    # Eq. (1): F^* F = n I
    np.testing.assert_allclose(F.conj().T @ F, n * np.eye(n), atol=1e-11 * n)
    # library special case: numpy.fft.fft uses the same unnormalised omega = e^{-2 pi i/n}
    x = rand(n)
    np.testing.assert_allclose(F @ x, np.fft.fft(x), atol=1e-12 * n)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_eq3_circulant_diagonalisation(n):
    """Eq. (3): F circ(v) F^{-1} = Diag(F v)."""
    v = rand(n)
    F = O.dft_matrix(n)
    lhs = F @ O.circ(v) @ np.linalg.inv(F)
    np.testing.assert_allclose(lhs, np.diag(F @ v), atol=1e-12)


@pytest.mark.parametrize("shape", [(3, 4, 5), (2, 2, 6), (1, 3, 1), (4, 1, 7)])
def test_dft_mode3_vs_numpy_fft_and_roundtrip(shape):
    A = rand(*shape)
    Ab = O.dft_mode3(A)
    np.testing.assert_allclose(Ab, np.fft.fft(A, axis=2), atol=1e-12)
    np.testing.assert_allclose(O.idft_mode3(Ab).real, A, atol=1e-13)
    np.testing.assert_allclose(O.hermitian_half(A), np.fft.rfft(A, axis=2), atol=1e-12)


@pytest.mark.parametrize("n3", [1, 2, 3, 4, 7, 8])
def test_eq8_conjugate_symmetry_and_parseval(n3):
    """Eq. (8) PAPER.md:L142-145 and Parseval (Eq. (1)) on the Hermitian half."""
    A = rand(3, 4, n3)
    Ab = O.dft_mode3(A)
    np.testing.assert_allclose(Ab[:, :, 0].imag, 0, atol=1e-13)
    for i in range(2, (n3 + 1) // 2 + 1):        # 1-based i as in Eq. (8)
        np.testing.assert_allclose(np.conj(Ab[:, :, i - 1]), Ab[:, :, n3 - i + 2 - 1], atol=1e-13)
    h = O.h_slices(n3)
    w = np.full(h, 2.0)
    w[0] = 1.0
    if n3 % 2 == 0:
        w[-1] = 1.0
    half = sum(w[f] * np.sum(np.abs(Ab[:, :, f]) ** 2) for f in range(h))
    assert half / n3 == pytest.approx(np.sum(A ** 2), rel=1e-12)


def test_h_slices():
    for n3 in range(1, 200):
        assert O.h_slices(n3) == n3 // 2 + 1 == int(np.ceil((n3 + 1) / 2))


# ---------------------------------------------------------------- t-product definition
def _brute_force(A, B):
    """Eq. (9) by explicit scalar loops: C[i,j,t] = sum_c sum_l bcirc-block(t,c)[i,l] B[l,j,c]."""
    n1, n2, n3 = A.shape
    n4 = B.shape[1]
    C = np.zeros((n1, n4, n3))
    for i, j, t in itertools.product(range(n1), range(n4), range(n3)):
        s = 0.0
        for c in range(n3):
            for l in range(n2):
                s += A[i, l, (t - c) % n3] * B[l, j, c]
        C[i, j, t] = s
    return C


@pytest.mark.parametrize("dims", [(2, 3, 4, 2), (1, 1, 3, 1), (3, 2, 1, 2), (2, 2, 5, 3), (1, 4, 2, 1)])
def test_bcirc_vs_brute_force(dims):
    n1, n2, n3, n4 = dims
    A, B = rand(n1, n2, n3), rand(n2, n4, n3)
    ref = _brute_force(A, B)
    np.testing.assert_allclose(O.tprod_bcirc(A, B), ref, atol=1e-12)
    np.testing.assert_allclose(O.tprod_blockrow(A, B), ref, atol=1e-12)
    np.testing.assert_allclose(O.tprod_columns(A, B, [n4 - 1])[:, 0, :], ref[:, n4 - 1, :], atol=1e-12)


def test_fold_unfold():
    A = rand(3, 2, 4)
    U = O.unfold(A)
    assert U.shape == (12, 2)
    np.testing.assert_array_equal(U[3:6], A[:, :, 1])
    np.testing.assert_array_equal(O.fold(U, 3, 2, 4), A)


def test_alg1_equals_definition_sweep():
    """SPEC.md:L183 acceptance shape: Alg. 1 vs Eq. (9) on >= 200 tiny instances."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(200):
        n1, n2, n4 = rng.integers(1, 6, size=3)
        n3 = int(rng.integers(1, 7))
        A, B = rng.standard_normal((n1, n2, n3)), rng.standard_normal((n2, n4, n3))
        C = O.tprod_bcirc(A, B)
        C1 = O.tprod_alg1(A, B)
        worst = max(worst, O.rel_err(C1.real, C))
        assert np.max(np.abs(C1.imag)) <= 1e-12 * max(1.0, np.max(np.abs(C)))
    assert worst < 1e-12


def test_library_fourier_path_equals_definition():
    """Special case reducing to library routines: numpy rfft + per-slice matmul + irfft."""
    A, B = rand(5, 6, 9), rand(6, 4, 9)
    Ab, Bb = np.fft.rfft(A, axis=2), np.fft.rfft(B, axis=2)
    Cb = np.einsum("ilf,ljf->ijf", Ab, Bb)
    C = np.fft.irfft(Cb, n=9, axis=2)
    assert O.rel_err(C, O.tprod_bcirc(A, B)) < 1e-13


def _config1():
    c = CONFIGS["c1"]
    A = normal((c["n1"], c["n2"], c["n3"]), c["seedA"], np.float64)
    B = normal((c["n2"], c["n4"], c["n3"]), c["seedB"], np.float64)
    D = normal((c["n4"], 8, c["n3"]), c["seedD"], np.float64)
    return A, B, D


def test_identity_eq7_block_diagonalisation():
    """Eq. (7) PAPER.md:L139 with literal Kronecker products, on config-1 dims."""
    A, _, _ = _config1()
    n1, n2, n3 = A.shape
    F = O.dft_matrix(n3)
    lhs = np.kron(F, np.eye(n1)) @ O.bcirc(A) @ np.kron(np.linalg.inv(F), np.eye(n2))
    rhs = O.bdiag(O.dft_mode3(A))
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-13


def test_identity_teye():
    """A * I = A and I * A = A; I-bar slices are all I (same line)."""
    A, _, _ = _config1()
    n1, n2, n3 = A.shape
    np.testing.assert_allclose(O.tprod_bcirc(A, O.teye(n2, n3)), A, atol=1e-15)
    np.testing.assert_allclose(O.tprod_bcirc(O.teye(n1, n3), A), A, atol=1e-15)
    Ib = O.dft_mode3(O.teye(4, n3))
    for f in range(n3):
        np.testing.assert_allclose(Ib[:, :, f], np.eye(4), atol=1e-14)
    # bcirc(I) is the identity matrix
    np.testing.assert_array_equal(O.bcirc(O.teye(3, 4)), np.eye(12))


def test_identity_associativity_and_bilinearity():
    A, B, D = _config1()
    lhs = O.tprod_bcirc(O.tprod_bcirc(A, B), D)
    rhs = O.tprod_bcirc(A, O.tprod_bcirc(B, D))
    assert O.rel_err(lhs, rhs) < 1e-13
    B2 = rand(*B.shape)
    lin = O.tprod_bcirc(A, B + 2.5 * B2)
    assert O.rel_err(lin, O.tprod_bcirc(A, B) + 2.5 * O.tprod_bcirc(A, B2)) < 1e-13


def test_identity_transpose_antihomomorphism():
    """(A*B)^* = B^* * A^* under Def. 2.2."""
    A, B, _ = _config1()
    lhs = O.tran(O.tprod_bcirc(A, B))
    rhs = O.tprod_bcirc(O.tran(B), O.tran(A))
    assert O.rel_err(lhs, rhs) < 1e-13
    np.testing.assert_array_equal(O.tran(O.tran(A)), A)


def test_real_in_real_out():
    """Lemma 2.1 / Eq. (8): the full complex Fourier route (all n3 slices multiplied, no
    conjugate fill) gives a real result equal to the definition."""
    A, B, _ = _config1()
    C = O.tprod_alg1(A, B, full=True)
    assert np.max(np.abs(C.imag)) / np.max(np.abs(C.real)) < 1e-13
    assert O.rel_err(C.real, O.tprod_bcirc(A, B)) < 1e-13


def test_shift_equivariance():
    """A * roll(B, s) = roll(A * B, s) along mode 3 (circular convolution of slice sequences)."""
    A, B = rand(3, 4, 7), rand(4, 2, 7)
    C = O.tprod_bcirc(A, B)
    for s in (1, 3):
        np.testing.assert_allclose(O.tprod_bcirc(A, np.roll(B, s, axis=2)), np.roll(C, s, axis=2), atol=1e-13)
        np.testing.assert_allclose(O.tprod_bcirc(np.roll(A, s, axis=2), B), np.roll(C, s, axis=2), atol=1e-13)


def test_tubal_rank_structure():
    """Def. 2.7: U*V with U n1 x r x n3 has every Fourier slice of rank <= r."""
    U, V = rand(9, 2, 5), rand(2, 8, 5)
    P = O.tprod_bcirc(U, V)
    Pb = O.dft_mode3(P)
    for f in range(5):
        s = np.linalg.svd(Pb[:, :, f], compute_uv=False)
        assert s[2] / s[0] < 1e-12


def test_shape_mismatch():
    with pytest.raises(ValueError):
        O.tprod_bcirc(rand(2, 3, 4), rand(2, 3, 4))


def test_generator_recipe():
    """synth.normal is Matlab-ordered default_rng(seed).standard_normal, rounded to the dtype."""
    x = normal((3, 4, 5), 7, np.float32)
    ref = np.random.default_rng(7).standard_normal(60).astype(np.float32)
    np.testing.assert_array_equal(x.ravel(order="F"), ref)
    assert x.flags.f_contiguous


@pytest.mark.parametrize("chunk", [5, 17, 1 << 24])
def test_normal_lateral_is_the_global_stream(monkeypatch, chunk):
    """synth.normal_lateral(shape, seed, j0, j1) equals normal(shape, seed)[:, j0:j1, :] for any
    chunking of the stream (the per-rank inputs of the strong-scaling bench)."""
    import synth
    monkeypatch.setattr(synth, "_CHUNK", chunk)
    full = synth.normal((7, 13, 5), 3)
    for j0, j1 in ((0, 13), (0, 1), (4, 9), (12, 13)):
        part = synth.normal_lateral((7, 13, 5), 3, j0, j1)
        assert part.flags.f_contiguous
        np.testing.assert_array_equal(part, full[:, j0:j1, :])


# ------------------------------------------------------------------ Definition 2.4 (NEXT-4)
def _well_conditioned(n, n3, seed):
    """Random n x n x n3 tensor whose spectral slices are diagonally dominant (well conditioned)."""
    A = normal((n, n, n3), seed, np.float64) * 0.2
    A[:, :, 0] += 2.0 * np.eye(n)                     # adds 2I to every spectral slice (DC of a delta)
    return A


def test_tinv_identity_and_worked_tubes(golden):
    """tinv(teye) = teye; SPEC's tube examples: (1, 0) and (0, 1) are their own inverses
    (circ((0,1)) = [[0,1],[1,0]], SPEC.md [OP] tinv examples)."""
    np.testing.assert_allclose(O.tinv(O.teye(3, 4)), O.teye(3, 4), atol=1e-15)
    np.testing.assert_allclose(O.tinv(np.array([1.0, 0.0]).reshape(1, 1, 2)).ravel(), [1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(O.tinv(np.array([0.0, 1.0]).reshape(1, 1, 2)).ravel(), [0.0, 1.0], atol=1e-15)


def test_tinv_eq11_both_sides_and_involution():
    """Eq. (11): A * B = I and B * A = I (the definition solves only the first); tinv(tinv(A)) = A."""
    for n, n3, seed in ((4, 5, 1), (3, 8, 2), (6, 1, 3)):
        A = _well_conditioned(n, n3, seed)
        B = O.tinv(A)
        I = O.teye(n, n3)
        assert O.rel_err(O.tprod_bcirc(A, B), I) < 1e-13
        assert O.rel_err(O.tprod_bcirc(B, A), I) < 1e-13
        assert O.rel_err(O.tinv(B), A) < 1e-13


def test_tinv_n3_1_is_matrix_inverse():
    """n3 = 1: bcirc(A) = A, so tinv is numpy.linalg.inv (library special case)."""
    A = _well_conditioned(7, 1, 4)
    np.testing.assert_allclose(O.tinv(A)[:, :, 0], np.linalg.inv(A[:, :, 0]), rtol=1e-12, atol=1e-14)


def test_tinv_singular():
    """The zero tensor and a tensor with one planted zero spectral slice have no inverse."""
    with pytest.raises(O.SingularTensor):
        O.tinv(np.zeros((3, 3, 4)))
    A = _well_conditioned(3, 5, 5)
    Ab = O.dft_mode3(A)
    Ab[:, :, 2] = 0.0
    Ab[:, :, 3] = 0.0                                   # its conjugate partner (5 - 2), keeps A real
    A0 = np.real(O.idft_mode3(Ab))
    with pytest.raises(O.SingularTensor):
        O.tinv(A0)


# ------------------------------------------------------------------ Algorithm 3 (NEXT-2)
def test_tsvt_limits():
    """tau = 0 is the identity; tau >= every spectral singular value gives the zero tensor."""
    Y = normal((5, 4, 6), 11, np.float64)
    assert O.rel_err(O.tsvt(Y, 0.0), Y) < 1e-14
    smax = max(np.linalg.svd(O.dft_mode3(Y)[:, :, f], compute_uv=False)[0] for f in range(6))
    assert np.abs(O.tsvt(Y, smax * 1.0001)).max() < 1e-14


def test_tsvt_tube_closed_form():
    """1 x 1 x n3 tubes: every spectral 'matrix' is a scalar y, whose SVT is y * (1 - tau/|y|)_+ ;
    worked by hand for the tube (3, 1): spectrum (4, 2), tau = 1 -> (3, 1) -> tube (2, 1)."""
    got = O.tsvt(np.array([3.0, 1.0]).reshape(1, 1, 2), 1.0).ravel()
    np.testing.assert_allclose(got, [2.0, 1.0], atol=1e-14)


def test_tsvt_is_the_prox_of_eq19():
    """Eq. (19): X = tsvt(Y, tau) minimises tau * TNN(X) + 1/2 ||X - Y||_F^2, with TNN through
    bcirc (Eq. (18), an independent route): no random perturbation lowers the objective, and
    moving towards Y or towards 0 does not either (first-order optimality, checked numerically)."""
    rng = np.random.default_rng(3)
    Y = normal((4, 3, 5), 12, np.float64)
    tau = 1.5
    X = O.tsvt(Y, tau)
    obj = lambda Z: tau * O.tnn_bcirc(Z) + 0.5 * np.sum((Z - Y) ** 2)
    f0 = obj(X)
    for _ in range(40):
        D = rng.standard_normal(Y.shape)
        for eps in (1e-3, 1e-2):
            assert obj(X + eps * D / np.linalg.norm(D)) >= f0 - 1e-10
    for t in (0.9, 1.1):
        assert obj(t * X) >= f0 - 1e-10
    assert obj(Y) >= f0 and obj(np.zeros_like(Y)) >= f0


def test_tsvt_keeps_low_tubal_rank():
    """Prox of a tubal-rank-2 tensor (U * V, Def. 2.7) has every spectral slice of rank <= 2."""
    U = normal((6, 2, 7), 13, np.float64)
    V = normal((2, 5, 7), 14, np.float64)
    X = O.tsvt(O.tprod_bcirc(U, V), 0.5)
    Xb = O.dft_mode3(X)
    for f in range(7):
        s = np.linalg.svd(Xb[:, :, f], compute_uv=False)
        assert s[2] < 1e-12 * max(s[0], 1.0)


# ------------------------------------------------------------------ t-SVD scalars (NEXT-3)
def test_tsvd_values_pins():
    """Eq. (13): S(i,i,1) non-increasing; Def. 2.9 TNN = ||bcirc||_* / n3 (Eq. (18), independent
    route); Def. 2.8 TSN = max spectral sigma_max (Eq. (17)); Eq. (16) tubal rank of U * V (rank 3)
    and of teye (n); n3 = 1 reduces to the matrix singular values."""
    A = normal((6, 5, 7), 21, np.float64)
    s, tnn, tsn, rank = O.tsvd_values(A)
    assert np.all(np.diff(s) <= 1e-12)
    assert abs(tnn - O.tnn_bcirc(A)) < 1e-10 * tnn
    Ab = O.dft_mode3(A)
    assert abs(tsn - max(np.linalg.svd(Ab[:, :, j], compute_uv=False)[0] for j in range(7))) < 1e-10 * tsn
    assert rank == 5
    U = normal((6, 3, 7), 22, np.float64)
    V = normal((3, 5, 7), 23, np.float64)
    assert O.tsvd_values(O.tprod_bcirc(U, V))[3] == 3
    assert O.tsvd_values(O.teye(4, 5))[3] == 4
    np.testing.assert_allclose(O.tsvd_values(A[:, :, :1])[0], np.linalg.svd(A[:, :, 0], compute_uv=False),
                               rtol=1e-12)


def test_tsvd_factors_pins():
    """Theorem 2.2 / Eq. (12): A = U * S * V^* (t-products through bcirc, Def. 2.2 transpose);
    skinny orthogonality U^* * U = V^* * V = I (Def. 2.5 on r columns); S f-diagonal (Def. 2.6)
    with S(:,:,1)'s diagonal = the Eq. (14) singular values; wide and tall shapes."""
    for dims, seed in (((6, 4, 5), 31), ((3, 7, 4), 32), ((5, 5, 1), 33)):
        A = normal(dims, seed, np.float64)
        U, S, V = O.tsvd(A)
        r = min(dims[0], dims[1])
        assert O.rel_err(O.tprod_bcirc(O.tprod_bcirc(U, S), O.tran(V)), A) < 1e-13
        assert O.rel_err(O.tprod_bcirc(O.tran(U), U), O.teye(r, dims[2])) < 1e-13
        assert O.rel_err(O.tprod_bcirc(O.tran(V), V), O.teye(r, dims[2])) < 1e-13
        off = S.copy()
        for k in range(dims[2]):
            off[:, :, k] -= np.diag(np.diag(S[:, :, k]))
        assert np.abs(off).max() < 1e-13
        np.testing.assert_allclose(np.diag(S[:, :, 0]), O.tsvd_values(A)[0], rtol=1e-12)


def test_tsvd_full_factors_pins():
    """Theorem 2.2 in its stated shapes: U n1 x n1, S n1 x n2 f-diagonal,
    V n2 x n2 with A = U * S * V^* and BOTH U^* * U = U * U^* = I_n1 and V^* * V = V * V^* = I_n2
    (orthogonal, Def. 2.5: square, so the product in either order is the identity); S's leading
    r x r block equals the skinny S; tall, wide and rank-deficient shapes."""
    U0 = normal((7, 2, 4), 36, np.float64)
    V0 = normal((2, 5, 4), 37, np.float64)
    cases = ((normal((6, 4, 5), 34, np.float64)), normal((3, 7, 4), 35, np.float64), O.tprod_bcirc(U0, V0))
    for A in cases:
        n1, n2, n3 = A.shape
        r = min(n1, n2)
        U, S, V = O.tsvd(A, full=True)
        assert U.shape == (n1, n1, n3) and S.shape == (n1, n2, n3) and V.shape == (n2, n2, n3)
        assert O.rel_err(O.tprod_bcirc(O.tprod_bcirc(U, S), O.tran(V)), A) < 1e-13
        for Q, n in ((U, n1), (V, n2)):
            assert O.rel_err(O.tprod_bcirc(O.tran(Q), Q), O.teye(n, n3)) < 1e-13
            assert O.rel_err(O.tprod_bcirc(Q, O.tran(Q)), O.teye(n, n3)) < 1e-13
        off = S.copy()
        for k in range(n3):
            off[np.arange(r), np.arange(r), k] = 0.0
        assert np.abs(off).max() < 1e-13
        _, Ss, _ = O.tsvd(A)
        assert O.rel_err(S[:r, :r, :], Ss) < 1e-13
