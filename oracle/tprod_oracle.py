"""fp64 CPU oracle for the t-product of Lu, *Tensor-Tensor Product Toolbox* (arXiv 1806.07247).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import or execute anything under ``oracle/``.
The product path (``paper_1806_07247_b200``) never imports this module, and this module never
imports the product path: the two share no kernels, headers, tables or helpers.  Only the seeded
input generators in ``synth/`` (which hold none of the method's arithmetic) serve both.

Everything here is plain numpy in float64 (complex128 where the paper goes to the Fourier
domain), written to be checked against the paper by eye.  Citations are ``PAPER.md:Lx-Ly``
(lines of /root/reference/PAPER.md) with the equation / definition / algorithm they fall in.

Conventions:
  * A tensor is a numpy array indexed ``A[i, j, k]`` (0-based); frontal slice ``A^(k+1)`` of
    the paper is ``A[:, :, k]`` (Matlab notation ``A(:,:,i)``).
  * The DFT is the unnormalised F_n with omega = exp(-2*pi*i/n) (Eq. (1)-(2)),
    and the inverse is F_n^{-1} = F_n^* / n.

Pins: every function below is checked by ``tests/test_oracle.py`` against something other than
itself (the paper's printed structural examples, SPEC's hand-derived worked examples in
``tests/golden/``, closed forms, numpy.fft as a library special case, and brute-force loops),
including the parity metric ``rel_err`` and ``inner`` (hand-evaluated values,
``test_rel_err_hand_values`` / ``test_inner_hand_values``).  No function here is "parity
unpinned".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "dft_matrix", "circ", "bcirc", "unfold", "fold", "tprod_bcirc", "tprod_blockrow",
    "tprod_columns", "dft_mode3", "idft_mode3", "bdiag", "teye", "tran", "tprod_alg1",
    "hermitian_half", "frobenius", "inner", "rel_err", "h_slices", "tinv", "SingularTensor",
    "tsvt", "tnn_bcirc", "tsvd_values", "tsvd",
]


def h_slices(n3: int) -> int:
    """Number of frequency slices Algorithm 1 multiplies: ceil((n3+1)/2).

    Equal to floor(n3/2)+1 for every integer n3 >= 1 (reading R1)."""
    return -(-(n3 + 1) // 2)


# --------------------------------------------------------------------------------------------
# Section 2.2: DFT machinery
# --------------------------------------------------------------------------------------------
def dft_matrix(n: int) -> np.ndarray:
    """The DFT matrix F_n of PAPER.md:L90-94 (display before Eq. (1)).

    F_n[j, k] = omega^(j*k), omega = exp(-2*pi*i/n), 0-based j, k.  The exponent j*k is reduced
    mod n first so that large products do not lose accuracy in the angle (same value)."""
    jk = np.outer(np.arange(n), np.arange(n)) % n
    return np.exp(-2j * np.pi * jk / n)


def circ(v: np.ndarray) -> np.ndarray:
    """circ(v) of PAPER.md:L104: first column is v, each next column is the previous one
    rotated down by one, i.e. circ(v)[r, c] = v[(r - c) mod n]."""
    v = np.asarray(v)
    n = v.shape[0]
    out = np.empty((n, n), dtype=v.dtype)
    for r in range(n):
        for c in range(n):
            out[r, c] = v[(r - c) % n]
    return out


def bcirc(A: np.ndarray) -> np.ndarray:
    """Block-circulant matrix of Eq. (6).

    Block (r, c) (0-based, each n1 x n2) is frontal slice A^((r - c) mod n3), so the first block
    column is A^(1), A^(2), ..., A^(n3) top to bottom, exactly as displayed."""
    n1, n2, n3 = A.shape
    M = np.empty((n1 * n3, n2 * n3), dtype=A.dtype)
    for r in range(n3):
        for c in range(n3):
            M[r * n1:(r + 1) * n1, c * n2:(c + 1) * n2] = A[:, :, (r - c) % n3]
    return M


def unfold(A: np.ndarray) -> np.ndarray:
    """unfold(A) of PAPER.md:L151-155: frontal slices A^(1..n3) stacked vertically, (n1*n3) x n2."""
    n1, n2, n3 = A.shape
    return np.concatenate([A[:, :, k] for k in range(n3)], axis=0)


def fold(M: np.ndarray, n1: int, n2: int, n3: int) -> np.ndarray:
    """Inverse of unfold (fold(unfold(A)) = A)."""
    if M.shape != (n1 * n3, n2):
        raise ValueError(f"fold: matrix {M.shape} does not match {(n1 * n3, n2)}")
    A = np.empty((n1, n2, n3), dtype=M.dtype)
    for k in range(n3):
        A[:, :, k] = M[k * n1:(k + 1) * n1, :]
    return A


def dft_mode3(A: np.ndarray) -> np.ndarray:
    """A-bar = fft(A, [], 3): the DFT of Eq. (2) (v-bar = F_n v, L100)
    applied to every tube A(i, j, :).  Written with the literal matrix F_n, no FFT."""
    n3 = A.shape[2]
    F = dft_matrix(n3)
    # Abar[i, j, f] = sum_k F[f, k] * A[i, j, k]
    return np.einsum("fk,ijk->ijf", F, A.astype(np.complex128))


def idft_mode3(Abar: np.ndarray) -> np.ndarray:
    """A = ifft(A-bar, [], 3) with F_n^{-1} = F_n^* / n."""
    n3 = Abar.shape[2]
    Finv = dft_matrix(n3).conj() / n3
    return np.einsum("kf,ijf->ijk", Finv, Abar)


def bdiag(Abar: np.ndarray) -> np.ndarray:
    """Block-diagonal matrix of Eq. (5): i-th diagonal block = A-bar^(i)."""
    n1, n2, n3 = Abar.shape
    M = np.zeros((n1 * n3, n2 * n3), dtype=np.complex128)
    for f in range(n3):
        M[f * n1:(f + 1) * n1, f * n2:(f + 1) * n2] = Abar[:, :, f]
    return M


def hermitian_half(A: np.ndarray) -> np.ndarray:
    """Frequency slices f = 0 .. h-1 of dft_mode3(A), h = ceil((n3+1)/2) (Alg. 1 step 2,
    PAPER.md:L177); by Eq. (8) the remaining slices are conjugates."""
    return dft_mode3(A)[:, :, :h_slices(A.shape[2])]


# --------------------------------------------------------------------------------------------
# Section 2.3: t-product and companions
# --------------------------------------------------------------------------------------------
def _check_pair(A: np.ndarray, B: np.ndarray) -> None:
    if A.ndim != 3 or B.ndim != 3 or A.shape[1] != B.shape[0] or A.shape[2] != B.shape[2]:
        raise ValueError(f"t-product shape mismatch: A {A.shape} vs B {B.shape}")


def tprod_bcirc(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Definition 2.1, Eq. (9): A * B = fold(bcirc(A) . unfold(B)).

    The literal definition: the n1n3 x n2n3 block-circulant matrix is materialised and
    multiplied with one dense (BLAS) product."""
    _check_pair(A, B)
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    n1, n2, n3 = A.shape
    n4 = B.shape[1]
    return fold(bcirc(A) @ unfold(B), n1, n4, n3)


def tprod_blockrow(A: np.ndarray, B: np.ndarray, t_list=None, cols=None) -> np.ndarray:
    """Eq. (9) evaluated one block row of bcirc(A) at a time, for sizes where bcirc(A) does not
    fit in memory.

    Block row t of bcirc(A) is [A^((t - c) mod n3)]_{c = 0..n3-1} (Eq. (6)); multiplying it by
    unfold(B) gives frontal slice t of C:  C^(t) = sum_c A^((t - c) mod n3) . B^(c).
    Lateral slices are independent (columns of unfold(B) map 1:1 to columns of unfold(C)),
    so ``cols`` restricts the computation to C(:, cols, :) exactly.  ``t_list`` restricts the
    frontal slices.  Returns an array of shape (n1, len(cols), len(t_list))."""
    _check_pair(A, B)
    n1, n2, n3 = A.shape
    n4 = B.shape[1]
    cols = np.arange(n4) if cols is None else np.asarray(cols)
    t_list = np.arange(n3) if t_list is None else np.asarray(t_list)
    Bc = np.asarray(B[:, cols, :], dtype=np.float64)              # n2 x |J| x n3
    unfB = Bc.transpose(2, 0, 1).reshape(n3 * n2, len(cols))       # = unfold(B(:, J, :))
    out = np.empty((n1, len(cols), len(t_list)), dtype=np.float64)
    A64 = np.asarray(A, dtype=np.float64)
    for ti, t in enumerate(t_list):
        idx = (t - np.arange(n3)) % n3                             # slice index of block (t, c)
        row = A64[:, :, idx].transpose(0, 2, 1).reshape(n1, n3 * n2)  # [A^(t-0) | A^(t-1) | ...]
        out[:, :, ti] = row @ unfB
    return out


def tprod_columns(A: np.ndarray, B: np.ndarray, cols) -> np.ndarray:
    """C(:, cols, :) of Eq. (9) for every frontal slice (block-row form, see tprod_blockrow)."""
    return tprod_blockrow(A, B, None, cols)


def teye(n: int, n3: int) -> np.ndarray:
    """Identity tensor, Definition 2.3: first frontal slice I_n, others zero."""
    I = np.zeros((n, n, n3))
    I[:, :, 0] = np.eye(n)
    return I


def tran(A: np.ndarray) -> np.ndarray:
    """Conjugate transpose, Definition 2.2: conjugate-transpose every
    frontal slice, then reverse the order of transposed slices 2 .. n3 (1-based)."""
    n1, n2, n3 = A.shape
    T = np.empty((n2, n1, n3), dtype=A.dtype)
    T[:, :, 0] = A[:, :, 0].conj().T
    for k in range(1, n3):
        T[:, :, k] = A[:, :, n3 - k].conj().T
    return T


class SingularTensor(ValueError):
    """No inverse to working precision (SPEC.md [OP] tinv errors; the paper is silent)."""


def tinv(A: np.ndarray, rtol: float | None = None) -> np.ndarray:
    """Tensor inverse, Definition 2.4, Eq. (11): the B with A * B = I.

    Literal form through Eq. (9): A * B = I  <=>  bcirc(A) . unfold(B) = unfold(I), so
    unfold(B) = bcirc(A)^-1 . unfold(teye(n, n3)) (one dense solve); then B * A = I holds as well.
    Existence check (reading R16; the paper gives none): every spectral slice A-bar^(f)
    (literal DFT, Eq. (2)) must have sigma_min > rtol * s_max, where s_max is the largest singular
    value over all slices (= ||bcirc(A)||_2, Eq. (7)) and rtol defaults to n * n3 * float64
    epsilon; otherwise SingularTensor.  (SPEC.md's per-slice ratio would accept a slice that is
    zero up to round-off.)"""
    A = np.asarray(A, dtype=np.float64)
    n1, n2, n3 = A.shape
    if n1 != n2:
        raise ValueError(f"tinv needs square frontal slices, got {A.shape}")
    if rtol is None:
        rtol = n1 * n3 * np.finfo(np.float64).eps
    Abar = dft_mode3(A)
    svs = [np.linalg.svd(Abar[:, :, f], compute_uv=False) for f in range(n3)]
    smax = max(float(sv[0]) for sv in svs)
    for f, sv in enumerate(svs):
        if not smax > 0 or sv[-1] <= rtol * smax:
            raise SingularTensor(f"spectral slice {f} is singular (sigma_min / max sigma = "
                                 f"{(sv[-1] / smax) if smax > 0 else 0.0:.3e})")
    X = np.linalg.solve(bcirc(A), unfold(teye(n1, n3)))
    return fold(X, n1, n1, n3)


def tsvt(Y: np.ndarray, tau: float) -> np.ndarray:
    """Algorithm 3, t-SVT, step by step: Prox of tau * TNN (Eq. (19)-(21)).

    1. Y-bar = fft(Y, [], 3) (literal DFT, Eq. (2)).
    2. For i = 1..ceil((n3+1)/2): [U, S, V] = SVD(Y-bar^(i)); W-bar^(i) = U (S - tau)_+ V^*;
       for the rest W-bar^(i) = conj(W-bar^(n3-i+2)) (the garbled "ena ioi" of L298-300 read as
       "end for", R5).
    3. Prox = ifft(W-bar, [], 3) (real for real Y; the imaginary round-off is dropped)."""
    Y = np.asarray(Y, dtype=np.float64)
    n1, n2, n3 = Y.shape
    Ybar = dft_mode3(Y)
    Wbar = np.empty_like(Ybar)
    hh = h_slices(n3)
    for i in range(1, hh + 1):
        U, S, Vh = np.linalg.svd(Ybar[:, :, i - 1], full_matrices=False)
        Wbar[:, :, i - 1] = (U * np.maximum(S - tau, 0.0)) @ Vh
    for i in range(hh + 1, n3 + 1):
        Wbar[:, :, i - 1] = np.conj(Wbar[:, :, (n3 - i + 2) - 1])
    return np.real(idft_mode3(Wbar))


def tsvd_values(A: np.ndarray, rtol: float = 1e-10):
    """Scalars of the t-SVD (Theorem 2.2, Algorithm 2 step 2), literally:
      singular values of A:  S(i, i, 1) = (1/n3) sum_j S-bar(i, i, j)         (Eq. (14)), i < min(n1, n2),
        S-bar(:, :, j) = the singular values of A-bar^(j) for ALL n3 slices (no symmetry used);
      tubal rank:  #{i : S(i, i, 1) > rtol * S(1, 1, 1)}                        (Eq. (16));
      TSN:  ||bcirc(A)||_2                                                       (Definition 2.8);
      TNN:  sum_i S(i, i, 1)                                                     (Definition 2.9).
    Returns (s, tnn, tsn, rank)."""
    A = np.asarray(A, dtype=np.float64)
    n1, n2, n3 = A.shape
    Abar = dft_mode3(A)
    Sbar = np.stack([np.linalg.svd(Abar[:, :, j], compute_uv=False) for j in range(n3)], axis=1)
    s = Sbar.mean(axis=1)
    tsn = float(np.linalg.norm(bcirc(A), 2))
    rank = int(np.sum(s > rtol * s[0])) if s[0] > 0 else 0
    return s, float(s.sum()), tsn, rank


def tsvd(A: np.ndarray, full: bool = False):
    """Algorithm 2, T-SVD, step by step: A-bar = fft(A, [], 3); for
    i = 1..ceil((n3+1)/2): [U-bar, S-bar, V-bar] = SVD(A-bar^(i)); the rest by conjugation (S-bar
    copied); U = ifft(U-bar), S = ifft(S-bar), V = ifft(V-bar).  full=False: the skinny form (r =
    min(n1, n2) columns, reading R17), U n1 x r x n3, S r x r x n3, V n2 x r x n3;
    full=True: Theorem 2.2's shapes, U n1 x n1 x n3, S n1 x n2 x n3 (f-diagonal), V n2 x n2 x n3.
    Either way A = U * S * V^* (Eq. (12)).  The factors are unique up to a unit phase per singular
    vector and spectral slice (and, full, up to a unitary mix of the null-space columns); S is
    unique."""
    A = np.asarray(A, dtype=np.float64)
    n1, n2, n3 = A.shape
    r = min(n1, n2)
    cu, cv = (n1, n2) if full else (r, r)
    Ab = dft_mode3(A)
    Ub = np.empty((n1, cu, n3), dtype=np.complex128)
    Sb = np.zeros((cu, cv, n3), dtype=np.complex128)
    Vb = np.empty((n2, cv, n3), dtype=np.complex128)
    hh = h_slices(n3)
    for i in range(1, hh + 1):
        M = Ab[:, :, i - 1]
        if i == 1 or 2 * (i - 1) == n3:
            # Eq. (8): the self-conjugate slices (DC, and Nyquist for even n3)
            # are real; the literal DFT leaves ~1e-16 imaginary noise, which would let LAPACK pick
            # complex null-space vectors that the conjugate fill cannot represent (R19)
            M = M.real
        U, S, Vh = np.linalg.svd(M, full_matrices=full)
        Sd = np.zeros((cu, cv))
        Sd[np.arange(r), np.arange(r)] = S
        Ub[:, :, i - 1], Sb[:, :, i - 1], Vb[:, :, i - 1] = U, Sd, Vh.conj().T
    for i in range(hh + 1, n3 + 1):
        j = (n3 - i + 2) - 1
        Ub[:, :, i - 1], Sb[:, :, i - 1], Vb[:, :, i - 1] = np.conj(Ub[:, :, j]), Sb[:, :, j], np.conj(Vb[:, :, j])
    return (np.real(idft_mode3(Ub)), np.real(idft_mode3(Sb)), np.real(idft_mode3(Vb)))


def tnn_bcirc(X: np.ndarray) -> float:
    """Tensor nuclear norm through Eq. (18): ||X||_* = ||bcirc(X)||_* / n3 (the 1/n3
    makes Eq. (18) agree with Definition 2.9, ||X||_* = sum_i S(i, i, 1), SPEC.md:L340 / DESIGN.md
    R5); an independent route to the objective of Eq. (19) for testing Algorithm 3."""
    X = np.asarray(X, dtype=np.float64)
    return float(np.linalg.svd(bcirc(X), compute_uv=False).sum()) / X.shape[2]


def tprod_alg1(A: np.ndarray, B: np.ndarray, full: bool = False) -> np.ndarray:
    """Algorithm 1, step by step, in complex128 with the literal DFT matrix.

    1. A-bar = fft(A,[],3), B-bar = fft(B,[],3).
    2. C-bar^(i) = A-bar^(i) B-bar^(i) for i = 1..ceil((n3+1)/2); C-bar^(i) = conj(C-bar^(n3-i+2))
       for the rest.  With ``full=True`` every slice is multiplied instead (no conjugate fill),
       used to test Lemma 2.1 / Eq. (8).
    3. C = ifft(C-bar,[],3).
    Returns the complex result (its imaginary part is round-off for real inputs)."""
    _check_pair(A, B)
    n1, n2, n3 = A.shape
    n4 = B.shape[1]
    Abar = dft_mode3(A)
    Bbar = dft_mode3(B)
    Cbar = np.empty((n1, n4, n3), dtype=np.complex128)
    hh = n3 if full else h_slices(n3)
    for i in range(1, hh + 1):                       # 1-based slice index as in the paper
        Cbar[:, :, i - 1] = Abar[:, :, i - 1] @ Bbar[:, :, i - 1]
    for i in range(hh + 1, n3 + 1):
        Cbar[:, :, i - 1] = np.conj(Cbar[:, :, (n3 - i + 2) - 1])
    return idft_mode3(Cbar)


# --------------------------------------------------------------------------------------------
# Section 2.1: norms, inner product, error metric
# --------------------------------------------------------------------------------------------
def frobenius(A: np.ndarray) -> float:
    """||A||_F = sqrt(sum |a_ijk|^2)."""
    return float(np.sqrt(np.sum(np.abs(np.asarray(A, dtype=np.complex128)) ** 2)))


def inner(A: np.ndarray, B: np.ndarray) -> complex:
    """<A, B> = sum_i <A^(i), B^(i)> with <A, B> = Tr(A^* B)."""
    return complex(sum(np.trace(A[:, :, k].conj().T @ B[:, :, k]) for k in range(A.shape[2])))


def rel_err(X: np.ndarray, Ref: np.ndarray) -> float:
    """Parity metric (BASELINE.json north_star): ||X - Ref||_F / ||Ref||_F, evaluated in fp64.

    Both arguments must be real (the t-product of real tensors is real):
    a complex argument raises TypeError instead of being cast silently, so a caller holding
    ``tprod_alg1``'s complex result takes ``.real`` explicitly.  A zero reference returns the
    absolute error ||X||_F."""
    if np.iscomplexobj(X) or np.iscomplexobj(Ref):
        raise TypeError("rel_err takes real arrays; take .real of a complex oracle result explicitly")
    X = np.asarray(X, dtype=np.float64)
    Ref = np.asarray(Ref, dtype=np.float64)
    if X.shape != Ref.shape:
        raise ValueError(f"rel_err: shape mismatch {X.shape} vs {Ref.shape}")
    den = float(np.linalg.norm(Ref.ravel()))
    num = float(np.linalg.norm((X - Ref).ravel()))
    return num / den if den > 0 else num
