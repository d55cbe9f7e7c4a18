/*
 * tprod.h -- C ABI of the B200-native t-product library (libtprod.so).
 *
 * Operation (Definition 2.1, Eq. (9)):
 *     C = A * B = fold( bcirc(A) . unfold(B) ),   A: n1 x n2 x n3,  B: n2 x n4 x n3,  C: n1 x n4 x n3
 * computed the fast way of Algorithm 1: a mode-3 DFT of every tube
 * (Eq. (2); fft(.,[],3), L120-122), one complex matrix product per frequency slice
 * for the ceil((n3+1)/2) slices of the Hermitian half (Eq. (8); Alg. 1 step 2, L177),
 * and an inverse DFT (L124-126, Alg. 1 step 3, L179) with the conjugate fill of the remaining
 * slices fused into it (those slices are never materialised).
 *
 * Memory layout of every tensor argument (Matlab linearisation): element (i,j,k),
 * 0-based, lives at offset i + n1*j + n1*n2*k (in elements of the tensor's dtype).  A torch
 * tensor of shape (n1, n2, n3) with strides (1, n1, n1*n2) has exactly this layout.
 *
 * Ownership: all tensor pointers are caller-owned; the library never frees or retains them past
 * the call.  The handle owns its plan cache, DFT tables and workspace (device memory, grown on
 * demand, freed by tprod_destroy) and an optional NCCL communicator.  Workspace growth is stream
 * ordered (cudaMallocAsync / cudaFreeAsync on the call's stream): it never synchronises the device,
 * so a handle must be used from one stream at a time (or the caller orders the streams).
 *
 * Errors: every entry point returns an int status (0 = TPROD_OK).  Argument errors are detected
 * synchronously, BEFORE anything is enqueued.  Device-side faults of enqueued kernels surface at
 * the caller's next synchronisation of the stream.  tprod_strerror() maps a status to text.
 *
 * Threading: one handle must not be used concurrently from two host threads.  Calls are
 * asynchronous with respect to the host (stream-ordered) unless stated otherwise.
 *
 * Precision: tprod_f32 takes and returns IEEE fp32; its result matches the fp64 definition
 * within a relative Frobenius error of 1e-5 (BASELINE.json north_star).  Internally the
 * per-frequency products run on tcgen05 tensor cores with operands split into two fp16 terms
 * (hi + lo, three cross products, fp32 accumulation) after an exact power-of-two row/column
 * scaling; see DESIGN.md.  tprod_f64 computes in fp64 throughout (<= 1e-12).
 * Inputs must be finite; NaN/Inf inputs give unspecified output.
 */
#ifndef TPROD_H
#define TPROD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tprod_ctx* tprod_handle;

/* Status codes. */
enum {
  TPROD_OK = 0,
  TPROD_EINVAL = 1,        /* a dimension < 1, a NULL pointer, element-count overflow, bad handle */
  TPROD_EALIAS = 2,        /* C overlaps A or B (in-place is not supported) */
  TPROD_ENOMEM = 3,        /* workspace or table allocation failed */
  TPROD_ECUDA = 4,         /* a CUDA runtime / launch error */
  TPROD_ENCCL = 5,         /* NCCL missing or an NCCL call failed */
  TPROD_EUNSUPPORTED = 6,  /* no kernel for this shape / device (not sm_100) */
  TPROD_ENOWORLD = 7,      /* tprod_bcast_* called before tprod_set_world */
  TPROD_ESINGULAR = 8      /* tprod_tinv_f32: a spectral slice has no inverse to working precision */
};

/* dtype selectors for tprod_workspace_bytes */
enum { TPROD_DTYPE_F32 = 0, TPROD_DTYPE_F64 = 1 };

/* Create a handle bound to CUDA device `device` (an ordinal as seen by the process).
 * Fails with TPROD_EUNSUPPORTED if the device is not compute capability 10.0 (B200). */
int tprod_create(int device, tprod_handle* out);

/* Destroy a handle: synchronises its device, frees workspace/tables, destroys the NCCL comm. */
int tprod_destroy(tprod_handle h);

/* The t-product, fp32.  A: n1*n2*n3 floats, B: n2*n4*n3, C: n1*n4*n3, all DEVICE pointers on
 * h's device, Matlab layout (see top).  A and B are read-only; C is written entirely.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Enqueues the whole path on
 * `stream` and returns; no host synchronisation.  Multi-GPU: n4 is the rank's LOCAL number of
 * lateral slices and B / C are the rank's compact shard tensors; the call has
 * no collective.  Deterministic: bitwise identical output for identical inputs, and column j of C
 * does not depend on n4 (no split-K, fixed K order), so sharding is bitwise invariant. */
int tprod_f32(const float* A, const float* B, float* C,
              int64_t n1, int64_t n2, int64_t n3, int64_t n4,
              void* stream, tprod_handle h);

/* Prepared left operand (fixed A, many B -- the broadcast-once scenario).
 * tprod_prepare_a_f32 runs the A half of the path once -- the row scales (K0) and the forward
 * mode-3 DFT of A's Hermitian half in the split GEMM-operand format (Alg. 1 step 1)
 * -- into handle-owned device memory (8*h*n2*roundup(n1,8) + 4*n1 bytes, h = n3/2+1).  A is read
 * during the call only (asynchronously on `stream`) and not retained; re-prepare if it changes.
 * tprod_f32_prepared then computes C = A * B for the prepared A (n1 x n2 x n3) and B (n2 x n4 x n3),
 * C (n1 x n4 x n3), both DEVICE pointers in Matlab layout, running only K0/K1 of B, the GEMM and
 * the inverse.  The result is bitwise identical to tprod_f32(A, B, C, ...) (same kernels, same
 * operand values, same K order).  Errors: TPROD_EINVAL if nothing is prepared or an argument is
 * invalid, TPROD_EALIAS if C overlaps B, TPROD_ENOMEM.  tprod_release_a frees the prepared
 * operand (also done by tprod_destroy and by the next tprod_prepare_a_f32).  Calls on one handle are
 * stream-ordered: prepare on the stream of the later tprod_f32_prepared calls, or synchronise. */
int tprod_prepare_a_f32(const float* A, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h);
int tprod_f32_prepared(const float* B, float* C, int64_t n4, void* stream, tprod_handle h);
int tprod_release_a(tprod_handle h);

/* NEXT-4 companion operations, DEVICE pointers in Matlab layout, asynchronous on
 * `stream` unless stated otherwise.
 * tprod_tran_*: At = A^* (Definition 2.2): A n1 x n2 x n3 -> At n2 x n1 x n3 with
 *   At(:,:,0) = A(:,:,0)^T and At(:,:,k) = A(:,:,n3-k)^T (real data).  At must not overlap A.
 * tprod_teye_*: I = the n x n x n3 identity tensor (Definition 2.3).
 * tprod_tinv_f32: X = A^-1 (Definition 2.4, Eq. (11)), A and X n x n x n3,
 *   1 <= n <= 8192: forward DFT (production K1 kernels), a complex Gauss-Jordan inverse with partial
 *   pivoting per spectral slice f < h (n <= 96: one CTA per slice in shared memory, fp32; larger: the
 *   augmented slices in the workspace, 32 n^2 h bytes, fp64, two launches per pivot column), inverse
 *   DFT with the conjugate fill (production K3 kernels).  A slice is singular when a pivot falls to
 *   <= n * 2^-20 times the largest spectral entry (X is then unspecified).  With
 *   TPROD_OPT_SYNC_CHECKS = 1 (default) the call is SYNCHRONOUS (waits for `stream`) and returns
 *   TPROD_ESINGULAR; with 0 it is asynchronous and sets TPROD_STATUS_SINGULAR in the handle's status
 *   word (tprod_status).  TPROD_EUNSUPPORTED for n > 8192. */
int tprod_tran_f32(const float* A, float* At, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h);
int tprod_tran_f64(const double* A, double* At, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h);
int tprod_teye_f32(float* I, int64_t n, int64_t n3, void* stream, tprod_handle h);
int tprod_teye_f64(double* I, int64_t n, int64_t n3, void* stream, tprod_handle h);
int tprod_tinv_f32(const float* A, float* X, int64_t n, int64_t n3, void* stream, tprod_handle h);

/* NEXT-2: t-SVT, the proximal operator of tau * TNN (Algorithm 3, Eq. (19)-(21)).
 * Y, X: n1 x n2 x n3 DEVICE pointers in Matlab layout, n1, n2 >= 1, tau >= 0.  Forward DFT
 * (production K1 kernels, decoded to fp32), one-sided Jacobi SVD in fp64 + singular-value shrinkage
 * per spectral slice f < h (slices up to 64 x 64: one CTA per slice in shared memory, at most 40
 * sweeps; larger: a blocked Jacobi over column blocks of 32 with the slices in the workspace,
 * about 16 (m n + n^2) h bytes, m = max(n1, n2), n = min(n1, n2) <= 65535, at most 30 sweeps),
 * inverse DFT with the conjugate fill (production K3 kernels).  Asynchronous.  A slice still
 * rotating at the sweep cap sets TPROD_STATUS_NOCONVERGE in the handle's status word (tprod_status).
 * TPROD_EINVAL for tau < 0 or NaN, TPROD_ENOMEM if the workspace does not fit. */
int tprod_tsvt_f32(const float* Y, float* X, int64_t n1, int64_t n2, int64_t n3, float tau, void* stream,
                   tprod_handle h);

/* NEXT-3: t-SVD scalars (Theorem 2.2 / Algorithm 2 step 2, Eq. (13)-(18)) of a
 * DEVICE n1 x n2 x n3 tensor A (Matlab layout, any slice size as tprod_tsvt_f32).  Writes to the DEVICE array
 * `out` (r + 3 floats, r = min(n1, n2)): out[0..r) = the singular values S(i,i,1) of A (Eq. (14),
 * non-increasing), out[r] = TNN (Def. 2.9), out[r+1] = TSN = ||bcirc(A)||_2 (Def. 2.8),
 * out[r+2] = tubal rank #{i : S(i,i,1) > rtol * S(1,1,1)} (Eq. (16)).  Same transforms and per-slice
 * Jacobi SVD (fp64) as tprod_tsvt_f32.  Asynchronous. */
int tprod_tsvd_values_f32(const float* A, int64_t n1, int64_t n2, int64_t n3, float rtol, float* out, void* stream,
                          tprod_handle h);
/* Skinny t-SVD factors (Algorithm 2, Theorem 2.2 Eq. (12); R17): A = U * S * V^* with
 * U n1 x r x n3, S r x r x n3 (f-diagonal), V n2 x r x n3, r = min(n1, n2), all DEVICE pointers in
 * Matlab layout, any slice size as tprod_tsvt_f32.  Per spectral slice f < h the Jacobi SVD's
 * factors (columns in non-increasing singular-value order), conjugate fill and inverse DFT of each
 * factor.  Singular vectors are unique up to a unit phase per column and slice (S is unique); a
 * left vector whose singular value is <= 1e-6 of the slice's largest is replaced by a unit vector
 * Gram-Schmidt-orthogonalised against the others, so U^* U = I holds for rank-deficient A too.
 * Asynchronous; non-convergence as tprod_tsvt_f32. */
int tprod_tsvd_f32(const float* A, float* U, float* S, float* V, int64_t n1, int64_t n2, int64_t n3, void* stream,
                   tprod_handle h);
/* Full t-SVD (Theorem 2.2 in its stated shapes, Eq. (12)): A = U * S * V^* with
 * U n1 x n1 x n3 and V n2 x n2 x n3 orthogonal (U^* U = U U^* = I) and S n1 x n2 x n3 f-diagonal, all
 * DEVICE pointers in Matlab layout, max(n1, n2) <= 65535.  Per spectral slice f < h the blocked
 * Jacobi SVD (any size) with the left basis of the processed slice completed to max(n1, n2)
 * orthonormal columns (the unit vector of the least-covered row, Gram-Schmidt twice, fp64); the
 * self-conjugate slices are taken as exactly real (Eq. (8), R19).  Columns follow
 * non-increasing singular values; the null-space columns are one valid orthonormal completion.
 * Workspace about 16 (m^2 + n^2) h bytes (m = max, n = min(n1, n2)).  Asynchronous;
 * non-convergence as tprod_tsvt_f32. */
int tprod_tsvd_full_f32(const float* A, float* U, float* S, float* V, int64_t n1, int64_t n2, int64_t n3,
                        void* stream, tprod_handle h);

/* Same in fp64 (all arithmetic fp64). */
int tprod_f64(const double* A, const double* B, double* C,
              int64_t n1, int64_t n2, int64_t n3, int64_t n4,
              void* stream, tprod_handle h);

/* End-to-end variants with HOST pointers (pinned memory recommended): copies A and B to device
 * buffers owned by the handle, runs tprod_*, copies C back, and synchronises `stream` before
 * returning (so C_host is valid on return).  Same layout and errors as above. */
int tprod_f32_host(const float* A_host, const float* B_host, float* C_host,
                   int64_t n1, int64_t n2, int64_t n3, int64_t n4,
                   void* stream, tprod_handle h);
int tprod_f64_host(const double* A_host, const double* B_host, double* C_host,
                   int64_t n1, int64_t n2, int64_t n3, int64_t n4,
                   void* stream, tprod_handle h);

/* Bytes of device workspace the handle needs for this shape (half-spectra of A, B, C plus
 * scale vectors; DFT tables excluded).  Pure function, no device access. */
int tprod_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t n4, int dtype, size_t* out);

/* Human-readable text for a status code (static storage, never NULL). */
const char* tprod_strerror(int status);

/* Number of kernel launches enqueued by the most recent tprod_* call on this handle. */
int tprod_last_launch_count(tprod_handle h, int64_t* out);

/* ---------------------------------------------------------------- multi-GPU (one process/GPU)
 * The NCCL library is the process's libnccl.so.2 (the one torch already loaded), opened with
 * dlopen at first use.  tprod_nccl_unique_id writes the 128-byte ncclUniqueId on one rank; the
 * caller exchanges it (e.g. through a torch.distributed process group) and every rank calls
 * tprod_set_world with the same bytes.  tprod_bcast_* broadcasts a device buffer in place from
 * `root` (ncclBroadcast over NVLink/NVSwitch): it is the one-time replication of A, a setup step
 * that tprod_f32/tprod_f64 never call. */
int tprod_nccl_unique_id(void* out_128_bytes);
int tprod_set_world(tprod_handle h, int rank, int world, const void* unique_id_128_bytes);
int tprod_bcast_f32(tprod_handle h, float* buf, int64_t count, int root, void* stream);
int tprod_bcast_f64(tprod_handle h, double* buf, int64_t count, int root, void* stream);

/* ---------------------------------------------------------------- stage entry points (tests)
 * Forward mode-3 DFT of a real X (p x q x n3, Matlab layout, device) on the Hermitian half
 * f = 0..h-1 (h = ceil((n3+1)/2)), written as fp32 planes Xre, Xim of layout [f][q][p]
 * (h*p*q floats each, device).  `role` 0 runs the A-operand transform (row scale on p), role 1
 * the B-operand transform (column scale on q); the production kernels run and their split fp16
 * planes are decoded back to fp32, so the result carries the production rounding. */
int tprod_dft_f32(const float* X, float* Xre, float* Xim, int64_t p, int64_t q, int64_t n3,
                  int role, void* stream, tprod_handle h);
/* Inverse with the fused conjugate fill (Alg. 1 steps 2b-3): planes [f][q][p] -> real X. */
int tprod_idft_f32(const float* Xre, const float* Xim, float* X, int64_t p, int64_t q, int64_t n3,
                   void* stream, tprod_handle h);

/* Options (tests / benchmarking).  TPROD_OPT_ENGINE: 0 = auto (tcgen05), 1 = SIMT reference
 * GEMM (a slower second GEMM on the same split operands; used to cross-check the tcgen05
 * kernel).  TPROD_OPT_GEMM_BN: force the tcgen05 N tile (0 = auto, else 64 or 128). */
enum { TPROD_OPT_ENGINE = 1, TPROD_OPT_GEMM_BN = 2, TPROD_OPT_TIMING = 3, TPROD_OPT_GEMM_CLUSTER = 4,
       TPROD_OPT_TRANSFORM = 5, TPROD_OPT_GRAPHS = 6, TPROD_OPT_POISON = 7, TPROD_OPT_SYNC_CHECKS = 8,
       TPROD_OPT_OVERLAP = 9, TPROD_OPT_FUSED_SCALES = 10 };
/* TPROD_OPT_FUSED_SCALES (tprod_f32 / tprod_f32_prepared): 1 (default) = for n3 <= 32 with n2 even and
 * <= 2048 and B of at most 8M elements (where it measured faster), B's column scales (the K0 reduction max |B(:, j, :)|) are computed inside B's forward
 * transform -- the blocks of one lateral slice form a thread-block cluster and exchange their partial
 * maxima through distributed shared memory -- so B is read once instead of twice; 0 = a separate K0
 * pass over B.  The same maxima either way: bitwise identical results. */
/* TPROD_OPT_OVERLAP (tprod_f32 / tprod_f32_prepared): 1 (default) = when the per-frequency GEMM runs on
 * CTA pairs in 2..8 tile rounds and K3 is the tube-pair register kernel (n3 <= 32), the GEMM takes
 * its tiles m-row by m-row (frequencies inside a row) and counts finished (m, n) output tiles in a device array of the
 * handle, and K3 is launched as a programmatic dependent whose blocks each wait for the tile they
 * read: the inverse of finished tiles runs on the SMs the GEMM's last round leaves idle (Alg. 1
 * steps 2-3 overlapped).  With n3 = 64 (K3 = the TMA tube inverse; config 5) the same
 * holds for a GEMM of any number of tile rounds: K3's CTAs take their work items from a device
 * counter in the GEMM's tile-completion order (m-row by m-row), so the inverse of one m-row runs on
 * the SMs the cluster grid leaves idle while the GEMM works on the next (config 5, same box, arms
 * alternated: 95.2 -> 94.0 ms per step).  2 = as 1 without that many-round case (measurement).
 * 0 = K3 strictly after the GEMM.  Bitwise identical results in every setting. */
/* TPROD_OPT_SYNC_CHECKS: 1 (default) = tprod_tinv_f32 waits for its stream and returns
 * TPROD_ESINGULAR for a singular tensor; 0 = it returns at once and reports singularity through
 * the status word (tprod_status). */
/* TPROD_OPT_POISON: 1 = before every call the handle fills the workspace it will use (and a prepared
 * operand's buffers) with 0xFF bytes -- NaN in fp16 / fp32 / fp64 -- on the call's stream, so that any
 * kernel reading workspace it has not written first turns the result into NaN (a test-time stand-in
 * for compute-sanitizer's initcheck).  Results are unchanged when the kernels are correct. */
/* TPROD_OPT_GRAPHS (tprod_f32 / tprod_f64 / tprod_f32_prepared): 1 (default) = the second and later
 * calls with the same operand pointers, shapes and options replay the call's launch sequence as
 * one CUDA graph (captured on a private stream at the second call, launched on the caller's
 * stream); 0 = always launch kernel by kernel.  Identical kernels and results either way; the
 * graph only removes per-kernel host work and launch gaps.  Bypassed while TPROD_OPT_TIMING is on
 * (stage events between direct launches) and when the caller's stream is being captured.  The
 * handle keeps at most 64 graphs (all are dropped when a 65th key arrives or the workspace grows;
 * an executable graph still in flight is released by the driver when it completes). */
/* TPROD_OPT_TRANSFORM (fp32 path): 0 = auto (the TMA-staged / tube-parallel / four-step transform
 * kernels where they apply, else the register-resident / mixed-radix / generic ones), 1 =
 * register-resident and generic transform kernels only, 2 = for 2 <= n3 <= 64 the tensor-core
 * DFT-matrix kernels (Eq. (2) as a tcgen05 3xTF32 contraction, transforms_tc.cu; measured slower
 * than auto on B200), else auto, 3 = auto except that n3 = 4096 takes the one-pass
 * 8-CTA cluster kernels (transforms_cluster.cu: the four-step intermediate kept in distributed shared
 * memory) instead of the two-pass four-step kernels.  Same result up to the rounding of the DFT sums
 * (all within the stage tolerances). */
/* TPROD_OPT_GEMM_CLUSTER: 0 = auto, 1 = independent CTAs, 2 = 2-CTA clusters along N sharing the
 * A tile by TMA multicast, 3 = CTA pairs issuing tcgen05.mma.cta_group::2 (256 x 128 tiles over two
 * SMs; requires the 128 N tile), 4 = 4-CTA clusters of two such pairs stacked along M sharing the B
 * tile by TMA multicast (512 x 128 cluster tiles).  None of the options changes the arithmetic (results are bitwise
 * identical for every option value except TPROD_OPT_ENGINE). */
int tprod_set_option(tprod_handle h, int option, int64_t value);

/* With TPROD_OPT_TIMING = 1, tprod_f32 records CUDA events on its stream between the stages of
 * the path; this returns the durations (ms) of the most recent call's stages, in order
 * [K0 scales, K1 forward DFTs, K2 per-frequency GEMMs, K3 inverse DFT], synchronising on the
 * last event.  When the call ran the A chain (K0 + K1 of A) concurrently with the B chain (operands
 * of at most 256M elements, no prepared A), the first entry covers K0 and K1 of both operands and
 * the second is exactly 0; when K3 ran overlapped with the GEMM (TPROD_OPT_OVERLAP), the third entry
 * covers K2 and K3 and the fourth is exactly 0.  `out` must hold 4 floats.  TPROD_EINVAL if timing was off for that
 * call. */
int tprod_last_stage_ms(tprod_handle h, float* out);

/* Status word of the handle: an OR of the TPROD_STATUS_* bits raised on the device by the handle's
 * kernels since the previous tprod_status call.  Enqueues a read and a clear of the word on
 * `stream`, waits for `stream`, and writes the bits to *bits (host).  Call it after the work to
 * check was enqueued on `stream` (or after synchronising the other streams that ran it). */
enum { TPROD_STATUS_SINGULAR = 1,     /* tprod_tinv_f32 with TPROD_OPT_SYNC_CHECKS = 0: singular */
       TPROD_STATUS_NOCONVERGE = 2 }; /* t-SVT / t-SVD: a spectral slice reached the sweep cap */
int tprod_status(tprod_handle h, void* stream, int* bits);

#ifdef __cplusplus
}
#endif
#endif /* TPROD_H */
