// Internal declarations shared by the libtprod.so translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace tprod {

// Number of frequency slices multiplied by Algorithm 1: ceil((n3+1)/2).
inline int64_t h_slices(int64_t n3) { return n3 / 2 + 1; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------------------ fp32 path data layout
// Split spectrum of a real p x q x n3 tensor X (Matlab layout, p fastest):
//   planes [f][s][q][ld] of __half, f < h, s in {Re_hi, Re_lo, Im_hi, Im_lo}, ld >= p, ld % 8 == 0
// value(f,p,q) = (hi + lo) * 2^-e  where e = scale exponent of p (A role) or q (B role).
// For A (p = i, q = l) this is an MN-major M x K operand; for B (p = l, q = j) a K-major N x K
// operand of the per-frequency GEMM.  C-bar is fp32 planes [f][re|im][j][ldc] (i fastest).
enum { PL_RE_HI = 0, PL_RE_LO = 1, PL_IM_HI = 2, PL_IM_LO = 3, NPLANES = 4 };

struct Twiddles32 {
  const float2* tw;              // tw[m] = (cos 2pi m/n3, sin 2pi m/n3)
  int n3;
  const float2* st = nullptr;    // Stockham per-pass twiddle table (FFT path only), see transforms_fft.cu
  int staged = 1;                // 0: skip the TMA-staged / tube kernels (TPROD_OPT_TRANSFORM = 1)
  int tc = 1;                    // tensor-core DFT-matrix kernels for n3 <= 64 (0: TPROD_OPT_TRANSFORM = 1, 2)
  int cluster = 0;               // one-pass cluster kernels for n3 = 4096 (TPROD_OPT_TRANSFORM = 3)
  // four-step long-tube forward (n3 = N1*N2 in {4096, 8192, 16384}): Stockham tables of the two
  // factors and a workspace the size of the larger operand
  const float2* st_n1 = nullptr;
  const float2* st_n2 = nullptr;
  float* scratch = nullptr;
  size_t scratch_bytes = 0;
};
struct Twiddles64 { const double2* tw; int n3; };

// K0: per-index max |x| as float bits (non-negative floats order like unsigned ints).
// role 0: max over (q,k) for every p;  role 1: max over (p,k) for every q.
void launch_absmax(const float* X, int64_t P, int64_t Q, int64_t n3, int role,
                   unsigned* maxbits, cudaStream_t s);
// Both operands in one vectorised launch (falls back to two launch_absmax calls if unaligned).
void launch_absmax2(const float* A, const float* B, int64_t n1, int64_t n2, int64_t n3, int64_t n4,
                    unsigned* maxA, unsigned* maxB, int num_sms, cudaStream_t s);

// K1: forward DFT (Hermitian half), exact power-of-two scaling 2^e, fp16 hi/lo split.  Also
// writes unscale[p] (role 0) or unscale[q] (role 1) = 2^-e, the exact factor the GEMM epilogue
// applies (one writer per index).
void launch_fwd_split(const float* X, int64_t P, int64_t Q, int64_t n3, int role,
                      const unsigned* maxbits, Twiddles32 tw, __half* out, int64_t ld,
                      float* unscale, int num_sms, cudaStream_t s);
// decode split planes back to fp32 planes [f][q][p] (stage test entry only)
void launch_decode_split(const __half* in, int64_t ld, int64_t P, int64_t Q, int64_t n3, int role,
                         const float* unscale, float* re, float* im, cudaStream_t s);

// K2 (reference SIMT engine): C-bar_f = A-bar_f B-bar_f on split operands, stored at the operands'
// exact scales (the inverse transform unscales per output tube, R18).
void launch_gemm_simt_split(const __half* Ab, int64_t lda, const __half* Bb, int64_t ldb,
                            float* Cb, int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h,
                            cudaStream_t s);

// K2 (tcgen05 engine).  Returns false if the shape/device is not supported by the kernel.
bool gemm_tc_supported();
// nyq = 1 if slice h-1 is a real Nyquist slice (n3 even): DC and Nyquist slices have exactly zero
// Im planes and run only the Ar.Br products.
// K2 -> K3 overlap (TPROD_OPT_OVERLAP): with `done` set, a CTA-pair GEMM of few tile
// rounds runs its tiles m-row by m-row and counts finished (m, n) output tiles in done[m * nt + n]
// (release: each CTA of the cluster adds 1 per frequency after its epilogue warps' stores, `target`
// in all); K3 is then launched as a programmatic dependent and each of its blocks waits (acquire) for
// the counter of the tile it reads, so the inverse of finished tiles runs on the SMs the GEMM's
// last partial round leaves idle.  `ov` is filled by the GEMM launch (used = false: no counters).
constexpr int OVERLAP_COUNTERS = 1024;   // (m, n) tile counters per handle
struct OverlapK3 {
  const int* done = nullptr;
  int target = 0;       // counter value of a finished (m, n) tile: h * 2 CM
  int pb_per_m = 1;     // 256-row K3 blocks per GEMM m tile (2 CM * 128 rows)
  int cols_per_n = 128; // GEMM N tile
  int nt = 0;           // GEMM n tiles
  bool used = false;
  // Streaming consumer (the tube inverse of n3 = 64, config 5): K3's CTAs take their items from
  // the work counter `work` in the GEMM's tile-completion order, so the overlap holds over any
  // number of tile rounds (set by the caller before the GEMM launch; `work` by the GEMM launch).
  bool stream = false;
  int* work = nullptr;
};
int launch_gemm_tc_split(const __half* Ab, int64_t lda, const __half* Bb, int64_t ldb,
                         float* Cb, int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h,
                         int nyq, int force_bn, int force_cn,
                         int num_sms, cudaStream_t s, int* done = nullptr, OverlapK3* ov = nullptr);

// K3: fused conjugate fill + inverse DFT, C-bar planes [f][re|im][q][ld] -> real X (p x q x n3).
// Cre/Cim: first planes; slice f at Cre + f*fstride (production: fstride = 2*Q*ld).  Output tube
// (p, q) is multiplied by urow[p] * ucol[q] (exact powers of two or 0; nullptr = 1) after the
// inverse FFT (R18: the t-product's C-bar arrives at the operands' scales).
struct OutUnscale {
  const float* row = nullptr;
  const float* col = nullptr;
};
void launch_inv_f32(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P,
                    int64_t Q, int64_t n3, Twiddles32 tw, OutUnscale u, float* X, int num_sms, cudaStream_t s,
                    OverlapK3* ov = nullptr);

// TMA-staged persistent dense transforms for n3 <= 64 (transforms_tma.cu); false = not handled
// (unaligned shapes fall back to the register kernels of transforms_dense.cu).  The inverse
// requires C-bar in the production layout (Cim = Cre + Q*ld, slice pitch 2*Q*ld).
bool launch_fwd_tma(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s);

// Tube-parallel TMA-staged Stockham transforms for power-of-two 32 <= n3 <= 256 (transforms_tma.cu);
// `st` = Stockham table of host_stockham_table.  false = not handled.  The inverse requires C-bar
// in the production layout (Cim = Cre + Q*ld, slice pitch 2*Q*ld).
bool tube_supported(int64_t n3);
// Four-step two-pass forward for long power-of-two tubes (transforms_tma.cu); false = not handled.
void fourstep_factors(int64_t n3, int* n1, int* n2);
bool launch_fwd_4step(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                      const Twiddles32& tw, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s);
// inverse: C-bar in the production layout (Cim = Cre + Q*ld, slice pitch 2*Q*ld)
bool launch_inv_4step(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const Twiddles32& tw,
                      OutUnscale u, float* X, int num_sms, cudaStream_t s);
// One-pass long-tube transforms for n3 = 4096 on 8-CTA clusters (transforms_cluster.cu): the
// four-step intermediate stays in distributed shared memory.  Same arguments and results as the
// four-step launchers; false = not handled (then the four-step kernels run).
bool cluster_fft_supported(int64_t n3);
bool launch_fwd_cluster(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                        const float2* tw, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s);
bool launch_inv_cluster(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const float2* tw,
                        OutUnscale u, float* X, int num_sms, cudaStream_t s);

bool launch_fwd_tube(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                     const float2* st, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s);
bool launch_inv_tube(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const float2* st,
                     OutUnscale u, float* X, int num_sms, cudaStream_t s, OverlapK3* ov = nullptr);
// the shapes whose K3 is the streaming tube inverse (OverlapK3::stream)
bool inv_tube_stream_ok(int64_t P, int64_t n3, int64_t ld, const float* X);

// ------------------------------------------------------------------ NEXT-4 (tensor_ops.cu)
template <typename T>
void launch_tran(const T* A, T* At, int64_t n1, int64_t n2, int64_t n3, cudaStream_t s);
template <typename T>
int launch_teye(T* I, int64_t n, int64_t n3, cudaStream_t s);
bool tinv_supported(int64_t n);
int launch_slice_inverse(const float* re, const float* im, float* xre, float* xim, int64_t n, int64_t h,
                         int64_t fstride, float rtol, const unsigned* maxp, int* singular, cudaStream_t s);
void launch_absmax_planes(const float* re, const float* im, int64_t count, unsigned* out, cudaStream_t s);
// n > 96: Gauss-Jordan in global memory (fp64), workspace gj_workspace_bytes(n, h)
size_t gj_workspace_bytes(int64_t n, int64_t h);
int launch_slice_inverse_large(const float* re, const float* im, float* xre, float* xim, int64_t n, int64_t h,
                               int64_t fstride, float rtol, const unsigned* maxp, int* singular, void* ws,
                               cudaStream_t s);
bool svt_supported(int64_t m, int64_t n);
int launch_slice_svt(const float* re, const float* im, float* wre, float* wim, int64_t m, int64_t n, int64_t h,
                     int64_t fstride, float tau, int* status, cudaStream_t s);
int launch_slice_svd_factors(const float* re, const float* im, int64_t m, int64_t n, int64_t h, int64_t fstride,
                             float* ure, float* uim, float* sre, float* vre, float* vim, int* status, cudaStream_t s);
// Blocked one-sided Jacobi of every spectral slice (tsvt_block.cu), any slice size.  BJ_SVT: t-SVT
// with threshold tau into wre / wim (planes [f][col][row] of the m x n slice, pitch fstride);
// BJ_VALUES: the singular values of every slice, non-increasing, into sv ([h][min(m, n)]);
// BJ_FACTORS: skinny factors into ure/uim ([h][r][m]), sre ([h][r][r], real), vre/vim ([h][r][n]);
// BJ_FACTORS_FULL: full factors, ure/uim [h][m][m], sre [h][n][m] (f-diagonal), vre/vim [h][n][n].
// `status` (device int) gets STATUS_NOCONV or-ed in when a slice hits the sweep cap.
constexpr int STATUS_SINGULAR = 1, STATUS_NOCONV = 2;
enum { BJ_SVT = 0, BJ_VALUES = 1, BJ_FACTORS = 2, BJ_FACTORS_FULL = 3 };
struct BjOut {
  float tau;
  float *wre, *wim;                  // BJ_SVT
  double* sv;                        // BJ_VALUES
  float *ure, *uim, *sre, *vre, *vim;  // BJ_FACTORS
};
size_t bj_workspace_bytes(int64_t m, int64_t n, int64_t h, bool full = false);
int launch_block_svd(const float* re, const float* im, int64_t m, int64_t n, int64_t h, int64_t fstride, int mode,
                     BjOut o, void* ws, int* status, cudaStream_t s);
// t-SVD scalars from per-slice singular values sv ([h][r], non-increasing), any r (tsvt_block.cu)
int launch_tsvd_reduce(const double* sv, int64_t r, int64_t h, int64_t n3, float rtol, float* out, cudaStream_t s);
int launch_tsvd_values(const float* re, const float* im, int64_t m, int64_t n, int64_t h, int64_t n3, int64_t fstride,
                       double* sv, float rtol, float* out, int* status, cudaStream_t s);

// ------------------------------------------------------------------ fp64 path
// spectra as fp64 planes [f][re|im][q][ld]
void launch_fwd_f64(const double* X, int64_t P, int64_t Q, int64_t n3, Twiddles64 tw,
                    double* out, int64_t ld, cudaStream_t s);
void launch_gemm_simt_f64(const double* Ab, int64_t lda, const double* Bb, int64_t ldb,
                          double* Cb, int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h,
                          cudaStream_t s);
void launch_inv_f64(const double* Cb, int64_t ld, int64_t P, int64_t Q, int64_t n3, Twiddles64 tw,
                    double* X, cudaStream_t s);
// In-smem mixed-radix fp64 FFT transforms (transforms_f64.cu) for 2 <= n3 <= 8192 (5-smooth, or
// Bluestein through a 5-smooth length <= 8192); launch_fwd_f64 / launch_inv_f64 take them first.
// fft64_prepare builds (and caches per device) the tables of n3 outside any stream capture.
bool fft64_prepare(int64_t n3);
bool launch_fwd_fft64(const double* X, int64_t P, int64_t Q, int64_t n3, double* out, int64_t ld, cudaStream_t s);
bool launch_inv_fft64(const double* Cb, int64_t ld, int64_t P, int64_t Q, int64_t n3, double* X, cudaStream_t s);

// Tensor-core (tcgen05) DFT-matrix transforms for 2 <= n3 <= 64 (transforms_tc.cu); false = not
// handled (P % 4 != 0, unaligned pointers).  The inverse requires C-bar in the production layout.
bool dft_tc_supported(int64_t n3);
bool launch_fwd_dft_tc(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                       __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s);
bool launch_inv_dft_tc(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, OutUnscale u, float* X,
                       int num_sms, cudaStream_t s);

// Register-resident dense transforms for n3 <= 64 (transforms_dense.cu); false = not handled.
bool dense_supported(int64_t n3);
bool launch_fwd_dense(const float* X, int64_t P, int64_t Q, int64_t n3, int role,
                      const unsigned* maxbits, __half* out, int64_t ld, float* unscale,
                      cudaStream_t s);
bool launch_inv_dense(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P,
                      int64_t Q, int64_t n3, OutUnscale u, float* X, cudaStream_t s,
                      OverlapK3* ov = nullptr);
// K1 of B with K0 of B fused (n3 <= 32, P = n2 even and <= 2048, 8-byte aligned): the column scales
// are reduced per lateral slice by a thread-block cluster inside the transform (no maxB pass).
bool fwd_colmax_ok(const float* X, int64_t P, int64_t n3);
bool launch_fwd_dense_colmax(const float* X, int64_t P, int64_t Q, int64_t n3, __half* out, int64_t ld,
                             float* unscale, cudaStream_t s);
// true if launch_inv_dense takes the tube-pair kernel for this n3 (the one that honours OverlapK3)
bool inv_dense_pair_ok(int64_t n3);

// In-smem mixed-radix (16/8/4/2, 3, 5) Stockham FFT transforms for 5-smooth 64 < n3 <= 16384
// (transforms_fft.cu).
// `st` is the Stockham table of host_stockham_table (device copy).
bool fft_supported(int64_t n3);
// Not 5-smooth 64 < n3 <= 8192: Bluestein's chirp-z through a 5-smooth FFT of length >= 2 n3 - 1
// (launch_fwd_fft / launch_inv_fft take that route themselves; `st` may then be null).
bool bluestein_supported(int64_t n3);
bool launch_fwd_fft(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    const float2* st, __half* out, int64_t ld, float* unscale, cudaStream_t s);
bool launch_inv_fft(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P, int64_t Q,
                    int64_t n3, const float2* st, OutUnscale u, float* X, cudaStream_t s);
// Per-pass twiddles of the mixed-radix Stockham FFT, laid out [pass][r-1][k] so that a warp's
// lookups are coalesced: entry (r, k) of the pass with span Ns and radix R is
// (cos, sin)(2 pi r k / (Ns R)), taken from the fp64 table cs (2n doubles) and rounded to fp32.
size_t stockham_table_len(int n);
void host_stockham_table(int n, const double* cs, float2* out);

// Host-side exact twiddle table: (cos, sin)(2 pi m / n), m = 0..n-1, computed in fp64 with exact
// quadrant reduction so that m = 0, n/4, n/2, 3n/4 give exactly 0 / +-1.
void host_twiddles(int n, double* cs /* 2n: cos,sin interleaved */);

}  // namespace tprod
