// NEXT-2 / NEXT-3 for slices larger than 64 x 64: the spectral step of t-SVT (Algorithm 3 step 2,
// PAPER.md:L290-296) and of the t-SVD scalars (Eq. (14)) by a BLOCKED one-sided (Hestenes) Jacobi
// SVD of every spectral slice f < h, in fp64, with the data in global memory.
//
// The slice (m x n complex, n <= m after taking the conjugate transpose of a wide slice) is split
// into column blocks of B = 32.  A sweep is a round-robin over block pairs (nb' - 1 rounds, nb'
// even); in one round every block pair (P, Q) of every slice is handled by one CTA:
//   1. G = X_S^H X_S, the 64 x 64 Gram matrix of the pair's columns S = P u Q (rows of X streamed
//      through shared memory);
//   2. one or two cyclic sweeps of two-sided Jacobi on G in shared memory (the one-sided rotation of
//      columns p, q is determined by alpha = G_pp, beta = G_qq, gamma = G_pq = x_p^H x_q),
//      accumulating the unitary R = J_1 J_2 ... (64 x 64);
//   3. X_S <- X_S R and V_S <- V_S R (rows streamed through shared memory).
// Because X itself is updated (not only G), every visit recomputes G from the current columns:
// this is the standard block one-sided Jacobi, accurate to the fp64 rounding of X (the Gram matrix
// only picks the rotations).  A slice is converged when a whole sweep made no rotation above the
// tolerance |gamma| <= 1e-8 sqrt(alpha beta) (the spectra in are fp32, ~1e-7 accurate); later
// launches return at once for it.  Then sigma_j = ||x_j|| and
//   t-SVT:          W = X diag((1 - tau / sigma_j)_+) V^H          (X = A V = U Sigma)
//   t-SVD scalars:  the sigma_j themselves.
#include "internal.h"
#include "common.cuh"

#include <algorithm>
#include <cstdio>
#include <vector>

namespace tprod {

namespace {

constexpr int BJ = 32;              // columns per block
constexpr int BS = 2 * BJ;          // columns of a block pair
constexpr int BJ_THREADS = 256;
constexpr int ROWS = 16;            // rows per streamed tile
constexpr int LP = BS + 1;          // padded shared-memory pitch (double2)
constexpr int MAX_SWEEPS = 30;

__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cmuld(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Circle method: player np - 1 fixed, pair k of round r = ((r + k) mod (np - 1), (r - k) mod (np - 1)),
// pair 0 = (r, np - 1).
__host__ __device__ inline void circle_pair(int np, int r, int k, int* p, int* q) {
  int a = r + k, b = r - k + np - 1;
  if (a >= np - 1) a -= np - 1;
  if (b >= np - 1) b -= np - 1;
  if (k == 0) b = np - 1;
  *p = a;
  *q = b;
}

// X (slice f at X + f * xs, column j at + j * m) from the fp32 spectral planes re / im [f][col][row]
// (m_in x n_in per slice, slice pitch fstride); tr = conjugate transpose.  V = I.
__global__ void bj_init_kernel(const float* __restrict__ re, const float* __restrict__ im, int64_t fstride, int m_in,
                               int n_in, int tr, double2* __restrict__ X, double2* __restrict__ V, int m, int n,
                               int64_t xs, int64_t vs) {
  const int f = blockIdx.y;
  const float* ar = re + (int64_t)f * fstride;
  const float* ai = im + (int64_t)f * fstride;
  double2* x = X + (int64_t)f * xs;
  double2* v = V + (int64_t)f * vs;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)m * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / m), i = (int)(idx - (int64_t)j * m);
    if (!tr) x[idx] = make_double2(ar[(int64_t)j * m_in + i], ai[(int64_t)j * m_in + i]);
    else x[idx] = make_double2(ar[(int64_t)i * m_in + j], -ai[(int64_t)i * m_in + j]);   // conj(Y(j, i))
  }
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x)
    v[idx] = make_double2(idx / n == idx % n ? 1.0 : 0.0, 0.0);
}

// One round of one sweep: CTA (pair k, slice f).  flags[f * MAX_SWEEPS + sweep] is set when a
// rotation above the tolerance happened; a slice whose previous sweep made none is done.
__global__ void __launch_bounds__(BJ_THREADS) bj_round_kernel(double2* __restrict__ X, double2* __restrict__ V, int m,
                                                             int n, int64_t xs, int64_t vs, int nbp, int round,
                                                             int sweep, int* __restrict__ flags) {
  extern __shared__ double2 sm[];
  double2* G = sm;                     // [BS][LP], column c at G + c * LP (padded pitch: no bank conflicts)
  double2* R = G + BS * LP;            // [BS][LP]
  double2* T = R + BS * LP;            // [ROWS][LP] row tile, row rr at T + rr * LP
  __shared__ int cols[BS];             // global column of local column c (-1: none)
  __shared__ double prm[BS / 2][4];    // per pair of the inner round: c, s, er, ei
  __shared__ int any_rot;
  const int f = blockIdx.y, tid = threadIdx.x;
  if (sweep > 0 && flags[f * MAX_SWEEPS + sweep - 1] == 0) return;
  int P, Q;
  circle_pair(nbp, round, blockIdx.x, &P, &Q);
  double2* x = X + (int64_t)f * xs;
  double2* v = V + (int64_t)f * vs;
  if (tid < BS) {
    const int blk = tid < BJ ? P : Q, c = blk * BJ + (tid % BJ);
    cols[tid] = c < n ? c : -1;
  }
  for (int idx = tid; idx < BS * BS; idx += BJ_THREADS) {
    const int c = idx / BS, r = idx % BS;
    R[c * LP + r] = make_double2(c == r ? 1.0 : 0.0, 0.0);
  }
  if (tid == 0) any_rot = 0;
  __syncthreads();
  // a ROWS x BS tile of rows r0.. of the pair's columns of M (rows of a column are contiguous in
  // global memory: consecutive threads take consecutive rows)
  auto load_tile = [&](const double2* M, int rows, int r0) {
    for (int idx = tid; idx < ROWS * BS; idx += BJ_THREADS) {
      const int c = idx / ROWS, rr = idx % ROWS, i = r0 + rr;
      T[rr * LP + c] = (i < rows && cols[c] >= 0) ? M[(int64_t)cols[c] * rows + i] : make_double2(0.0, 0.0);
    }
  };
  // ---- 1. G = X_S^H X_S: thread (a0, b0) owns the 4 x 4 entries (a0 + 16 i, b0 + 16 j)
  {
    const int a0 = tid % 16, b0 = tid / 16;
    double2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
    for (int r0 = 0; r0 < m; r0 += ROWS) {
      __syncthreads();
      load_tile(x, m, r0);
      __syncthreads();
#pragma unroll 2
      for (int rr = 0; rr < ROWS; ++rr) {
        double2 ta[4], tb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ta[i] = T[rr * LP + a0 + 16 * i];
          tb[i] = T[rr * LP + b0 + 16 * i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double2 p = cmulc(ta[i], tb[j]);
            acc[i][j].x += p.x;
            acc[i][j].y += p.y;
          }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) G[(b0 + 16 * j) * LP + a0 + 16 * i] = acc[i][j];   // (row a, column b) = x_a^H x_b
    __syncthreads();
  }
  // ---- 2. two-sided Jacobi on G (rotations of column pairs), R accumulates.  One inner sweep per
  // visit is the classic block Jacobi (the outer sweeps repeat the pairs until nothing rotates);
  // a second one when the first rotated keeps the block nearly orthogonal for the next visit.
  for (int isw = 0; isw < 2; ++isw) {
    __shared__ int rotated;
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int rr = 0; rr < BS - 1; ++rr) {
      if (tid < BS / 2) {
        int p, q;
        circle_pair(BS, rr, tid, &p, &q);
        const double al = G[p * LP + p].x, be = G[q * LP + q].x;
        const double2 g = G[q * LP + p];                 // x_p^H x_q
        const double g2 = g.x * g.x + g.y * g.y;
        double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
        // rotate while |gamma| > 1e-8 sqrt(alpha beta): the spectra in are fp32 (~1e-7 accurate), so
        // columns orthogonal to 1e-8 are orthogonal to working precision
        if (g2 > 1e-16 * al * be && g2 > 0.0) {
          rotated = 1;
          any_rot = 1;
          // fp64 division / square root are slow: 1/|g| and c = 1/sqrt(1+t^2) from fp32 estimates with
          // one fp64 Newton step (exact to ~1e-14: the rotation stays unitary), the angle from fp32
          // (an approximate Jacobi angle still converges); a subnormal fp32 g2 takes the fp64 route
          double ig;
          if (g2 > 1e-36) {
            const float ig32 = rsqrtf((float)g2);
            ig = (double)ig32 * (1.5 - 0.5 * g2 * (double)ig32 * (double)ig32);
          } else {
            ig = 1.0 / sqrt(g2);
          }
          const float zeta = (float)((be - al) * 0.5 * ig);
          const double t = copysignf(1.f, zeta) / (fabsf(zeta) + sqrtf(1.f + zeta * zeta));
          const double t2p1 = 1.0 + t * t;
          const float c32 = rsqrtf((float)t2p1);
          c = (double)c32 * (1.5 - 0.5 * t2p1 * (double)c32 * (double)c32);
          s = c * t;
          er = g.x * ig;
          ei = -g.y * ig;                                 // e = conj(g) / |g|
        }
        prm[tid][0] = c;
        prm[tid][1] = s;
        prm[tid][2] = er;
        prm[tid][3] = ei;
      }
      __syncthreads();
      // columns p, q of G and R:  new_p = c x_p - s e x_q,  new_q = s x_p + c e x_q
      for (int idx = tid; idx < (BS / 2) * BS * 2; idx += BJ_THREADS) {
        const int k = idx / (2 * BS), rem = idx % (2 * BS), row = rem % BS;
        double2* M = rem < BS ? G : R;
        int p, q;
        circle_pair(BS, rr, k, &p, &q);
        const double c = prm[k][0], s = prm[k][1];
        const double2 e = make_double2(prm[k][2], prm[k][3]);
        if (s == 0.0 && e.x == 1.0 && e.y == 0.0) continue;
        const double2 xp = M[p * LP + row], xq = cmuld(e, M[q * LP + row]);
        M[p * LP + row] = make_double2(c * xp.x - s * xq.x, c * xp.y - s * xq.y);
        M[q * LP + row] = make_double2(s * xp.x + c * xq.x, s * xp.y + c * xq.y);
      }
      __syncthreads();
      // rows p, q of G (G <- J^H G):  new_p = c g_p - s conj(e) g_q,  new_q = s g_p + c conj(e) g_q
      for (int idx = tid; idx < (BS / 2) * BS; idx += BJ_THREADS) {
        const int k = idx / BS, col = idx % BS;
        int p, q;
        circle_pair(BS, rr, k, &p, &q);
        const double c = prm[k][0], s = prm[k][1];
        const double2 ec = make_double2(prm[k][2], -prm[k][3]);
        if (s == 0.0 && ec.x == 1.0 && ec.y == 0.0) continue;
        const double2 gp = G[col * LP + p], gq = cmuld(ec, G[col * LP + q]);
        G[col * LP + p] = make_double2(c * gp.x - s * gq.x, c * gp.y - s * gq.y);
        G[col * LP + q] = make_double2(s * gp.x + c * gq.x, s * gp.y + c * gq.y);
      }
      __syncthreads();
    }
    if (!rotated) break;
  }
  if (tid == 0 && any_rot) flags[f * MAX_SWEEPS + sweep] = 1;
  // ---- 3. X_S <- X_S R, V_S <- V_S R, rows streamed through T; thread (rr, c0) writes row rr of
  // columns c0 + 16 u (16 consecutive rows of a column per half-warp: coalesced stores)
  {
    const int rr = tid % ROWS, c0 = tid / ROWS;
    for (int pass = 0; pass < 2; ++pass) {
      double2* M = pass == 0 ? x : v;
      const int rows = pass == 0 ? m : n;
      for (int r0 = 0; r0 < rows; r0 += ROWS) {
        __syncthreads();
        load_tile(M, rows, r0);
        __syncthreads();
        double2 acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int k = 0; k < BS; ++k) {
          const double2 t = T[rr * LP + k];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 p = cmuld(t, R[(c0 + 16 * u) * LP + k]);
            acc[u].x += p.x;
            acc[u].y += p.y;
          }
        }
        const int i = r0 + rr;
        if (i < rows)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = cols[c0 + 16 * u];
            if (c >= 0) M[(int64_t)c * rows + i] = acc[u];
          }
      }
    }
  }
}

// sigma_j = ||x_j|| (one warp per column)
__global__ void bj_sigma_kernel(const double2* __restrict__ X, int m, int n, int64_t xs, double* __restrict__ sig) {
  const int f = blockIdx.y;
  const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const double2* x = X + (int64_t)f * xs + (int64_t)w * m;
  double s = 0.0;
  for (int i = lane; i < m; i += 32) s += x[i].x * x[i].x + x[i].y * x[i].y;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sig[(int64_t)f * n + w] = sqrt(s);
}

// t-SVT output: W(i, k) = sum_j x_j[i] w_j conj(v_j[k]),  w_j = (1 - tau / sigma_j)_+ ; 32 x 32 tiles.
// Written as fp32 planes [f][col][row] of the m_in x n_in slice (transposed + conjugated back when
// the slice was processed as its conjugate transpose).
__global__ void __launch_bounds__(256) bj_svt_out_kernel(const double2* __restrict__ X, const double2* __restrict__ V,
                                                        const double* __restrict__ sig, int m, int n, int64_t xs,
                                                        int64_t vs, float tau, int tr, int m_in, float* __restrict__ wre,
                                                        float* __restrict__ wim, int64_t fstride) {
  __shared__ double2 sx[32][33], sv[32][33];
  __shared__ double sw[32];
  const int f = blockIdx.z;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;            // 32 x 8
  const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const double2* x = X + (int64_t)f * xs;
  const double2* v = V + (int64_t)f * vs;
  const double* sg = sig + (int64_t)f * n;
  double2 acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
  for (int j0 = 0; j0 < n; j0 += 32) {
    for (int u = 0; u < 4; ++u) {
      const int jj = ty + 8 * u, j = j0 + jj;
      sx[jj][tx] = (j < n && i0 + tx < m) ? x[(int64_t)j * m + i0 + tx] : make_double2(0.0, 0.0);
      sv[jj][tx] = (j < n && k0 + tx < n) ? v[(int64_t)j * n + k0 + tx] : make_double2(0.0, 0.0);
    }
    if (threadIdx.x < 32) {
      const int j = j0 + threadIdx.x;
      const double s = j < n ? sg[j] : 0.0;
      sw[threadIdx.x] = s > (double)tau ? 1.0 - (double)tau / s : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < 32; ++jj) {
      const double2 a = sx[jj][tx];
      const double w = sw[jj];
      if (w == 0.0) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 b = sv[jj][ty + 8 * u];                          // conj(v_j[k])
        acc[u].x += w * (a.x * b.x + a.y * b.y);
        acc[u].y += w * (a.y * b.x - a.x * b.y);
      }
    }
    __syncthreads();
  }
  float* orr = wre + (int64_t)f * fstride;
  float* oii = wim + (int64_t)f * fstride;
  const int i = i0 + tx;
  if (i >= m) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = k0 + ty + 8 * u;
    if (k >= n) continue;
    if (!tr) {
      orr[(int64_t)k * m_in + i] = (float)acc[u].x;
      oii[(int64_t)k * m_in + i] = (float)acc[u].y;
    } else {                                                          // W = (W')^H
      orr[(int64_t)i * m_in + k] = (float)acc[u].x;
      oii[(int64_t)i * m_in + k] = -(float)acc[u].y;
    }
  }
}

// Non-increasing order of the slice's sigma_j: perm[f][pos] = j (ties by index), sorted[f][pos] = sigma_j.
__global__ void bj_rank_kernel(const double* __restrict__ sig, int n, int* __restrict__ perm,
                               double* __restrict__ sorted) {
  const int f = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double* sg = sig + (int64_t)f * n;
  const double sj = sg[j];
  int pos = 0;
  for (int k = 0; k < n; ++k) {
    const double sk = sg[k];
    pos += (sk > sj) || (sk == sj && k < j);
  }
  if (perm) perm[(int64_t)f * n + pos] = j;
  if (sorted) sorted[(int64_t)f * n + pos] = sj;
}

__device__ __forceinline__ double block_reduce(double v, bool is_max, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, t) : v + t;
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int k = 1; k < nw; ++k) r = is_max ? fmax(r, red[k]) : r + red[k];
  return r;
}

// Left singular vectors of the processed slice: x_j / sigma_j, normalised in place (fp64).  A column
// whose sigma is at the rounding level of the slice (sigma_j <= 1e-6 sigma_max: rank-deficient input)
// has no reliable direction: it is replaced by the unit vector e_c of the row c least covered by the
// columns so far (row coverage rc_i = sum_k |x_k[i]|^2; e_c keeps a residual >= 1 - k/m after the
// projection), Gram-Schmidt-orthogonalised twice against all other columns and normalised -- the
// same rule as the per-slice kernel, so U^* U = I (Theorem 2.2) for any rank.  One CTA per slice;
// dots ([h][n]) and rc ([h][m]) are workspace.
__global__ void __launch_bounds__(1024) bj_left_kernel(double2* __restrict__ X, const double* __restrict__ sig, int m,
                                                       int n, int64_t xs, double2* __restrict__ dots,
                                                       double* __restrict__ rcov) {
  __shared__ double red[32];
  __shared__ double bestv[32];
  __shared__ int besti[32];
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  double2* x = X + (int64_t)f * xs;
  const double* sg = sig + (int64_t)f * n;
  double2* d = dots + (int64_t)f * n;
  double* rc = rcov + (int64_t)f * m;
  double mx = 0.0;
  for (int k = tid; k < n; k += blockDim.x) mx = fmax(mx, sg[k]);
  const double thr = block_reduce(mx, true, red) * 1e-6;
  for (int64_t idx = tid; idx < (int64_t)m * n; idx += blockDim.x) {
    const double sj = sg[idx / m];
    const double inv = sj > thr ? 1.0 / sj : 0.0;
    x[idx] = make_double2(x[idx].x * inv, x[idx].y * inv);
  }
  int z = 0;
  for (int k = tid; k < n; k += blockDim.x) z += sg[k] > thr ? 0 : 1;
  if (block_reduce((double)z, false, red) == 0.0) return;   // full rank: nothing to complete
  for (int i = tid; i < m; i += blockDim.x) {
    double c = 0.0;
    for (int k = 0; k < n; ++k) c += x[(int64_t)k * m + i].x * x[(int64_t)k * m + i].x +
                                     x[(int64_t)k * m + i].y * x[(int64_t)k * m + i].y;
    rc[i] = c;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (sg[j] > thr) continue;                               // block-uniform
    double2* xj = x + (int64_t)j * m;
    // least-covered row
    double bv = 3.0;
    int bi = 0;
    for (int i = tid; i < m; i += blockDim.x)
      if (rc[i] < bv) { bv = rc[i]; bi = i; }
    for (int o = 16; o; o >>= 1) {
      const double tv = __shfl_xor_sync(0xffffffffu, bv, o);
      const int ti = __shfl_xor_sync(0xffffffffu, bi, o);
      if (tv < bv || (tv == bv && ti < bi)) { bv = tv; bi = ti; }
    }
    if (lane == 0) { bestv[w] = bv; besti[w] = bi; }
    __syncthreads();
    int c = besti[0];
    double cv = bestv[0];
    for (int k = 1; k < nw; ++k)
      if (bestv[k] < cv || (bestv[k] == cv && besti[k] < c)) { cv = bestv[k]; c = besti[k]; }
    for (int i = tid; i < m; i += blockDim.x) xj[i] = make_double2(i == c ? 1.0 : 0.0, 0.0);
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = w; k < n; k += nw) {                      // d_k = x_k^H x_j (zero columns pending: 0)
        double pr = 0.0, pi = 0.0;
        if (k != j) {
          const double2* y = x + (int64_t)k * m;
          for (int i = lane; i < m; i += 32) {
            const double2 a = y[i], b = xj[i];
            pr += a.x * b.x + a.y * b.y;
            pi += a.x * b.y - a.y * b.x;
          }
        }
        for (int o = 16; o; o >>= 1) {
          pr += __shfl_xor_sync(0xffffffffu, pr, o);
          pi += __shfl_xor_sync(0xffffffffu, pi, o);
        }
        if (lane == 0) d[k] = make_double2(pr, pi);
      }
      __syncthreads();
      for (int i = tid; i < m; i += blockDim.x) {            // x_j -= sum_k x_k d_k
        double ar = 0.0, ai = 0.0;
        for (int k = 0; k < n; ++k) {
          const double2 a = x[(int64_t)k * m + i], dk = d[k];
          ar += a.x * dk.x - a.y * dk.y;
          ai += a.x * dk.y + a.y * dk.x;
        }
        xj[i] = make_double2(xj[i].x - ar, xj[i].y - ai);
      }
      __syncthreads();
    }
    double nn = 0.0;
    for (int i = tid; i < m; i += blockDim.x) nn += xj[i].x * xj[i].x + xj[i].y * xj[i].y;
    nn = block_reduce(nn, false, red);
    const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
    for (int i = tid; i < m; i += blockDim.x) {
      const double2 v = make_double2(xj[i].x * inv, xj[i].y * inv);
      xj[i] = v;
      rc[i] += v.x * v.x + v.y * v.y;
    }
    __syncthreads();
  }
}

// Factors in non-increasing sigma order (column pos = blockIdx.y): ml left vectors of the processed
// slice (length m; ml = n skinny, m full) and n right vectors (length n); a transposed (wide) slice
// swaps the roles: Y^H = L S R^H gives Y = R S^T L^H, i.e. U = R and V = L.  perm: [f][ml].
// S (the slice's m_s x n_s plane, f-diagonal) is written whole by the CTAs with blockIdx.x == 0:
// column pos < n_s holds sigma at row pos.
__global__ void bj_factors_kernel(const double2* __restrict__ X, const double2* __restrict__ V,
                                  const double* __restrict__ sig, const int* __restrict__ perm, int m, int n, int ml,
                                  int64_t xs, int64_t vs, int tr, int m_s, int n_s, float* __restrict__ ure,
                                  float* __restrict__ uim, float* __restrict__ sre, float* __restrict__ vre,
                                  float* __restrict__ vim) {
  const int f = blockIdx.z, pos = blockIdx.y;
  const int j = perm[(int64_t)f * ml + pos];
  // left planes [f][ml][m], right planes [f][n][n]
  float* lre = tr ? vre : ure;
  float* lim = tr ? vim : uim;
  float* rre = tr ? ure : vre;
  float* rim = tr ? uim : vim;
  const int64_t lo = (int64_t)f * ml * m + (int64_t)pos * m, ro = (int64_t)f * n * n + (int64_t)pos * n;
  const double2* xj = X + (int64_t)f * xs + (int64_t)j * m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    lre[lo + i] = (float)xj[i].x;
    lim[lo + i] = (float)xj[i].y;
  }
  if (pos < n) {                                               // the first n positions are columns j < n
    const double2* vj = V + (int64_t)f * vs + (int64_t)j * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      rre[ro + i] = (float)vj[i].x;
      rim[ro + i] = (float)vj[i].y;
    }
  }
  if (blockIdx.x == 0 && pos < n_s) {
    const float sv = pos < n ? (float)sig[(int64_t)f * ml + j] : 0.f;
    for (int i = threadIdx.x; i < m_s; i += blockDim.x)
      sre[(int64_t)f * m_s * n_s + (int64_t)pos * m_s + i] = i == pos ? sv : 0.f;
  }
}

// A slice whose last allowed sweep still rotated is not certified converged: reported, not silent.
__global__ void bj_status_kernel(const int* __restrict__ flags, int h, int* __restrict__ status) {
  for (int f = threadIdx.x; f < h; f += blockDim.x)
    if (flags[f * MAX_SWEEPS + MAX_SWEEPS - 1]) atomicOr(status, STATUS_NOCONV);
}

// t-SVD scalars (Eq. (14), Def. 2.8, 2.9, Eq. (16)) from sorted per-slice singular values, any r:
// out[i] = (1/n3) sum_{j < n3} S-bar(i,i,j) (conjugate slices counted twice), out[r] = TNN,
// out[r+1] = TSN = max_f sv[f][0], out[r+2] = #{i : out[i] > rtol out[0]}.  One CTA.
__global__ void __launch_bounds__(1024) bj_reduce_kernel(const double* __restrict__ sv, int r, int h, int n3,
                                                         float rtol, float* __restrict__ out) {
  __shared__ double red[32];
  auto S = [&](int i) {
    double acc = 0.0;
    for (int f = 0; f < h; ++f) acc += ((f == 0 || 2 * f == n3) ? 1.0 : 2.0) * sv[(int64_t)f * r + i];
    return acc / n3;
  };
  const double s0 = S(0);
  double tnn = 0.0, rank = 0.0, tsn = 0.0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    const double si = S(i);
    out[i] = (float)si;
    tnn += si;
    rank += (s0 > 0.0 && si > (double)rtol * s0) ? 1.0 : 0.0;
  }
  for (int f = threadIdx.x; f < h; f += blockDim.x) tsn = fmax(tsn, sv[(int64_t)f * r]);
  tnn = block_reduce(tnn, false, red);
  rank = block_reduce(rank, false, red);
  tsn = block_reduce(tsn, true, red);
  if (threadIdx.x == 0) {
    out[r] = (float)tnn;
    out[r + 1] = (float)tsn;
    out[r + 2] = (float)rank;
  }
}

}  // namespace

size_t bj_workspace_bytes(int64_t m_in, int64_t n_in, int64_t h, bool full) {
  const int64_t m = std::max(m_in, n_in), n = std::min(m_in, n_in), ml = full ? m : n;
  // X (m x ml), V, sigma, flags, perm, dots, row coverage (+ alignment slack)
  return 16 * (size_t)h * (size_t)(m * ml + n * n) + 8 * (size_t)h * ml + 4 * (size_t)h * MAX_SWEEPS +
         4 * (size_t)h * ml + 16 * (size_t)h * ml + 8 * (size_t)h * m + 8192;
}

int launch_tsvd_reduce(const double* sv, int64_t r, int64_t h, int64_t n3, float rtol, float* out, cudaStream_t s) {
  bj_reduce_kernel<<<1, 1024, 0, s>>>(sv, (int)r, (int)h, (int)n3, rtol, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// Blocked Jacobi of all h spectral slices (re / im planes [f][col][row], m_in x n_in, pitch
// fstride) in the workspace `ws` (bj_workspace_bytes); `mode` / `o` as in internal.h.
int launch_block_svd(const float* re, const float* im, int64_t m_in, int64_t n_in, int64_t h, int64_t fstride,
                     int mode, BjOut o, void* ws, int* status, cudaStream_t s) {
  const bool tr = m_in < n_in;
  const int m = (int)std::max(m_in, n_in), n = (int)std::min(m_in, n_in);
  const bool full = mode == BJ_FACTORS_FULL;
  const int ml = full ? m : n;                                      // columns of X (left vectors)
  const int64_t xs = (int64_t)m * ml, vs = (int64_t)n * n;
  double2* X = (double2*)ws;
  double2* V = X + h * xs;
  double* sig = (double*)(V + h * vs);
  int* flags = (int*)(sig + h * ml);
  int* perm = flags + h * MAX_SWEEPS;
  double2* dots = (double2*)(((uintptr_t)(perm + h * ml) + 15) & ~(uintptr_t)15);
  double* rcov = (double*)(dots + h * ml);
  cudaMemsetAsync(flags, 0, 4 * (size_t)h * MAX_SWEEPS, s);
  if (ml > n)                                                       // full factors: columns n.. start at 0
    cudaMemset2DAsync(X + (int64_t)n * m, 16 * (size_t)xs, 0, 16 * (size_t)(ml - n) * m, (size_t)h, s);
  {
    const int64_t work = (int64_t)m * n;
    const int gx = (int)std::min<int64_t>((work + 255) / 256, 1024);
    bj_init_kernel<<<dim3(gx, (unsigned)h), 256, 0, s>>>(re, im, fstride, (int)m_in, (int)n_in, tr ? 1 : 0, X, V, m, n,
                                                        xs, vs);
  }
  const int nb = (n + BJ - 1) / BJ;
  const int nbp = std::max(2, nb + (nb & 1));                     // even number of players (>= 2)
  const size_t smem = sizeof(double2) * (2 * BS + ROWS) * LP;
  if (cudaFuncSetAttribute(bj_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 4;
  // a single block (n <= 32) is the pair (block 0, empty block 1); every sweep's launches return at
  // once for a slice whose previous sweep rotated nothing
  for (int sw = 0; sw < MAX_SWEEPS; ++sw)
    for (int r = 0; r < nbp - 1; ++r)
      bj_round_kernel<<<dim3(nbp / 2, (unsigned)h), BJ_THREADS, smem, s>>>(X, V, m, n, xs, vs, nbp, r, sw, flags);
  if (status) bj_status_kernel<<<1, 256, 0, s>>>(flags, (int)h, status);
#ifdef TPROD_SVT_DEBUG
  {
    std::vector<int> fl((size_t)h * MAX_SWEEPS);
    cudaMemcpyAsync(fl.data(), flags, fl.size() * 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    for (int64_t f = 0; f < h; ++f) {
      int used = 0;
      while (used < MAX_SWEEPS && fl[f * MAX_SWEEPS + used]) ++used;
      fprintf(stderr, "bj slice %lld: %d rotating sweeps\n", (long long)f, used);
    }
  }
#endif
  bj_sigma_kernel<<<dim3((ml * 32 + 255) / 256, (unsigned)h), 256, 0, s>>>(X, m, ml, xs, sig);
  if (mode == BJ_SVT) {
    dim3 g((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32), (unsigned)h);
    bj_svt_out_kernel<<<g, 256, 0, s>>>(X, V, sig, m, n, xs, vs, o.tau, tr ? 1 : 0, (int)m_in, o.wre, o.wim, fstride);
  } else if (mode == BJ_VALUES) {
    bj_rank_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)h), 256, 0, s>>>(sig, n, nullptr, o.sv);
  } else {
    // (full: the extra columns have sigma 0 and sort last, so positions < n are the columns j < n)
    bj_rank_kernel<<<dim3((unsigned)((ml + 255) / 256), (unsigned)h), 256, 0, s>>>(sig, ml, perm, nullptr);
    bj_left_kernel<<<(unsigned)h, 1024, 0, s>>>(X, sig, m, ml, xs, dots, rcov);
    const int gx = std::min(8, (m + 255) / 256);
    // S: r x r (skinny) or the slice's m_in x n_in plane (full)
    const int m_s = full ? (int)m_in : n, n_s = full ? (int)n_in : n;
    bj_factors_kernel<<<dim3((unsigned)gx, (unsigned)std::max(ml, n_s), (unsigned)h), 256, 0, s>>>(
        X, V, sig, perm, m, n, ml, xs, vs, tr ? 1 : 0, m_s, n_s, o.ure, o.uim, o.sre, o.vre, o.vim);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tprod
