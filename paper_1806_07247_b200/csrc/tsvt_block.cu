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

}  // namespace

size_t bj_workspace_bytes(int64_t m_in, int64_t n_in, int64_t h) {
  const int64_t m = std::max(m_in, n_in), n = std::min(m_in, n_in);
  return 16 * (size_t)h * (size_t)(m * n + n * n) + 8 * (size_t)h * n + 4 * (size_t)h * MAX_SWEEPS + 4096;
}

// Blocked Jacobi of all h spectral slices (re / im planes [f][col][row], m_in x n_in, pitch
// fstride) in the workspace `ws` (bj_workspace_bytes).  tau >= 0: t-SVT into wre / wim; tau < 0:
// the singular values only, into `sig_out` (h x min(m, n) doubles, unsorted per slice).
int launch_block_svt(const float* re, const float* im, int64_t m_in, int64_t n_in, int64_t h, int64_t fstride,
                     float tau, float* wre, float* wim, double* sig_out, void* ws, cudaStream_t s) {
  const bool tr = m_in < n_in;
  const int m = (int)std::max(m_in, n_in), n = (int)std::min(m_in, n_in);
  const int64_t xs = (int64_t)m * n, vs = (int64_t)n * n;
  double2* X = (double2*)ws;
  double2* V = X + h * xs;
  double* sig = (double*)(V + h * vs);
  int* flags = (int*)(sig + h * n);
  cudaMemsetAsync(flags, 0, 4 * (size_t)h * MAX_SWEEPS, s);
  {
    const int64_t work = (int64_t)m * n;
    const int gx = (int)std::min<int64_t>((work + 255) / 256, 1024);
    bj_init_kernel<<<dim3(gx, (unsigned)h), 256, 0, s>>>(re, im, fstride, (int)m_in, (int)n_in, tr ? 1 : 0, X, V, m, n,
                                                        xs, vs);
  }
  const int nb = (n + BJ - 1) / BJ;
  const int nbp = nb + (nb & 1);                                   // even number of players
  const size_t smem = sizeof(double2) * (2 * BS + ROWS) * LP;
  if (cudaFuncSetAttribute(bj_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 4;
  if (nb == 1) {
    // a single block: one "pair" of block 0 with the empty block 1 orthogonalises all n columns
    for (int sw = 0; sw < 2; ++sw)
      bj_round_kernel<<<dim3(1, (unsigned)h), BJ_THREADS, smem, s>>>(X, V, m, n, xs, vs, 2, 0, sw, flags);
  } else {
    for (int sw = 0; sw < MAX_SWEEPS; ++sw)
      for (int r = 0; r < nbp - 1; ++r)
        bj_round_kernel<<<dim3(nbp / 2, (unsigned)h), BJ_THREADS, smem, s>>>(X, V, m, n, xs, vs, nbp, r, sw, flags);
  }
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
  bj_sigma_kernel<<<dim3((n * 32 + 255) / 256, (unsigned)h), 256, 0, s>>>(X, m, n, xs, sig_out ? sig_out : sig);
  if (tau >= 0.f) {
    dim3 g((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32), (unsigned)h);
    bj_svt_out_kernel<<<g, 256, 0, s>>>(X, V, sig, m, n, xs, vs, tau, tr ? 1 : 0, (int)m_in, wre, wim, fstride);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tprod
