// NEXT-4: the t-product's companion operations on the GPU.
//
//   tran  -- conjugate transpose, Definition 2.2: slice k of A^* is
//            (A^((n3 - k) mod n3))^T (real data: conjugation is the identity);
//   teye  -- identity tensor, Definition 2.3: I_n in slice 0, zeros elsewhere;
//   tinv  -- tensor inverse, Definition 2.4, Eq. (11), the Fourier way of
//            Algorithm 1: forward mode-3 DFT (the production K1 kernels, decoded to fp32), one
//            complex Gauss-Jordan inverse per spectral slice f < h (Eq. (8): the rest are the
//            conjugates), inverse DFT with the fused conjugate fill (the production K3 kernels).
#include "internal.h"
#include "common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace tprod {

// ---------------------------------------------------------------------------------------- tran
template <typename T>
__global__ void tran_kernel(const T* __restrict__ A, T* __restrict__ At, int64_t n1, int64_t n2, int64_t n3) {
  __shared__ T tile[32][33];
  const int64_t k = blockIdx.z;                         // destination slice
  const int64_t ks = k == 0 ? 0 : n3 - k;               // source slice (Def. 2.2 reversal)
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;   // source (row i, col j)
  const T* src = A + n1 * n2 * ks;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + threadIdx.x, j = j0 + r;
    if (i < n1 && j < n2) tile[r][threadIdx.x] = src[i + n1 * j];
  }
  __syncthreads();
  T* dst = At + n2 * n1 * k;                            // At is n2 x n1 x n3: (j, i) at j + n2 * i
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + threadIdx.x, i = i0 + r;
    if (i < n1 && j < n2) dst[j + n2 * i] = tile[threadIdx.x][r];
  }
}

// fp32 with n1, n2 multiples of 4 and 16-byte aligned slices: 64 x 64 tiles moved as float4 on both
// sides (each thread keeps four 16-byte loads in flight), staged transposed through shared memory
// with a 65-float pitch.  A float4 is entirely inside or outside the slice, so the ragged edge
// needs no scalar tail.
__global__ void __launch_bounds__(256) tran4_kernel(const float* __restrict__ A, float* __restrict__ At, int n1, int n2,
                                                    int64_t n3) {
  __shared__ float tile[64][65];                        // tile[j][i]: source column j, row i
  const int64_t k = blockIdx.z;
  const int64_t ks = k == 0 ? 0 : n3 - k;               // source slice (Def. 2.2 reversal)
  const int i0 = blockIdx.x * 64, j0 = blockIdx.y * 64;
  const float* src = A + (int64_t)n1 * n2 * ks;
  const int t = threadIdx.x, c4 = (t & 15) * 4, r0 = t >> 4;
  float4 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {                         // source column j = j0 + r0 + 16 r, rows i0 + c4 .. +3
    const int i = i0 + c4, j = j0 + r0 + 16 * r;
    v[r] = (i < n1 && j < n2) ? __ldg(reinterpret_cast<const float4*>(src + i + (int64_t)n1 * j))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    float* row = &tile[r0 + 16 * r][c4];
    row[0] = v[r].x;
    row[1] = v[r].y;
    row[2] = v[r].z;
    row[3] = v[r].w;
  }
  __syncthreads();
  float* dst = At + (int64_t)n2 * n1 * k;               // At is n2 x n1 x n3: (j, i) at j + n2 * i
#pragma unroll
  for (int r = 0; r < 4; ++r) {                         // destination column i = i0 + r0 + 16 r, rows j0 + c4 .. +3
    const int i = i0 + r0 + 16 * r, j = j0 + c4;
    if (i < n1 && j < n2) {
      const int ii = r0 + 16 * r;
      *reinterpret_cast<float4*>(dst + j + (int64_t)n2 * i) =
          make_float4(tile[c4][ii], tile[c4 + 1][ii], tile[c4 + 2][ii], tile[c4 + 3][ii]);
    }
  }
}

template <typename T>
void launch_tran(const T* A, T* At, int64_t n1, int64_t n2, int64_t n3, cudaStream_t s) {
  if (sizeof(T) == 4 && n1 % 4 == 0 && n2 % 4 == 0 && n1 * n2 < (1ll << 31) && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(At) & 15) == 0) {
    dim3 grid((unsigned)((n1 + 63) / 64), (unsigned)((n2 + 63) / 64), (unsigned)n3);
    tran4_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float*>(A), reinterpret_cast<float*>(At), (int)n1,
                                      (int)n2, n3);
    return;
  }
  dim3 grid((unsigned)((n1 + 31) / 32), (unsigned)((n2 + 31) / 32), (unsigned)n3);
  tran_kernel<T><<<grid, dim3(32, 8), 0, s>>>(A, At, n1, n2, n3);
}
template void launch_tran<float>(const float*, float*, int64_t, int64_t, int64_t, cudaStream_t);
template void launch_tran<double>(const double*, double*, int64_t, int64_t, int64_t, cudaStream_t);

// ---------------------------------------------------------------------------------------- teye
template <typename T>
__global__ void teye_diag_kernel(T* __restrict__ I, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) I[i + n * i] = T(1);
}

template <typename T>
int launch_teye(T* I, int64_t n, int64_t n3, cudaStream_t s) {
  if (cudaMemsetAsync(I, 0, sizeof(T) * (size_t)(n * n * n3), s) != cudaSuccess) return 4;
  teye_diag_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(I, n);
  return 0;
}
template int launch_teye<float>(float*, int64_t, int64_t, cudaStream_t);
template int launch_teye<double>(double*, int64_t, int64_t, cudaStream_t);

// ---------------------------------------------------------------------- batched slice inverse
// One CTA per spectral slice f: Gauss-Jordan with partial pivoting on the augmented n x 2n complex
// matrix [A-bar_f | I] in shared memory (row-major, fp32 complex).  Planes: re/im [f][q][p], the
// (p, q) element at f * fstride + q * n + p.  A pivot |a_kk| <= rtol * max_f |A-bar_f| (the largest
// entry magnitude over all slices, passed in) marks the tensor singular (flag set, no inverse).
constexpr int TINV_MAX = 96;

__global__ void __launch_bounds__(256) slice_inverse_kernel(const float* __restrict__ re, const float* __restrict__ im,
                                                           float* __restrict__ xre, float* __restrict__ xim, int n,
                                                           int64_t fstride, float rtol, const unsigned* __restrict__ maxp,
                                                           int* __restrict__ singular) {
  extern __shared__ float2 aug[];                       // [n][2n]
  __shared__ float red_v[256];
  __shared__ int red_i[256];
  __shared__ int piv_row;
  const int f = blockIdx.x, w = 2 * n;
  const float thresh = rtol * __uint_as_float(*maxp);
  const float* ar = re + (int64_t)f * fstride;
  const float* ai = im + (int64_t)f * fstride;
  for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) {
    const int r = idx / w, c = idx - r * w;
    aug[idx] = c < n ? make_float2(ar[(int64_t)c * n + r], ai[(int64_t)c * n + r])
                     : make_float2(c - n == r ? 1.f : 0.f, 0.f);
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    // pivot: max |a_rk|^2 over rows r >= k
    float best = -1.f;
    int bi = k;
    for (int r = k + threadIdx.x; r < n; r += blockDim.x) {
      const float2 v = aug[r * w + k];
      const float m = v.x * v.x + v.y * v.y;
      if (m > best) { best = m; bi = r; }
    }
    red_v[threadIdx.x] = best;
    red_i[threadIdx.x] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o && red_v[threadIdx.x + o] > red_v[threadIdx.x]) {
        red_v[threadIdx.x] = red_v[threadIdx.x + o];
        red_i[threadIdx.x] = red_i[threadIdx.x + o];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      piv_row = red_i[0];
      if (!(sqrtf(red_v[0]) > thresh)) atomicOr(singular, STATUS_SINGULAR);
    }
    __syncthreads();
    const int pr = piv_row;
    if (pr != k)
      for (int c = threadIdx.x; c < w; c += blockDim.x) {
        const float2 t = aug[k * w + c];
        aug[k * w + c] = aug[pr * w + c];
        aug[pr * w + c] = t;
      }
    __syncthreads();
    // scale row k by 1 / a_kk
    const float2 p = aug[k * w + k];
    const float den = p.x * p.x + p.y * p.y;
    const float2 inv = den > 0.f ? make_float2(p.x / den, -p.y / den) : make_float2(0.f, 0.f);
    __syncthreads();
    for (int c = threadIdx.x; c < w; c += blockDim.x) {
      const float2 v = aug[k * w + c];
      aug[k * w + c] = make_float2(v.x * inv.x - v.y * inv.y, v.x * inv.y + v.y * inv.x);
    }
    __syncthreads();
    // eliminate column k from every other row
    for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) {
      const int r = idx / w, c = idx - r * w;
      if (r == k || c == k) continue;
      const float2 fct = aug[r * w + k], pk = aug[k * w + c];
      float2 v = aug[idx];
      v.x -= fct.x * pk.x - fct.y * pk.y;
      v.y -= fct.x * pk.y + fct.y * pk.x;
      aug[idx] = v;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      if (r != k) aug[r * w + k] = make_float2(0.f, 0.f);
    __syncthreads();
  }
  float* orr = xre + (int64_t)f * fstride;
  float* oii = xim + (int64_t)f * fstride;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int q = idx / n, pp = idx - q * n;            // (pp, q) element of the inverse
    const float2 v = aug[pp * w + n + q];
    orr[(int64_t)q * n + pp] = v.x;
    oii[(int64_t)q * n + pp] = v.y;
  }
}

bool tinv_supported(int64_t n) { return n >= 1 && n <= TINV_MAX; }

int launch_slice_inverse(const float* re, const float* im, float* xre, float* xim, int64_t n, int64_t h,
                         int64_t fstride, float rtol, const unsigned* maxp, int* singular, cudaStream_t s) {
  if (!tinv_supported(n)) return 6;
  const size_t smem = sizeof(float2) * (size_t)(n * 2 * n);
  if (cudaFuncSetAttribute(slice_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return 4;
  slice_inverse_kernel<<<(unsigned)h, 256, smem, s>>>(re, im, xre, xim, (int)n, fstride, rtol, maxp, singular);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// ---------------------------------------------------------------------- large slices (n > 96)
// Gauss-Jordan with partial pivoting on [A-bar_f | I] in global memory, fp64 complex, all h slices
// at once: per pivot column k one pivot launch (one CTA per slice: pivot among the rows not yet
// used, multipliers l_i = a_ik / a_pk) and one elimination launch (a_ij -= l_i a_pj, j > k, i != p;
// the pivot row is never scaled, so nothing reads a row while it changes).  Rows are not swapped:
// piv[k] = p records the order, and X(k, :) = right half of row piv[k] / a_{piv[k], k} at the end.
// Row-major augmented slices: (i, j) at f * n * 2n + i * 2n + j.
__global__ void gj_init_kernel(const float* __restrict__ re, const float* __restrict__ im, int n, int64_t fstride,
                               double2* __restrict__ aug, int* __restrict__ used) {
  const int f = blockIdx.y, w = 2 * n;
  double2* a = aug + (int64_t)f * n * w;
  const float* ar = re + (int64_t)f * fstride;
  const float* ai = im + (int64_t)f * fstride;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)n * w;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / w), c = (int)(idx - (int64_t)r * w);
    a[idx] = c < n ? make_double2(ar[(int64_t)c * n + r], ai[(int64_t)c * n + r])
                   : make_double2(c - n == r ? 1.0 : 0.0, 0.0);
  }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    used[(int64_t)f * n + r] = 0;
}

__global__ void __launch_bounds__(256) gj_pivot_kernel(const double2* __restrict__ aug, int n, int k, float rtol,
                                                       const unsigned* __restrict__ maxp, int* __restrict__ used,
                                                       int* __restrict__ piv, double2* __restrict__ fac,
                                                       int* __restrict__ singular) {
  __shared__ double bv_s[8];
  __shared__ int bi_s[8];
  __shared__ int p_s;
  const int f = blockIdx.x, w = 2 * n, tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const double2* a = aug + (int64_t)f * n * w;
  int* u = used + (int64_t)f * n;
  double bv = -1.0;
  int bi = n;
  for (int r = tid; r < n; r += blockDim.x) {
    if (u[r]) continue;
    const double2 v = a[(int64_t)r * w + k];
    const double m2 = v.x * v.x + v.y * v.y;
    if (m2 > bv) { bv = m2; bi = r; }
  }
  for (int o = 16; o; o >>= 1) {
    const double tv = __shfl_xor_sync(0xffffffffu, bv, o);
    const int ti = __shfl_xor_sync(0xffffffffu, bi, o);
    if (tv > bv || (tv == bv && ti < bi)) { bv = tv; bi = ti; }
  }
  if (lane == 0) { bv_s[wp] = bv; bi_s[wp] = bi; }
  __syncthreads();
  if (tid == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (bv_s[q] > bv_s[0] || (bv_s[q] == bv_s[0] && bi_s[q] < bi_s[0])) { bv_s[0] = bv_s[q]; bi_s[0] = bi_s[q]; }
    const int p = bi_s[0] < n ? bi_s[0] : 0;
    const double thresh = (double)rtol * (double)__uint_as_float(*maxp);
    if (!(sqrt(bv_s[0]) > thresh)) atomicOr(singular, STATUS_SINGULAR);
    u[p] = 1;
    piv[(int64_t)f * n + k] = p;
    p_s = p;
  }
  __syncthreads();
  const int p = p_s;
  const double2 pk = a[(int64_t)p * w + k];
  const double den = pk.x * pk.x + pk.y * pk.y;
  const double2 ipk = den > 0.0 ? make_double2(pk.x / den, -pk.y / den) : make_double2(0.0, 0.0);
  for (int r = tid; r < n; r += blockDim.x) {
    const double2 v = a[(int64_t)r * w + k];
    fac[(int64_t)f * n + r] = r == p ? make_double2(0.0, 0.0)
                                     : make_double2(v.x * ipk.x - v.y * ipk.y, v.x * ipk.y + v.y * ipk.x);
  }
}

// one CTA per (row i, slice f); columns j > k of the row
__global__ void __launch_bounds__(256) gj_elim_kernel(double2* __restrict__ aug, int n, int k,
                                                      const int* __restrict__ piv, const double2* __restrict__ fac) {
  const int i = blockIdx.x, f = blockIdx.y, w = 2 * n;
  const double2 l = fac[(int64_t)f * n + i];
  if (l.x == 0.0 && l.y == 0.0) return;                  // pivot row, or nothing to eliminate
  const int p = piv[(int64_t)f * n + k];
  double2* a = aug + (int64_t)f * n * w;
  const double2* ap = a + (int64_t)p * w;
  double2* ai = a + (int64_t)i * w;
  for (int j = k + 1 + threadIdx.x; j < w; j += blockDim.x) {
    const double2 b = ap[j];
    double2 v = ai[j];
    v.x -= l.x * b.x - l.y * b.y;
    v.y -= l.x * b.y + l.y * b.x;
    ai[j] = v;
  }
}

// X(q, c) = a(piv[q], n + c) / a(piv[q], q) into fp32 planes [f][c][q]
__global__ void gj_out_kernel(const double2* __restrict__ aug, int n, const int* __restrict__ piv,
                              float* __restrict__ xre, float* __restrict__ xim, int64_t fstride) {
  const int q = blockIdx.x, f = blockIdx.y, w = 2 * n;
  const int p = piv[(int64_t)f * n + q];
  const double2* ap = aug + (int64_t)f * n * w + (int64_t)p * w;
  const double2 d = ap[q];
  const double den = d.x * d.x + d.y * d.y;
  const double2 id = den > 0.0 ? make_double2(d.x / den, -d.y / den) : make_double2(0.0, 0.0);
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double2 v = ap[n + c];
    xre[(int64_t)f * fstride + (int64_t)c * n + q] = (float)(v.x * id.x - v.y * id.y);
    xim[(int64_t)f * fstride + (int64_t)c * n + q] = (float)(v.x * id.y + v.y * id.x);
  }
}

size_t gj_workspace_bytes(int64_t n, int64_t h) {
  return 16 * (size_t)(h * n * 2 * n) + 16 * (size_t)(h * n) + 8 * (size_t)(h * n) + 1024;
}

int launch_slice_inverse_large(const float* re, const float* im, float* xre, float* xim, int64_t n, int64_t h,
                               int64_t fstride, float rtol, const unsigned* maxp, int* singular, void* ws,
                               cudaStream_t s) {
  double2* aug = (double2*)ws;
  double2* fac = aug + h * n * 2 * n;
  int* piv = (int*)(fac + h * n);
  int* used = piv + h * n;
  const int gx = (int)std::min<int64_t>((n * 2 * n + 255) / 256, 2048);
  gj_init_kernel<<<dim3(gx, (unsigned)h), 256, 0, s>>>(re, im, (int)n, fstride, aug, used);
  for (int k = 0; k < (int)n; ++k) {
    gj_pivot_kernel<<<(unsigned)h, 256, 0, s>>>(aug, (int)n, k, rtol, maxp, used, piv, fac, singular);
    gj_elim_kernel<<<dim3((unsigned)n, (unsigned)h), 256, 0, s>>>(aug, (int)n, k, piv, fac);
  }
  gj_out_kernel<<<dim3((unsigned)n, (unsigned)h), 256, 0, s>>>(aug, (int)n, piv, xre, xim, fstride);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// largest |entry| over the decoded spectral planes (for the singularity threshold)
__global__ void absmax_planes_kernel(const float* __restrict__ re, const float* __restrict__ im, int64_t count,
                                     unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, sqrtf(re[i] * re[i] + im[i] * im[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

void launch_absmax_planes(const float* re, const float* im, int64_t count, unsigned* out, cudaStream_t s) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  absmax_planes_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(re, im, count, out);
}

}  // namespace tprod

namespace tprod {

// ------------------------------------------------------------------------------ batched slice SVT
// NEXT-2, Algorithm 3 step 2: for each spectral slice f < h,
// W-bar_f = U (S - tau)_+ V^*.  One CTA per slice: one-sided (Hestenes) Jacobi on the m x n complex
// slice in shared memory -- columns p, q orthogonalised by the complex rotation
//   a_q' = a_q e (e = conj(g)/|g|, g = a_p^H a_q),  [a_p, a_q'] <- [a_p, a_q'] [[c, s], [-s, c]],
//   zeta = (beta - alpha) / (2|g|), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), c = 1/sqrt(1+t^2), s = c t
// over round-robin pair schedules (a group of G lanes per pair), V accumulating the same rotations -- until
// every |g| <= 1e-10 sqrt(alpha beta) (the fp32 spectra in are accurate to ~1e-7).  Then A V = U S, sigma_j = ||(A V)_j|| and
// W = (A V) diag((1 - tau/sigma_j)_+) V^H.  The Jacobi iteration runs in fp64 (an fp32 one stalls at
// its round-off floor, ~m eps, above a useful orthogonality tolerance for 64 columns); the
// spectra in and W out are fp32.
constexpr int SVT_MAX = 64;

template <int G>
__device__ __forceinline__ double group_sum(double x) {   // sum over an aligned group of G lanes
  for (int o = G / 2; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_sum(double x) { return group_sum<32>(x); }

struct SvdOut {               // per-slice skinny SVD factors (t-SVD), planes [f][col][row], r = min(M, N)
  float *ure, *uim, *sre, *vre, *vim;
};

template <int G>
__global__ void __launch_bounds__(G * SVT_MAX / 2) slice_svt_kernel(const float* __restrict__ re, const float* __restrict__ im,
                                                        float* __restrict__ wre, float* __restrict__ wim, int m, int n,
                                                        int64_t fstride, float tau, double* __restrict__ sv,
                                                        SvdOut fo, int* __restrict__ status) {
  extern __shared__ double2 sm[];
  double2* a = sm;                                      // column j at a + j*m
  double2* v = a + n * m;                               // column j at v + j*n
  __shared__ int rotated[3];                            // per-sweep "some pair rotated" flags, cycled mod 3
  __shared__ double wgt[SVT_MAX];
  const int f = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const float* ar = re + (int64_t)f * fstride;
  const float* ai = im + (int64_t)f * fstride;
  // wide slices (m < n) are processed as their conjugate transpose: SVT(Y^H) = SVT(Y)^H, so the
  // Jacobi iteration always orthogonalises min(m, n) columns of length max(m, n)
  const int M = m, N = n;
  const bool tr = m < n;
  if (tr) {
    m = N;
    n = M;
  }
  for (int idx = tid; idx < n * m; idx += blockDim.x) {
    if (!tr) {
      a[idx] = make_double2(ar[idx], ai[idx]);
    } else {                                            // a(i, j) = conj(Y(j, i)), Y(r, c) at c*M + r
      const int j = idx / m, i = idx - j * m;
      a[idx] = make_double2(ar[(int64_t)i * M + j], -ai[(int64_t)i * M + j]);
    }
  }
  if (sv == nullptr)                                    // V is not formed for singular values only
    for (int idx = tid; idx < n * n; idx += blockDim.x) v[idx] = make_double2((idx / n) == (idx % n) ? 1.0 : 0.0, 0.0);
  __syncthreads();
  if (tid < 3) rotated[tid] = 0;
  __syncthreads();
  const int np = (n + 1) & ~1;                          // players (one dummy when n is odd)
  const bool want_v = sv == nullptr;                    // singular values only: V is never formed
  constexpr int GPW = 32 / G;                           // pairs per warp
  constexpr int L = (G == 8 ? 32 : SVT_MAX) / G;        // elements per lane (G = 8 only for columns <= 32)
  const int gl = lane & (G - 1), gw = lane / G;
#ifdef TPROD_SVT_DEBUG
  const long long t0 = clock64();
  int nsweeps = 0;
#endif
  bool converged = false;
  for (int sweep = 0; sweep < 40; ++sweep) {
#ifdef TPROD_SVT_DEBUG
    nsweeps = sweep + 1;
#endif
    // rotated[(sweep+1)%3] was last read at the end of sweep - 2 and is next written in sweep + 1:
    // both separated from this store by barriers
    if (tid == 0) rotated[(sweep + 1) % 3] = 0;
    for (int r = 0; r < np - 1; ++r) {
      // warp-uniform trip count (the group sums shuffle across the whole warp)
      for (int kb = warp * GPW; kb < np / 2; kb += nw * GPW) {
        // circle method: player np-1 fixed, pairs (r+k, r-k) mod (np-1)
        const int k = kb + gw;
        int p = r + k, q = r - k + np - 1;              // (r + k) mod (np - 1), (r - k) mod (np - 1): one wrap each
        if (p >= np - 1) p -= np - 1;
        if (q >= np - 1) q -= np - 1;
        if (k == 0) q = np - 1;
        const bool valid = k < np / 2 && p < n && q < n;
        double2* ap = a + (valid ? p : 0) * m;
        double2* aq = a + (valid ? q : 0) * m;
        double2* vp = v + (valid ? p : 0) * n;
        double2* vq = v + (valid ? q : 0) * n;
        // this group owns columns p, q for the round: they are read once (predicated, so the loads
        // batch), kept in registers through the reductions and the angle, and written back rotated;
        // V's columns are fetched at the same time so their latency hides behind the reductions
        const double2 z = make_double2(0.0, 0.0);
        double2 xs[L], ys[L], vx[L], vy[L];
#pragma unroll
        for (int it = 0; it < L; ++it) {
          const int i = gl + it * G;
          xs[it] = valid && i < m ? ap[i] : z;
          ys[it] = valid && i < m ? aq[i] : z;
          vx[it] = want_v && valid && i < n ? vp[i] : z;
          vy[it] = want_v && valid && i < n ? vq[i] : z;
        }
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
        for (int it = 0; it < L; ++it) {
          const double2 x = xs[it], y = ys[it];
          al += x.x * x.x + x.y * x.y;
          be += y.x * y.x + y.y * y.y;
          gr += x.x * y.x + x.y * y.y;                  // conj(x) * y
          gi += x.x * y.y - x.y * y.x;
        }
        al = group_sum<G>(al);
        be = group_sum<G>(be);
        gr = group_sum<G>(gr);
        gi = group_sum<G>(gi);
        const double g2 = gr * gr + gi * gi;
        if (!valid || !(g2 > 1e-20 * al * be) || !(g2 > 0.0)) continue;   // already orthogonal (or a zero column)
        if (gl == 0) rotated[sweep % 3] = 1;
        // fp64 divisions / square roots are slow: the angle comes from fp32 estimates (an approximate
        // Jacobi angle still converges), and the quantities that must be exact to fp64 -- the unit
        // phase e and the rotation's c^2 + s^2 = 1 -- get one Newton step of rsqrt in fp64
        // (below ~1e-36 the fp32 estimate of g2 is subnormal and rsqrtf loses all accuracy -- measured
        // |e|^2 - 1 = -0.14 on a rank-deficient slice, which broke V's orthonormality -- so those rare
        // pairs take the exact fp64 route)
        double ig;
        if (g2 > 1e-36) {
          const float ig32 = rsqrtf((float)g2);
          ig = (double)ig32 * (1.5 - 0.5 * g2 * (double)ig32 * (double)ig32);   // 1 / |g|
        } else {
          ig = 1.0 / sqrt(g2);
        }
        const float zeta = (float)((be - al) * 0.5 * ig);
        const float t32 = copysignf(1.f, zeta) / (fabsf(zeta) + sqrtf(1.f + zeta * zeta));
        const double t = t32, t2p1 = 1.0 + t * t;
        const float c32 = rsqrtf((float)t2p1);
        const double c = (double)c32 * (1.5 - 0.5 * t2p1 * (double)c32 * (double)c32), s = c * t;
        const double er = gr * ig, ei = -gi * ig;         // e = conj(g) / |g|
#pragma unroll
        for (int it = 0; it < L; ++it) {
          const int i = gl + it * G;
          const double2 x = xs[it], y0 = ys[it];
          const double2 y = make_double2(y0.x * er - y0.y * ei, y0.x * ei + y0.y * er);
          if (i < m) {
            ap[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
            aq[i] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
          }
        }
        if (want_v) {
#pragma unroll
          for (int it = 0; it < L; ++it) {
            const int i = gl + it * G;
            const double2 x = vx[it], y0 = vy[it];
            const double2 y = make_double2(y0.x * er - y0.y * ei, y0.x * ei + y0.y * er);
            if (i < n) {
              vp[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
              vq[i] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
            }
          }
        }
      }
      __syncthreads();
    }
    if (!rotated[sweep % 3]) {                          // no pair above the tolerance: read after a barrier
      converged = true;
      break;
    }
  }
  if (!converged && tid == 0 && status) atomicOr(status, STATUS_NOCONV);   // sweep cap reached: reported
#ifdef TPROD_SVT_DEBUG
  if (tid == 0 && f < 2) printf("svt f=%d m=%d n=%d G=%d sweeps=%d cycles=%lld\n", f, m, n, G, nsweeps, clock64() - t0);
#endif
#ifdef TPROD_SVT_DEBUG
  __syncthreads();
  if (tid == 0 && want_v && f < 2) {
    double dev = 0.0, imx = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        double gr = 0.0, gi = 0.0;
        for (int i = 0; i < n; ++i) {
          const double2 x = v[p * n + i], y = v[q * n + i];
          gr += x.x * y.x + x.y * y.y;
          gi += x.x * y.y - x.y * y.x;
          imx = fmax(imx, fabs(x.y));
        }
        dev = fmax(dev, fabs(gr - (p == q ? 1.0 : 0.0)) + fabs(gi));
      }
    printf("svd f=%d tr=%d m=%d n=%d |V^H V - I|=%g max|Im V|=%g\n", f, (int)tr, m, n, dev, imx);
  }
  __syncthreads();
#endif
  // sigma_j = ||(A V)_j||, weights (1 - tau / sigma_j)_+
  for (int j = warp; j < n; j += nw) {
    double ss = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double2 x = a[j * m + i];
      ss += x.x * x.x + x.y * x.y;
    }
    ss = warp_sum(ss);
    if (lane == 0) {
      const double sg = sqrt(ss);
      wgt[j] = (sv || fo.ure) ? sg : (sg > (double)tau ? 1.0 - (double)tau / sg : 0.0);   // sigma or SVT weight
    }
  }
  __syncthreads();
  if (sv) {
    // singular values only (t-SVD scalars): slice f's n values in non-increasing order
    for (int j = tid; j < n; j += blockDim.x) {
      int pos = 0;
      for (int k = 0; k < n; ++k) pos += (wgt[k] > wgt[j]) || (wgt[k] == wgt[j] && k < j);
      sv[(int64_t)f * n + pos] = wgt[j];
    }
    return;
  }
  if (fo.ure) {
    // skinny SVD factors, columns in non-increasing sigma order: left vectors (A V)_j / sigma_j
    // (zero for sigma_j = 0), right vectors v_j; for a transposed (wide) slice the roles swap:
    // Y^H = L S R^H gives Y = R S L^H, i.e. U = R and V = L (no conjugation)
    const int r = n;                                     // n = min(M, N) after the swap
    const int64_t uo = (int64_t)f * M * r, vo = (int64_t)f * N * r, so = (int64_t)f * r * r;
    for (int idx = tid; idx < r * r; idx += blockDim.x) fo.sre[so + idx] = 0.f;
    // Left vectors (A V)_j / sigma_j, normalised in place.  A column whose sigma is at the rounding
    // level of the slice (rank-deficient input) has no reliable direction: it is replaced by a unit
    // vector Gram-Schmidt-orthogonalised (twice) against the other columns, so the factor keeps
    // orthonormal columns (Theorem 2.2: U^* U = I) while A = U S V^* still holds to that level.
    double smax = 0.0;
    for (int k = 0; k < n; ++k) smax = fmax(smax, wgt[k]);
    const double thr = smax * 1e-6;
    for (int idx = tid; idx < m * n; idx += blockDim.x) {
      const int j = idx / m;
      const double sg = wgt[j];
      const double inv = sg > thr ? 1.0 / sg : 0.0;
      a[idx] = make_double2(a[idx].x * inv, a[idx].y * inv);
    }
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < n; ++j) {
        if (wgt[j] > thr) continue;
        for (int e = 0; e < m; ++e) {                    // try e_0, e_1, ... until one survives
          double2* x = a + j * m;
          for (int i = 0; i < m; ++i) x[i] = make_double2(i == e ? 1.0 : 0.0, 0.0);
          for (int pass = 0; pass < 2; ++pass)
            for (int k = 0; k < n; ++k) {
              if (k == j) continue;
              const double2* y = a + k * m;              // (zero columns still pending contribute nothing)
              double pr = 0.0, pi = 0.0;                 // <y, x> = y^H x
              for (int i = 0; i < m; ++i) {
                pr += y[i].x * x[i].x + y[i].y * x[i].y;
                pi += y[i].x * x[i].y - y[i].y * x[i].x;
              }
              for (int i = 0; i < m; ++i)
                x[i] = make_double2(x[i].x - (pr * y[i].x - pi * y[i].y), x[i].y - (pr * y[i].y + pi * y[i].x));
            }
          double nn = 0.0;
          for (int i = 0; i < m; ++i) nn += x[i].x * x[i].x + x[i].y * x[i].y;
          if (nn > 0.25) {
            const double inv = 1.0 / sqrt(nn);
            for (int i = 0; i < m; ++i) x[i] = make_double2(x[i].x * inv, x[i].y * inv);
            break;
          }
        }
      }
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
      int pos = 0;
      for (int k = 0; k < n; ++k) pos += (wgt[k] > wgt[j]) || (wgt[k] == wgt[j] && k < j);
      const double sg = wgt[j];
      const double inv = 1.0;                            // columns already normalised above
      fo.sre[so + (int64_t)pos * r + pos] = (float)sg;
      // left vectors: length m (rows of the processed matrix), right: length n
      float* lre = tr ? fo.vre + vo : fo.ure + uo;        // left vectors of the processed matrix
      float* lim = tr ? fo.vim + vo : fo.uim + uo;
      float* rre = tr ? fo.ure + uo : fo.vre + vo;
      float* rim = tr ? fo.uim + uo : fo.vim + vo;
      for (int i = 0; i < m; ++i) {
        const double2 x = a[j * m + i];
        lre[(int64_t)pos * m + i] = (float)(x.x * inv);
        lim[(int64_t)pos * m + i] = (float)(x.y * inv);
      }
      for (int i = 0; i < n; ++i) {
        const double2 y = v[j * n + i];
        rre[(int64_t)pos * n + i] = (float)y.x;
        rim[(int64_t)pos * n + i] = (float)y.y;
      }
    }
    return;
  }
  // W = (A V) diag(w) V^H : W(i, k) = sum_j a_j[i] w_j conj(v_j[k])
  float* orr = wre + (int64_t)f * fstride;
  float* oii = wim + (int64_t)f * fstride;
  for (int idx = tid; idx < m * n; idx += blockDim.x) {
    const int k = idx / m, i = idx - k * m;
    double xr = 0.0, xi = 0.0;
    for (int j = 0; j < n; ++j) {
      const double w = wgt[j];
      if (w == 0.0) continue;
      const double2 x = a[j * m + i], y = v[j * n + k];
      xr += w * (x.x * y.x + x.y * y.y);                // x * conj(y)
      xi += w * (x.y * y.x - x.x * y.y);
    }
    if (!tr) {
      orr[idx] = (float)xr;
      oii[idx] = (float)xi;
    } else {                                            // W = (W')^H: W(k, i) = conj(W'(i, k))
      orr[(int64_t)i * M + k] = (float)xr;
      oii[(int64_t)i * M + k] = -(float)xi;
    }
  }
}

bool svt_supported(int64_t m, int64_t n) { return m >= 1 && n >= 1 && m <= SVT_MAX && n <= SVT_MAX; }

// One CTA per slice.  G lanes per column pair: a pair's reductions and angle are warp-instruction
// overhead shared by the 32/G pairs of a warp, so narrow groups cut the instruction count (the
// iteration is issue-bound on one SM); columns are max(m, n) <= 64 long.  The pairs of a round
// (ceil(min(m, n) / 2)) fill ceil(pairs * G / 32) warps.
static int launch_svt_common(const float* re, const float* im, float* wre, float* wim, int64_t m, int64_t n,
                             int64_t h, int64_t fstride, float tau, double* sv, SvdOut fo, int* status,
                             cudaStream_t s) {
  if (!svt_supported(m, n)) return 6;
  // the slice (m n) and, unless only singular values are wanted, V (r x r, r = min(m, n))
  const int64_t len = std::max(m, n), r = std::min(m, n), pairs = (r + 1) / 2;
  const size_t smem = sizeof(double2) * (size_t)(n * m + (sv ? 0 : r * r));
  int G = len > 32 ? 16 : 8;
  if (const char* e = getenv("TPROD_SVT_GROUP")) {     // tuning override (G = 8 needs columns <= 32)
    const int g = atoi(e);
    if ((g == 8 && len <= 32) || g == 16 || g == 32) G = g;
  }
  int threads = (int)(((pairs * G + 31) / 32) * 32);
  if (threads < 64) threads = 64;
  auto go = [&](auto kern) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 4;
    kern<<<(unsigned)h, threads, smem, s>>>(re, im, wre, wim, (int)m, (int)n, fstride, tau, sv, fo, status);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
  };
  return G == 8 ? go(slice_svt_kernel<8>) : G == 16 ? go(slice_svt_kernel<16>) : go(slice_svt_kernel<32>);
}

int launch_slice_svt(const float* re, const float* im, float* wre, float* wim, int64_t m, int64_t n, int64_t h,
                     int64_t fstride, float tau, int* status, cudaStream_t s) {
  return launch_svt_common(re, im, wre, wim, m, n, h, fstride, tau, nullptr,
                           SvdOut{nullptr, nullptr, nullptr, nullptr, nullptr}, status, s);
}

// t-SVD scalars (NEXT-3).  sv: [h][r] per-slice singular values (r = min(m, n), non-increasing).
// out[0..r) = S(i, i, 1) = (1/n3) sum_{j < n3} S-bar(i, i, j) (Eq. (14)) with the conjugate pairs
// j, n3 - j sharing singular values (Eq. (8)); out[r] = TNN = sum_i S(i,i,1) (Def. 2.9);
// out[r+1] = TSN = max_j S-bar(1, 1, j) (Def. 2.8, Eq. (17)); out[r+2] = #{i : S(i,i,1) > rtol S(1,1,1)}
// (Eq. (16)).  One CTA.
__global__ void tsvd_reduce_kernel(const double* __restrict__ sv, int r, int h, int n3, float rtol,
                                   float* __restrict__ out) {
  __shared__ double s[SVT_MAX];
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double acc = 0.0;
    for (int f = 0; f < h; ++f) {
      const double w = (f == 0 || 2 * f == n3) ? 1.0 : 2.0;
      acc += w * sv[(int64_t)f * r + i];
    }
    s[i] = acc / n3;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tnn = 0.0, tsn = 0.0;
    int rank = 0;
    for (int i = 0; i < r; ++i) {
      tnn += s[i];
      out[i] = (float)s[i];
      if (s[0] > 0.0 && s[i] > (double)rtol * s[0]) ++rank;
    }
    for (int f = 0; f < h; ++f) tsn = fmax(tsn, sv[(int64_t)f * r]);
    out[r] = (float)tnn;
    out[r + 1] = (float)tsn;
    out[r + 2] = (float)rank;
  }
}

int launch_slice_svd_factors(const float* re, const float* im, int64_t m, int64_t n, int64_t h, int64_t fstride,
                             float* ure, float* uim, float* sre, float* vre, float* vim, int* status, cudaStream_t s) {
  return launch_svt_common(re, im, nullptr, nullptr, m, n, h, fstride, 0.f, nullptr, SvdOut{ure, uim, sre, vre, vim},
                           status, s);
}

int launch_tsvd_values(const float* re, const float* im, int64_t m, int64_t n, int64_t h, int64_t n3, int64_t fstride,
                       double* sv, float rtol, float* out, int* status, cudaStream_t s) {
  const int rc = launch_svt_common(re, im, nullptr, nullptr, m, n, h, fstride, 0.f, sv,
                                   SvdOut{nullptr, nullptr, nullptr, nullptr, nullptr}, status, s);
  if (rc) return rc;
  tsvd_reduce_kernel<<<1, 64, 0, s>>>(sv, (int)std::min(m, n), (int)h, (int)n3, rtol, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tprod
