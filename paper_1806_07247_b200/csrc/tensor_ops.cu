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

template <typename T>
void launch_tran(const T* A, T* At, int64_t n1, int64_t n2, int64_t n3, cudaStream_t s) {
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
      if (!(sqrtf(red_v[0]) > thresh)) atomicExch(singular, 1);
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
