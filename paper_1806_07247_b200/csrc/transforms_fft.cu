// Long-tube mode-3 transforms (power-of-two n3 > 64, e.g. config 4's n3 = 4096): in-shared-memory
// radix-4 (+ one radix-2) decimation-in-frequency FFT, O(n3 log n3) per tube.
//
// Two real tubes x, y share one complex FFT z = x + i y (real-input packing):
//   forward  (Alg. 1 step 1, L174):  X_f = (Z_f + conj Z_{N-f}) / 2,  Y_f = (Z_f - conj Z_{N-f}) / (2i),
//            f = 0..N/2 only (Hermitian half, Eq. (8)), then the exact 2^e scaling and the
//            fp16 hi/lo split of the GEMM operand format;
//   inverse  (Alg. 1 step 2b + 3, L177-179): the conjugate fill X_{N-f} = conj X_f is built in
//            shared memory (Im of DC/Nyquist dropped), Z = X + i Y, z = conj(FFT(conj Z)) / N,
//            x = Re z, y = Im z.
// A CTA owns TUB = 2F consecutive tubes (F complex FFTs of N points, F*N = 16384 -> 128 KB smem),
// so every global load/store touches TUB consecutive elements of the contiguous dimension.
// Twiddles come from the handle's fp64-derived table (exact quadrant reduction), read through L1.
#include "internal.h"
#include "common.cuh"

namespace tprod {

constexpr int FFT_POINTS = 16384;        // complex points held in smem per CTA (128 KB)
constexpr int FFT_THREADS = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// forward twiddle w^m = e^{-2 pi i m/N} from the (cos, sin) table
__device__ __forceinline__ float2 twf(const float2* __restrict__ tw, int m) {
  float2 t = __ldg(tw + m);
  return make_float2(t.x, -t.y);
}

// In-place DIF FFT (forward sign) of F buffers of N points; buffer c starts at s + c*(N+1).
// Stages: radix 4 while the span is divisible by 4, then a final radix 2 if log2 N is odd.
// Result: frequency f at position pos_of(f).
__device__ void fft_dif_inplace(float2* s, int N, int logN, int F, const float2* __restrict__ tw) {
  const int stride_buf = N + 1;
  int L = N, scale = 1;                   // span of the current stage, twiddle index multiplier
  while (L >= 4) {
    const int Lq = L >> 2;
    const int nbf = F * (N >> 2);         // butterflies in this stage (all buffers)
    for (int b = threadIdx.x; b < nbf; b += blockDim.x) {
      const int c = b / (N >> 2);
      const int r = b - c * (N >> 2);
      const int g = r / Lq, j = r - g * Lq;
      float2* base = s + c * stride_buf + g * L + j;
      const float2 x0 = base[0], x1 = base[Lq], x2 = base[2 * Lq], x3 = base[3 * Lq];
      const float2 a0 = make_float2(x0.x + x2.x, x0.y + x2.y), a1 = make_float2(x0.x - x2.x, x0.y - x2.y);
      const float2 b0 = make_float2(x1.x + x3.x, x1.y + x3.y), b1 = make_float2(x1.x - x3.x, x1.y - x3.y);
      // -i * b1 = (b1.y, -b1.x)
      const float2 y0 = make_float2(a0.x + b0.x, a0.y + b0.y);
      const float2 y2 = make_float2(a0.x - b0.x, a0.y - b0.y);
      const float2 y1 = make_float2(a1.x + b1.y, a1.y - b1.x);
      const float2 y3 = make_float2(a1.x - b1.y, a1.y + b1.x);
      base[0] = y0;
      if (j == 0) {
        base[Lq] = y1;
        base[2 * Lq] = y2;
        base[3 * Lq] = y3;
      } else {
        base[Lq] = cmul(y1, twf(tw, (j * scale) & (N - 1)));
        base[2 * Lq] = cmul(y2, twf(tw, (2 * j * scale) & (N - 1)));
        base[3 * Lq] = cmul(y3, twf(tw, (3 * j * scale) & (N - 1)));
      }
    }
    __syncthreads();
    L = Lq;
    scale <<= 2;
  }
  if (L == 2) {
    const int nbf = F * (N >> 1);
    for (int b = threadIdx.x; b < nbf; b += blockDim.x) {
      const int c = b / (N >> 1);
      const int g = b - c * (N >> 1);
      float2* base = s + c * stride_buf + 2 * g;
      const float2 x0 = base[0], x1 = base[1];
      base[0] = make_float2(x0.x + x1.x, x0.y + x1.y);
      base[1] = make_float2(x0.x - x1.x, x0.y - x1.y);
    }
    __syncthreads();
  }
}

// position of frequency f after fft_dif_inplace: f = m0 + 4 m1 + 16 m2 + ... (+ 4^S m_last for
// the radix-2 stage); position = sum m_s * (span_s / radix_s)
__device__ __forceinline__ int pos_of(int f, int N, int logN) {
  int pos = 0, L = N;
  while (L >= 4) {
    L >>= 2;
    pos += (f & 3) * L;
    f >>= 2;
  }
  if (L == 2) pos += f & 1;
  return pos;
}

template <int ROLE>
__global__ void __launch_bounds__(FFT_THREADS) fft_fwd_split_kernel(
    const float* __restrict__ X, int64_t P, int64_t Q, int N, int logN,
    const unsigned* __restrict__ maxbits, const float2* __restrict__ tw, __half* __restrict__ out,
    int64_t ld, float* __restrict__ unscale) {
  extern __shared__ float2 sz[];
  const int F = FFT_POINTS / N, TUB = 2 * F;
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int64_t PQ = P * Q;
  const float* x = X + P * q + p0;
  // load: element (tube t, k) -> buffer t/2, real (t even) or imaginary (t odd) part
  for (int idx = threadIdx.x; idx < TUB * N; idx += blockDim.x) {
    const int t = idx % TUB, k = idx / TUB;
    const float v = (p0 + t < P) ? __ldg(x + PQ * k + t) : 0.f;
    float* d = reinterpret_cast<float*>(sz + (t >> 1) * (N + 1) + k);
    d[t & 1] = v;
  }
  __syncthreads();
  fft_dif_inplace(sz, N, logN, F, tw);
  const int H = N / 2 + 1;
  const int64_t plane = Q * ld;
  int eq = 0;
  if (ROLE == 1) eq = scale_exp(__ldg(maxbits + q), N);
  for (int idx = threadIdx.x; idx < H * TUB; idx += blockDim.x) {
    const int t = idx % TUB, f = idx / TUB;
    const int64_t p = p0 + t;
    if (p >= P) continue;
    const int c = t >> 1;
    const float2 zf = sz[c * (N + 1) + pos_of(f, N, logN)];
    const float2 zm = sz[c * (N + 1) + pos_of((N - f) & (N - 1), N, logN)];
    float re, im;
    if ((t & 1) == 0) {        // X_f = (Z_f + conj Z_{N-f}) / 2
      re = 0.5f * (zf.x + zm.x);
      im = 0.5f * (zf.y - zm.y);
    } else {                   // Y_f = (Z_f - conj Z_{N-f}) / (2i)
      re = 0.5f * (zf.y + zm.y);
      im = -0.5f * (zf.x - zm.x);
    }
    const int e = ROLE == 0 ? scale_exp(__ldg(maxbits + p), N) : eq;
    if (f == 0 && (ROLE == 0 ? q == 0 : p == 0)) unscale[ROLE == 0 ? p : q] = pow2f(-e);
    const float sc = pow2f(e);
    __half hi, lo;
    __half* o = out + q * ld + p;
    split_f16(re * sc, hi, lo);
    o[(int64_t)(4 * f + PL_RE_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_RE_LO) * plane] = lo;
    split_f16(im * sc, hi, lo);
    o[(int64_t)(4 * f + PL_IM_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_IM_LO) * plane] = lo;
  }
}

__global__ void __launch_bounds__(FFT_THREADS) fft_inv_kernel(const float* __restrict__ Cre,
                                                             const float* __restrict__ Cim, int64_t ld,
                                                             int64_t fstride, int64_t P, int64_t Q,
                                                             int N, int logN,
                                                             const float2* __restrict__ tw,
                                                             float* __restrict__ X) {
  extern __shared__ float2 sz[];
  const int F = FFT_POINTS / N, TUB = 2 * F;
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int H = N / 2 + 1;
  // conj(Z) into smem, natural order, with the conjugate fill of f > N/2
  for (int idx = threadIdx.x; idx < H * TUB; idx += blockDim.x) {
    const int t = idx % TUB, f = idx / TUB;
    const int64_t p = p0 + t;
    float xr = 0.f, xi = 0.f;
    if (p < P) {
      xr = __ldg(Cre + fstride * f + q * ld + p);
      xi = (f == 0 || 2 * f == N) ? 0.f : __ldg(Cim + fstride * f + q * ld + p);   // C2R
    }
    float* zf = reinterpret_cast<float*>(sz + (t >> 1) * (N + 1) + f);
    float* zm = reinterpret_cast<float*>(sz + (t >> 1) * (N + 1) + ((N - f) & (N - 1)));
    // conj(Z_f) = conj(X_f) - i conj(Y_f);  conj(Z_{N-f}) = X_f - i Y_f.  x-tube (t even)
    // contributes (xr, -xi) at f and (xr, xi) at N-f; y-tube (t odd) contributes (-yi, -yr) at f
    // and (yi, -yr) at N-f.  Both tubes of a pair write disjoint components -> combine via atomics-
    // free two-pass: even tubes first, then odd tubes add.
    if ((t & 1) == 0) {
      zf[0] = xr;
      zf[1] = -xi;
      if (f != 0 && 2 * f != N) {
        zm[0] = xr;
        zm[1] = xi;
      }
    }
    (void)zm;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < H * TUB; idx += blockDim.x) {
    const int t = idx % TUB, f = idx / TUB;
    if ((t & 1) == 0) continue;
    const int64_t p = p0 + t;
    float yr = 0.f, yi = 0.f;
    if (p < P) {
      yr = __ldg(Cre + fstride * f + q * ld + p);
      yi = (f == 0 || 2 * f == N) ? 0.f : __ldg(Cim + fstride * f + q * ld + p);
    }
    float* zf = reinterpret_cast<float*>(sz + (t >> 1) * (N + 1) + f);
    float* zm = reinterpret_cast<float*>(sz + (t >> 1) * (N + 1) + ((N - f) & (N - 1)));
    zf[0] += -yi;
    zf[1] += -yr;
    if (f != 0 && 2 * f != N) {
      zm[0] += yi;
      zm[1] += -yr;
    }
  }
  __syncthreads();
  fft_dif_inplace(sz, N, logN, F, tw);
  const float inv_n = 1.f / (float)N;
  const int64_t PQ = P * Q;
  float* xo = X + P * q + p0;
  for (int idx = threadIdx.x; idx < TUB * N; idx += blockDim.x) {
    const int t = idx % TUB, k = idx / TUB;
    if (p0 + t >= P) continue;
    const float2 v = sz[(t >> 1) * (N + 1) + pos_of(k, N, logN)];
    // z = conj(FFT(conj Z)) / N:  x = Re z = v.x / N,  y = Im z = -v.y / N
    xo[PQ * k + t] = ((t & 1) == 0 ? v.x : -v.y) * inv_n;
  }
}

static int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

bool fft_supported(int64_t n3) {
  return n3 > 64 && n3 <= FFT_POINTS && (n3 & (n3 - 1)) == 0;
}

static bool fft_smem_ok(const void* kern, int N) {
  const size_t smem = sizeof(float2) * (size_t)(FFT_POINTS / N) * (N + 1);
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
}

bool launch_fwd_fft(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    const float2* tw, __half* out, int64_t ld, float* unscale, cudaStream_t s) {
  if (!fft_supported(n3)) return false;
  const int N = (int)n3, logN = ilog2(n3);
  const int TUB = 2 * (FFT_POINTS / N);
  const size_t smem = sizeof(float2) * (size_t)(FFT_POINTS / N) * (N + 1);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  if (role == 0) {
    if (!fft_smem_ok((const void*)fft_fwd_split_kernel<0>, N)) return false;
    fft_fwd_split_kernel<0><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, logN, maxbits, tw, out, ld, unscale);
  } else {
    if (!fft_smem_ok((const void*)fft_fwd_split_kernel<1>, N)) return false;
    fft_fwd_split_kernel<1><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, logN, maxbits, tw, out, ld, unscale);
  }
  return cudaGetLastError() == cudaSuccess;
}

bool launch_inv_fft(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P, int64_t Q,
                    int64_t n3, const float2* tw, float* X, cudaStream_t s) {
  if (!fft_supported(n3)) return false;
  const int N = (int)n3, logN = ilog2(n3);
  const int TUB = 2 * (FFT_POINTS / N);
  const size_t smem = sizeof(float2) * (size_t)(FFT_POINTS / N) * (N + 1);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  if (!fft_smem_ok((const void*)fft_inv_kernel, N)) return false;
  fft_inv_kernel<<<(unsigned)blocks, FFT_THREADS, smem, s>>>(Cre, Cim, ld, fstride, P, Q, N, logN, tw, X);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace tprod
