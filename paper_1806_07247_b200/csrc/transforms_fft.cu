// Long-tube mode-3 transforms (power-of-two 64 < n3 <= 16384, e.g. config 4's n3 = 4096):
// in-shared-memory Stockham FFT, O(n3 log n3) per tube, radix-16 passes with the
// 16-point DFTs held in registers (a final radix-8/4/2 pass when log2 n3 is not a multiple of 4).
//
// Two real tubes x, y share one complex FFT z = x + i y (real-input packing):
//   forward  (Alg. 1 step 1, L174):  X_f = (Z_f + conj Z_{N-f}) / 2,  Y_f = (Z_f - conj Z_{N-f}) / (2i),
//            f = 0..N/2 only (Hermitian half, Eq. (8)), then the exact 2^e scaling and the
//            fp16 hi/lo split of the GEMM operand format;
//   inverse  (Alg. 1 step 2b + 3, L177-179): the conjugate fill X_{N-f} = conj X_f is built while
//            loading (Im of DC/Nyquist dropped), Z = X + i Y, z = IFFT(Z) (sign +, 1/N), x = Re z,
//            y = Im z.
// A CTA (512 threads) owns TUB = 2F consecutive tubes, F complex FFTs of N points with F*N = 16384
// (128 KB of data + 1/16 bank padding), so every global row access touches TUB consecutive
// elements of the contiguous dimension (float4-vectorised when aligned).
//
// Stockham pass (radix R, current span Ns), butterfly j in [0, N/R):
//   v[r] = z[j + r N/R] * w_N^{r k N/(Ns R)},  k = j mod Ns;   v = DFT_R(v);
//   z[(j - k) R + k + r Ns] = v[r]
// Every thread loads all of its butterflies into registers, the CTA synchronises, then writes
// (in place).  Output is in natural order.  Twiddles come from the handle's fp64-derived table
// (exact quadrant reduction), read through L1; the DFT_R constants are fp64 literals rounded to fp32.
#include "internal.h"
#include "common.cuh"

namespace tprod {

namespace {

constexpr int FFT_POINTS = 16384;        // complex points held in smem per CTA (128 KB)
constexpr int FFT_THREADS = 512;       // forward kernel
constexpr int IFFT_THREADS = 1024;     // inverse kernel (measured: 512 better for K1, 1024 for K3)

// padded smem index: one float2 of padding per 16 (breaks the radix-16 store stride)
__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int n) { return n + n / 16; }
// float2 stride between the F buffers of a CTA: the padded length rounded to 16, plus 16/F (>= 1)
// so that the F buffers of a half-warp's (f, c) items start in different banks
__host__ __device__ constexpr int bstride(int n) {
  return (padded_len(n) + 15) / 16 * 16 + ((16 * n / FFT_POINTS) > 1 ? 16 * n / FFT_POINTS : 1);
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// w_M^i = exp(DIR * 2 pi i * i / M) for M <= 16, DIR = -1 forward / +1 inverse
template <int DIR>
__device__ __forceinline__ float2 wconst(int M, int i) {
  // cos / sin of 2 pi i / M for M | 16, from fp64 literals (compile-time after unrolling)
  constexpr double C16[16] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
                              0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
                              -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
                              0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};
  const int m = i * (16 / M);
  const float c = (float)C16[m & 15];
  const float s = (float)C16[(m + 12) & 15];      // sin(x) = cos(x - pi/2)
  return make_float2(c, DIR < 0 ? -s : s);
}

// In-register DFT of R = 2^m points (radix-2 DIF, bit-reversed result reordered by renaming).
template <int R, int DIR>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * half) {
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float2 a = v[blk + i], b = v[blk + i + half];
        v[blk + i] = cadd(a, b);
        const float2 d = csub(a, b);
        if (i == 0) {
          v[blk + i + half] = d;
        } else if (4 * i == 2 * half) {            // w = -+i
          v[blk + i + half] = DIR < 0 ? make_float2(d.y, -d.x) : make_float2(-d.y, d.x);
        } else {
          v[blk + i + half] = cmul(d, wconst<DIR>(2 * half, i));
        }
      }
    }
  }
  float2 t[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int r = 0;
#pragma unroll
    for (int b = 1; b < R; b <<= 1) r = (r << 1) | ((k & b) ? 1 : 0);   // bit reversal of k
    t[k] = v[r];
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = t[k];
}

// table twiddle (cos, DIR*sin)
template <int DIR>
__device__ __forceinline__ float2 twN(const float2* __restrict__ tw, int m) {
  const float2 t = __ldg(tw + m);
  return make_float2(t.x, DIR < 0 ? -t.y : t.y);
}

// One Stockham pass of radix R over all F buffers (F*N = FFT_POINTS).
template <int R, int DIR, int NT>
__device__ __forceinline__ void stockham_pass(float2* z, int N, int logN, int Ns, int logNs,
                                              const float2* __restrict__ tp) {
  constexpr int BPT = FFT_POINTS / R / NT;            // butterflies per thread
  const int logR = R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1));
  const int nb_log = logN - logR;                     // log2(N / R)
  const int Np = bstride(N);
  float2 v[BPT][R];
  int dst[BPT], cb[BPT];
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int b = threadIdx.x + u * NT;
    const int c = b >> nb_log, j = b & ((1 << nb_log) - 1);
    const int k = j & (Ns - 1);
    float2* zc = z + c * Np;
#pragma unroll
    for (int r = 0; r < R; ++r) v[u][r] = zc[pad(j + (r << nb_log))];
    if (Ns > 1) {
      // w_{Ns R}^{r k} = tp[(r - 1) Ns + k]: consecutive k of a warp read consecutive entries
#pragma unroll
      for (int r = 1; r < R; ++r) v[u][r] = cmul(v[u][r], twN<DIR>(tp, (r - 1) * Ns + k));
    }
    dft_reg<R, DIR>(v[u]);
    cb[u] = c * Np;
    dst[u] = ((j - k) << logR) + k;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
#pragma unroll
    for (int r = 0; r < R; ++r) z[cb[u] + pad(dst[u] + r * Ns)] = v[u][r];
  }
  __syncthreads();
}

// Passes: radix 16 while >= 4 bits remain, then one radix 8/4/2 pass.  The table of the pass with
// span Ns > 1 and radix R starts after those of the earlier passes (Ns' R' - Ns' entries each).
template <int DIR, int NT>
__device__ void fft_smem(float2* z, int N, int logN, const float2* __restrict__ st) {
  int Ns = 1, logNs = 0;
  const float2* tp = st;
  while (logN - logNs >= 4) {
    stockham_pass<16, DIR, NT>(z, N, logN, Ns, logNs, tp);
    if (Ns > 1) tp += 15 * Ns;
    Ns <<= 4;
    logNs += 4;
  }
  const int rem = logN - logNs;
  if (rem == 3) stockham_pass<8, DIR, NT>(z, N, logN, Ns, logNs, tp);
  else if (rem == 2) stockham_pass<4, DIR, NT>(z, N, logN, Ns, logNs, tp);
  else if (rem == 1) stockham_pass<2, DIR, NT>(z, N, logN, Ns, logNs, tp);
}

template <int ROLE>
__global__ void __launch_bounds__(FFT_THREADS, 1) fft_fwd_split_kernel(
    const float* __restrict__ X, int64_t P, int64_t Q, int N, int logN,
    const unsigned* __restrict__ maxbits, const float2* __restrict__ st, __half* __restrict__ out,
    int64_t ld, float* __restrict__ unscale, int vec) {
  extern __shared__ float2 z[];
  const int F = FFT_POINTS >> logN, TUB = 2 * F;
  const int Np = bstride(N);
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int64_t PQ = P * Q;
  const float* x = X + P * q + p0;
  // ---- load: tube t = p0 + t, element k -> buffer t/2, real (t even) / imaginary (t odd) part
  if (vec) {   // TUB % 4 == 0, P % 4 == 0, 16-byte aligned, full block
    const int V = TUB >> 2;                         // float4 per row
    const int total = V * N;
#pragma unroll 8
    for (int idx = threadIdx.x; idx < total; idx += FFT_THREADS) {
      const int vv = idx % V, k = idx / V;
      const float4 a = __ldg(reinterpret_cast<const float4*>(x + PQ * k) + vv);
      z[(2 * vv) * Np + pad(k)] = make_float2(a.x, a.y);
      z[(2 * vv + 1) * Np + pad(k)] = make_float2(a.z, a.w);
    }
  } else {
    for (int idx = threadIdx.x; idx < TUB * N; idx += FFT_THREADS) {
      const int t = idx % TUB, k = idx / TUB;
      const float v = (p0 + t < P) ? __ldg(x + PQ * k + t) : 0.f;
      reinterpret_cast<float*>(z + (t >> 1) * Np + pad(k))[t & 1] = v;
    }
  }
  __syncthreads();
  fft_smem<-1, FFT_THREADS>(z, N, logN, st);
  // ---- Hermitian half, real-pair separation, 2^e scaling, fp16 hi/lo split
  const int H = N / 2 + 1;
  const int64_t plane = Q * ld;
  // FFT_THREADS % F == 0: every item of this thread has the same c, hence the same two tubes
  const int c = threadIdx.x % F;
  const int64_t p = p0 + 2 * c;
  const bool two = p + 1 < P;
  int e0 = 0, e1 = 0;
  if (p < P) {
    if (ROLE == 0) {
      e0 = scale_exp(__ldg(maxbits + p), N);
      e1 = two ? scale_exp(__ldg(maxbits + p + 1), N) : 0;
      if (q == 0) {
        unscale[p] = pow2f(-e0);
        if (two) unscale[p + 1] = pow2f(-e1);
      }
    } else {
      e0 = e1 = scale_exp(__ldg(maxbits + q), N);
      if (p0 == 0 && c == 0) unscale[q] = pow2f(-e0);
    }
  }
  const float s0 = pow2f(e0), s1 = pow2f(e1);
  for (int idx = threadIdx.x; idx < H * F; idx += FFT_THREADS) {
    const int f = idx / F;
    if (p >= P) break;
    const float2 zf = z[c * Np + pad(f)];
    const float2 zm = z[c * Np + pad((N - f) & (N - 1))];
    // X_f = (Z_f + conj Z_{N-f}) / 2 ;  Y_f = (Z_f - conj Z_{N-f}) / (2i)
    const float xr = 0.5f * (zf.x + zm.x), xi = 0.5f * (zf.y - zm.y);
    const float yr = 0.5f * (zf.y + zm.y), yi = -0.5f * (zf.x - zm.x);
    __half* o = out + q * ld + p;
    __half h0, l0, h1, l1;
    __half* ore = o + (int64_t)(4 * f) * plane;
    split_f16(xr * s0, h0, l0);
    split_f16(yr * s1, h1, l1);
    if (two && ((p & 1) == 0)) {
      *reinterpret_cast<__half2*>(ore + PL_RE_HI * plane) = __halves2half2(h0, h1);
      *reinterpret_cast<__half2*>(ore + PL_RE_LO * plane) = __halves2half2(l0, l1);
    } else {
      ore[PL_RE_HI * plane] = h0;
      ore[PL_RE_LO * plane] = l0;
      if (two) { ore[PL_RE_HI * plane + 1] = h1; ore[PL_RE_LO * plane + 1] = l1; }
    }
    split_f16(xi * s0, h0, l0);
    split_f16(yi * s1, h1, l1);
    if (two && ((p & 1) == 0)) {
      *reinterpret_cast<__half2*>(ore + PL_IM_HI * plane) = __halves2half2(h0, h1);
      *reinterpret_cast<__half2*>(ore + PL_IM_LO * plane) = __halves2half2(l0, l1);
    } else {
      ore[PL_IM_HI * plane] = h0;
      ore[PL_IM_LO * plane] = l0;
      if (two) { ore[PL_IM_HI * plane + 1] = h1; ore[PL_IM_LO * plane + 1] = l1; }
    }
  }
}

__global__ void __launch_bounds__(IFFT_THREADS, 1) fft_inv_kernel(const float* __restrict__ Cre,
                                                                const float* __restrict__ Cim, int64_t ld,
                                                                int64_t fstride, int64_t P, int64_t Q,
                                                                int N, int logN,
                                                                const float2* __restrict__ st,
                                                                float* __restrict__ X, int vec) {
  extern __shared__ float2 z[];
  const int F = FFT_POINTS >> logN, TUB = 2 * F;
  const int Np = bstride(N);
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int H = N / 2 + 1;
  // ---- Z = X + iY with the conjugate fill, natural order
  for (int idx = threadIdx.x; idx < H * F; idx += IFFT_THREADS) {
    const int c = idx % F, f = idx / F;
    const int64_t p = p0 + 2 * c;
    float xr = 0.f, xi = 0.f, yr = 0.f, yi = 0.f;
    const float* cr = Cre + fstride * f + q * ld + p;
    const float* ci = Cim + fstride * f + q * ld + p;
    const bool self = (f == 0 || 2 * f == N);        // DC / Nyquist: imaginary part dropped (C2R)
    if (vec) {                                       // p even, ld even, both tubes in range
      const float2 r2 = __ldg(reinterpret_cast<const float2*>(cr));
      xr = r2.x; yr = r2.y;
      if (!self) { const float2 i2 = __ldg(reinterpret_cast<const float2*>(ci)); xi = i2.x; yi = i2.y; }
    } else {
      if (p < P) { xr = __ldg(cr); if (!self) xi = __ldg(ci); }
      if (p + 1 < P) { yr = __ldg(cr + 1); if (!self) yi = __ldg(ci + 1); }
    }
    z[c * Np + pad(f)] = make_float2(xr - yi, xi + yr);                 // X_f + i Y_f
    if (!self) z[c * Np + pad(N - f)] = make_float2(xr + yi, yr - xi);  // conj X_f + i conj Y_f
  }
  __syncthreads();
  fft_smem<+1, IFFT_THREADS>(z, N, logN, st);
  const float inv_n = 1.f / (float)N;
  const int64_t PQ = P * Q;
  float* xo = X + P * q + p0;
  if (vec && (TUB % 4) == 0 && p0 + TUB <= P && (P % 4) == 0 && (((uintptr_t)X) & 15) == 0) {
    const int V = TUB >> 2;
    const int total = V * N;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < total; idx += IFFT_THREADS) {
      const int vv = idx % V, k = idx / V;
      const float2 a = z[(2 * vv) * Np + pad(k)], b = z[(2 * vv + 1) * Np + pad(k)];
      reinterpret_cast<float4*>(xo + PQ * k)[vv] = make_float4(a.x * inv_n, a.y * inv_n, b.x * inv_n, b.y * inv_n);
    }
  } else {
    for (int idx = threadIdx.x; idx < TUB * N; idx += IFFT_THREADS) {
      const int t = idx % TUB, k = idx / TUB;
      if (p0 + t >= P) continue;
      const float2 v = z[(t >> 1) * Np + pad(k)];
      xo[PQ * k + t] = ((t & 1) == 0 ? v.x : v.y) * inv_n;
    }
  }
}

int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

size_t fft_smem_bytes(int N) { return sizeof(float2) * (size_t)(FFT_POINTS / N) * bstride(N); }

bool fft_smem_ok(const void* kern, int N) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem_bytes(N)) ==
         cudaSuccess;
}

}  // namespace

size_t stockham_table_len(int n) {
  size_t len = 0;
  int Ns = 1;
  int rem = 0;
  while ((1 << rem) < n) ++rem;          // log2 n
  while (rem > 0) {
    const int R = rem >= 4 ? 16 : (1 << rem);
    if (Ns > 1) len += (size_t)(R - 1) * Ns;
    Ns *= R;
    rem -= rem >= 4 ? 4 : rem;
  }
  return len;
}

void host_stockham_table(int n, const double* cs, float2* out) {
  int Ns = 1, rem = 0;
  while ((1 << rem) < n) ++rem;
  size_t o = 0;
  while (rem > 0) {
    const int R = rem >= 4 ? 16 : (1 << rem);
    if (Ns > 1) {
      for (int r = 1; r < R; ++r)
        for (int k = 0; k < Ns; ++k) {
          const long long m = (long long)r * k * (n / (Ns * R));   // w_{Ns R}^{r k} = w_n^m, m < n
          out[o++] = make_float2((float)cs[2 * m], (float)cs[2 * m + 1]);
        }
    }
    Ns *= R;
    rem -= rem >= 4 ? 4 : rem;
  }
}

bool fft_supported(int64_t n3) {
  return n3 > 64 && n3 <= FFT_POINTS && (n3 & (n3 - 1)) == 0;
}

bool launch_fwd_fft(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    const float2* st, __half* out, int64_t ld, float* unscale, cudaStream_t s) {
  if (!fft_supported(n3)) return false;
  const int N = (int)n3, logN = ilog2(n3);
  const int TUB = 2 * (FFT_POINTS / N);
  const size_t smem = fft_smem_bytes(N);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  // vectorised loads need every block full and 16-byte aligned rows
  const int vec = (TUB % 4 == 0) && (P % TUB == 0) && (((uintptr_t)X) & 15) == 0;
  const void* k = role == 0 ? (const void*)fft_fwd_split_kernel<0> : (const void*)fft_fwd_split_kernel<1>;
  if (!fft_smem_ok(k, N)) return false;
  if (role == 0)
    fft_fwd_split_kernel<0><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, logN, maxbits, st, out, ld,
                                                                       unscale, vec);
  else
    fft_fwd_split_kernel<1><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, logN, maxbits, st, out, ld,
                                                                       unscale, vec);
  return cudaGetLastError() == cudaSuccess;
}

bool launch_inv_fft(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P, int64_t Q,
                    int64_t n3, const float2* st, float* X, cudaStream_t s) {
  if (!fft_supported(n3)) return false;
  const int N = (int)n3, logN = ilog2(n3);
  const int TUB = 2 * (FFT_POINTS / N);
  const size_t smem = fft_smem_bytes(N);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  // paired float2 loads of C-bar need both tubes of every pair in range and 8-byte alignment
  const int vec = (P % TUB == 0) && (ld % 2 == 0) && (fstride % 2 == 0) && (((uintptr_t)Cre) & 7) == 0 &&
                  (((uintptr_t)Cim) & 7) == 0;
  if (!fft_smem_ok((const void*)fft_inv_kernel, N)) return false;
  fft_inv_kernel<<<(unsigned)blocks, IFFT_THREADS, smem, s>>>(Cre, Cim, ld, fstride, P, Q, N, logN, st, X, vec);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace tprod
