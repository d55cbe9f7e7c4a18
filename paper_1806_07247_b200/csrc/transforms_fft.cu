// Long-tube mode-3 transforms (5-smooth 64 < n3 <= 16384, e.g. config 4's n3 = 4096): in-shared-
// memory mixed-radix Stockham FFT, O(n3 log n3) per tube (the mixed radix-2/3/5
// decomposition of the north star), radix-16 passes while the power-of-two part allows, then
// radix 8/4/2, then radix 3 and radix 5 passes, each R-point DFT held in registers.
//
// Two real tubes x, y share one complex FFT z = x + i y (real-input packing):
//   forward  (Alg. 1 step 1, L174):  X_f = (Z_f + conj Z_{N-f}) / 2,  Y_f = (Z_f - conj Z_{N-f}) / (2i),
//            f = 0..N/2 only (Hermitian half, Eq. (8)), then the exact 2^e scaling and the
//            fp16 hi/lo split of the GEMM operand format;
//   inverse  (Alg. 1 step 2b + 3, L177-179): the conjugate fill X_{N-f} = conj X_f is built while
//            loading (Im of DC/Nyquist dropped), Z = X + i Y, z = IFFT(Z) (sign +, 1/N), x = Re z,
//            y = Im z.
// A CTA owns TUB = 2F consecutive tubes, F = the largest power of two with F*N <= 16384 complex
// FFTs (<= 128 KB of data + 1/16 bank padding), so every global row access touches TUB consecutive
// elements of the contiguous dimension (float4-vectorised when aligned).
//
// Stockham pass (radix R, span Ns = product of the earlier radices), butterfly j in [0, N/R):
//   v[r] = z[j + r N/R] * w_{Ns R}^{r k},  k = j mod Ns;   v = DFT_R(v);
//   z[(j - k) R + k + r Ns] = v[r]
// Every thread loads all of its butterflies into registers, the CTA synchronises, then writes
// (in place).  Output is in natural order.  Twiddles w_{Ns R}^{r k} come from a per-pass table
// laid out [pass][r-1][k] (coalesced for consecutive k) built from the handle's fp64 table with
// exact quadrant reduction; the DFT_R constants are fp64 literals rounded to fp32.
#include "internal.h"
#include "common.cuh"
#include "fft_reg.cuh"

#include <complex>
#include <map>
#include <math.h>
#include <mutex>
#include <vector>

namespace tprod {

namespace {

using namespace fftreg;

constexpr int FFT_POINTS = 16384;      // complex points held in smem per CTA (128 KB; measured: 64 KB tiles are 1.3-1.6x slower)
constexpr int FFT_THREADS = 512;       // forward kernel
constexpr int IFFT_THREADS = 1024;     // inverse kernel (measured: 512 better for K1, 1024 for K3)
constexpr int MAX_PASSES = 16;

// Radix plan of N: radix-16 passes, one radix 8/4/2 pass for the rest of the power of two, then
// radix-3 and radix-5 passes.  Ns[i] = product of R[0..i-1]; toff[i] = offset of pass i's twiddle
// table ((R - 1) Ns entries, none for Ns = 1).
struct FftPlan {
  int np;
  int R[MAX_PASSES];
  int Ns[MAX_PASSES];
  int toff[MAX_PASSES];
};

bool make_plan(int n, FftPlan* pl) {
  if (n < 1) return false;
  int m = n, a = 0;
  while (m % 2 == 0) { m /= 2; ++a; }
  int b = 0, c = 0;
  while (m % 3 == 0) { m /= 3; ++b; }
  while (m % 5 == 0) { m /= 5; ++c; }
  if (m != 1) return false;
  std::vector<int> rs;
  while (a >= 4) { rs.push_back(16); a -= 4; }
  if (a > 0) rs.push_back(1 << a);
  for (int i = 0; i < b; ++i) rs.push_back(3);
  for (int i = 0; i < c; ++i) rs.push_back(5);
  if ((int)rs.size() > MAX_PASSES) return false;
  pl->np = (int)rs.size();
  int Ns = 1, off = 0;
  for (int i = 0; i < pl->np; ++i) {
    pl->R[i] = rs[i];
    pl->Ns[i] = Ns;
    pl->toff[i] = off;
    if (Ns > 1) off += (rs[i] - 1) * Ns;
    Ns *= rs[i];
  }
  return true;
}

int fft_F(int n) {             // complex FFTs per CTA: largest power of two with F * n <= FFT_POINTS
  int F = 1;
  while (2 * F * n <= FFT_POINTS) F *= 2;
  return F;
}

// padded smem index: one float2 of padding per 16 (breaks the radix-16 store stride)
__host__ __device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
// float2 stride between the F buffers of a CTA: the padded length rounded to 16, plus 16/F (>= 1)
// so that the F buffers of a half-warp's (f, c) items start in different banks
__host__ __device__ __forceinline__ int bstride(int n, int F) {
  const int pl = n + n / 16 + 1;
  return (pl + 15) / 16 * 16 + (16 / F > 1 ? 16 / F : 1);
}

// Largest F * N / R over the N this file handles (F * N <= 16384).
template <int R>
__host__ __device__ constexpr int max_butterflies() {
  return FFT_POINTS / R;
}

// Butterfly b of a pass -> (buffer c, butterfly j of that FFT, group g = j / Ns, k = j mod Ns).
// Power-of-two N uses shifts, other N integer division.
struct PassIdx {
  int c, j, g, k;
};
__device__ __forceinline__ PassIdx pass_idx(int b, int NB, int Ns, int lognb, int logns) {
  PassIdx x;
  if (lognb >= 0) {
    x.c = b >> lognb;
    x.j = b & (NB - 1);
    x.g = x.j >> logns;
    x.k = x.j & (Ns - 1);
  } else {
    x.c = b / NB;
    x.j = b - x.c * NB;
    x.g = x.j / Ns;
    x.k = x.j - x.g * Ns;
  }
  return x;
}

// One Stockham pass of radix R over all F buffers (buffer stride Np).  lognb / logns are log2 of
// N/R and Ns when N is a power of two, else -1.
template <int R, int DIR, int NT>
__device__ __forceinline__ void stockham_pass(float2* z, int N, int F, int Np, int Ns, int lognb, int logns,
                                              const float2* __restrict__ tp) {
  constexpr int BPT = (max_butterflies<R>() + NT - 1) / NT;   // butterflies per thread (upper bound)
  const int NB = N / R;                                        // butterflies per FFT
  const int total = F * NB;
  float2 v[BPT][R];
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    // past-the-end butterflies redo the last one (registers stay unconditionally defined; their
    // results are not stored)
    const int b = min((int)threadIdx.x + u * NT, total - 1);
    {
      const PassIdx x = pass_idx(b, NB, Ns, lognb, logns);
      const float2* zc = z + x.c * Np;
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = zc[pad(x.j + r * NB)];
      if (Ns > 1) {
        // w_{Ns R}^{r k} = tp[(r - 1) Ns + k]: consecutive k of a warp read consecutive entries
#pragma unroll
        for (int r = 1; r < R; ++r) v[u][r] = cmul(v[u][r], twN<DIR>(tp, (r - 1) * Ns + x.k));
      }
      dft_reg<R, DIR>(v[u]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int b = threadIdx.x + u * NT;
    if (b < total) {
      const PassIdx x = pass_idx(b, NB, Ns, lognb, logns);
      float2* zc = z + x.c * Np;
      const int d0 = x.g * Ns * R + x.k;
#pragma unroll
      for (int r = 0; r < R; ++r) zc[pad(d0 + r * Ns)] = v[u][r];
    }
  }
  __syncthreads();
}

template <int DIR, int NT>
__device__ void fft_smem(float2* z, int N, int F, int Np, const FftPlan& pl, const float2* __restrict__ st) {
  const bool p2 = (N & (N - 1)) == 0;
  for (int i = 0; i < pl.np; ++i) {
    const float2* tp = st + pl.toff[i];
    const int R = pl.R[i], Ns = pl.Ns[i];
    const int lognb = p2 ? __ffs(N / R) - 1 : -1, logns = p2 ? __ffs(Ns) - 1 : -1;
    switch (R) {
      case 16: stockham_pass<16, DIR, NT>(z, N, F, Np, Ns, lognb, logns, tp); break;
      case 8: stockham_pass<8, DIR, NT>(z, N, F, Np, Ns, lognb, logns, tp); break;
      case 4: stockham_pass<4, DIR, NT>(z, N, F, Np, Ns, lognb, logns, tp); break;
      case 2: stockham_pass<2, DIR, NT>(z, N, F, Np, Ns, lognb, logns, tp); break;
      case 3: stockham_pass<3, DIR, NT>(z, N, F, Np, Ns, -1, -1, tp); break;
      default: stockham_pass<5, DIR, NT>(z, N, F, Np, Ns, -1, -1, tp); break;
    }
  }
}

// Bluestein's chirp-z transform (for n3 that are not 5-smooth): the length-N DFT of each of the F
// buffers, Z_f = sum_k z_k w^{fk} (w = e^{-2 pi i/N}), through one length-M (5-smooth, M >= 2N - 1)
// cyclic convolution:  w^{fk} = c_f c_k / c_{f-k} with the chirp c_k = e^{-pi i k^2 / N}, so
//   Z_f = c_f sum_k (z_k c_k) b_{f-k},   b_m = e^{+pi i m^2 / N} = conj(c_m)
// and the sum is IFFT_M(FFT_M(z c) . FFT_M(b)) with b wrapped cyclically (bh = FFT_M(b) / M is
// precomputed in fp64).  In / out: z_k, k < N, at pad(k) of each buffer (stride Np >= padded M).
template <int NT>
__device__ void bluestein(float2* z, int N, int M, int F, int Np, const FftPlan& pl, const float2* __restrict__ st,
                          const float2* __restrict__ chirp, const float2* __restrict__ bh) {
  for (int idx = threadIdx.x; idx < F * M; idx += NT) {
    const int c = idx / M, k = idx - c * M;
    float2* e = z + c * Np + pad(k);
    *e = k < N ? cmul(*e, __ldg(chirp + k)) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  fft_smem<-1, NT>(z, M, F, Np, pl, st);
  for (int idx = threadIdx.x; idx < F * M; idx += NT) {
    const int c = idx / M, k = idx - c * M;
    float2* e = z + c * Np + pad(k);
    *e = cmul(*e, __ldg(bh + k));
  }
  __syncthreads();
  fft_smem<+1, NT>(z, M, F, Np, pl, st);
  for (int idx = threadIdx.x; idx < F * N; idx += NT) {
    const int c = idx / N, f = idx - c * N;
    float2* e = z + c * Np + pad(f);
    *e = cmul(*e, __ldg(chirp + f));
  }
  __syncthreads();
}

// Plan of one transform length: the FFT itself (M = 0) or Bluestein of length N through a
// length-M FFT (pl / st then describe M).
struct FftJob {
  int M;
  const float2* chirp;
  const float2* bh;
};

template <int DIR, int NT>
__device__ void fft_core(float2* z, int N, int F, int Np, const FftPlan& pl, const float2* __restrict__ st,
                         const FftJob& job) {
  if (!job.M) {
    fft_smem<DIR, NT>(z, N, F, Np, pl, st);
    return;
  }
  if (DIR < 0) {
    bluestein<NT>(z, N, job.M, F, Np, pl, st, job.chirp, job.bh);
  } else {                                            // inverse DFT = conj(DFT(conj z))
    for (int idx = threadIdx.x; idx < F * N; idx += NT) {
      float2* e = z + (idx / N) * Np + pad(idx % N);
      e->y = -e->y;
    }
    __syncthreads();
    bluestein<NT>(z, N, job.M, F, Np, pl, st, job.chirp, job.bh);
    for (int idx = threadIdx.x; idx < F * N; idx += NT) {
      float2* e = z + (idx / N) * Np + pad(idx % N);
      e->y = -e->y;
    }
    __syncthreads();
  }
}

template <int ROLE>
__global__ void __launch_bounds__(FFT_THREADS, 1) fft_fwd_split_kernel(
    const float* __restrict__ X, int64_t P, int64_t Q, int N, int F, const __grid_constant__ FftPlan pl,
    const unsigned* __restrict__ maxbits, const float2* __restrict__ st, __half* __restrict__ out,
    int64_t ld, float* __restrict__ unscale, int vec, FftJob job) {
  extern __shared__ float2 z[];
  const int TUB = 2 * F;
  const int Np = bstride(job.M ? job.M : N, F);
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int64_t PQ = P * Q;
  const float* x = X + P * q + p0;
  // A (ROLE 0): each tube's exact row scale is applied as it is loaded, before two tubes share one
  // complex FFT (neither tube's rounding is then large relative to the other's scale); B's pair
  // shares its column scale, applied after the FFT
  __shared__ float rsc[256];                      // TUB = 2F <= 256 (F * N <= FFT_POINTS, N > 64)
  if (ROLE == 0) {
    for (int t = threadIdx.x; t < TUB; t += FFT_THREADS)
      rsc[t] = p0 + t < P ? pow2f(scale_exp(__ldg(maxbits + p0 + t), N)) : 1.f;
    __syncthreads();
  }
  // ---- load: tube t = p0 + t, element k -> buffer t/2, real (t even) / imaginary (t odd) part
  if (vec) {   // TUB % 4 == 0, P % TUB == 0, 16-byte aligned
    const int V = TUB >> 2;                         // float4 per row
    const int total = V * N;
#pragma unroll 8
    for (int idx = threadIdx.x; idx < total; idx += FFT_THREADS) {
      const int vv = idx % V, k = idx / V;
      float4 a = __ldg(reinterpret_cast<const float4*>(x + PQ * k) + vv);
      if (ROLE == 0) {
        a.x *= rsc[4 * vv];
        a.y *= rsc[4 * vv + 1];
        a.z *= rsc[4 * vv + 2];
        a.w *= rsc[4 * vv + 3];
      }
      z[(2 * vv) * Np + pad(k)] = make_float2(a.x, a.y);
      z[(2 * vv + 1) * Np + pad(k)] = make_float2(a.z, a.w);
    }
  } else {
    for (int idx = threadIdx.x; idx < TUB * N; idx += FFT_THREADS) {
      const int t = idx % TUB, k = idx / TUB;
      float v = (p0 + t < P) ? __ldg(x + PQ * k + t) : 0.f;
      if (ROLE == 0) v *= rsc[t];
      reinterpret_cast<float*>(z + (t >> 1) * Np + pad(k))[t & 1] = v;
    }
  }
  __syncthreads();
  fft_core<-1, FFT_THREADS>(z, N, F, Np, pl, st, job);
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
        unscale[p] = unscale_of(__ldg(maxbits + p), e0);
        if (two) unscale[p + 1] = unscale_of(__ldg(maxbits + p + 1), e1);
      }
    } else {
      e0 = e1 = scale_exp(__ldg(maxbits + q), N);
      if (p0 == 0 && c == 0) unscale[q] = unscale_of(__ldg(maxbits + q), e0);
    }
  }
  const float s0 = ROLE == 0 ? 1.f : pow2f(e0), s1 = ROLE == 0 ? 1.f : pow2f(e1);   // A: applied at load
  if (p >= P) return;
  for (int idx = threadIdx.x; idx < H * F; idx += FFT_THREADS) {
    const int f = idx / F;
    const float2 zf = z[c * Np + pad(f)];
    const float2 zm = z[c * Np + pad(f == 0 ? 0 : N - f)];
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
                                                                 int N, int F, const __grid_constant__ FftPlan pl,
                                                                 const float2* __restrict__ st, OutUnscale u,
                                                                 float* __restrict__ X, int vec, FftJob job) {
  extern __shared__ float2 z[];
  __shared__ float2 ssc[2 * (FFT_POINTS / 64)];   // per-tube output scale (1/N and R18), TUB <= 256
  const int TUB = 2 * F;
  const int Np = bstride(job.M ? job.M : N, F);
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
  for (int t = threadIdx.x; t < TUB; t += IFFT_THREADS)
    ssc[t] = p0 + t < P ? out_scale(u.row, p0 + t, u.col, q, 1.f / (float)N) : make_float2(0.f, 0.f);
  __syncthreads();
  fft_core<+1, IFFT_THREADS>(z, N, F, Np, pl, st, job);
  const int64_t PQ = P * Q;
  float* xo = X + P * q + p0;
  if (vec && (TUB % 4) == 0 && p0 + TUB <= P && (P % 4) == 0 && (((uintptr_t)X) & 15) == 0) {
    const int V = TUB >> 2;
    const int total = V * N;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < total; idx += IFFT_THREADS) {
      const int vv = idx % V, k = idx / V;
      const float2 a = z[(2 * vv) * Np + pad(k)], b = z[(2 * vv + 1) * Np + pad(k)];
      reinterpret_cast<float4*>(xo + PQ * k)[vv] =
          make_float4(apply_scale(a.x, ssc[4 * vv]), apply_scale(a.y, ssc[4 * vv + 1]),
                      apply_scale(b.x, ssc[4 * vv + 2]), apply_scale(b.y, ssc[4 * vv + 3]));
    }
  } else {
    for (int idx = threadIdx.x; idx < TUB * N; idx += IFFT_THREADS) {
      const int t = idx % TUB, k = idx / TUB;
      if (p0 + t >= P) continue;
      const float2 v = z[(t >> 1) * Np + pad(k)];
      xo[PQ * k + t] = apply_scale((t & 1) == 0 ? v.x : v.y, ssc[t]);
    }
  }
}

size_t fft_smem_bytes(int N) {
  const int F = fft_F(N);
  return sizeof(float2) * (size_t)F * bstride(N, F);
}

bool fft_smem_ok(const void* kern, int N) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem_bytes(N)) ==
         cudaSuccess;
}

}  // namespace

size_t stockham_table_len(int n) {
  FftPlan pl;
  if (!make_plan(n, &pl)) return 0;
  const int last = pl.np - 1;
  if (last < 0) return 0;
  return (size_t)pl.toff[last] + (pl.Ns[last] > 1 ? (size_t)(pl.R[last] - 1) * pl.Ns[last] : 0);
}

void host_stockham_table(int n, const double* cs, float2* out) {
  FftPlan pl;
  if (!make_plan(n, &pl)) return;
  for (int i = 0; i < pl.np; ++i) {
    const int R = pl.R[i], Ns = pl.Ns[i];
    if (Ns == 1) continue;
    float2* o = out + pl.toff[i];
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < Ns; ++k) {
        const long long m = (long long)r * k * (n / (Ns * R));   // w_{Ns R}^{r k} = w_n^m, m < n
        o[(size_t)(r - 1) * Ns + k] = make_float2((float)cs[2 * m], (float)cs[2 * m + 1]);
      }
  }
}

bool fft_supported(int64_t n3) {
  FftPlan pl;
  return n3 > 64 && n3 <= FFT_POINTS && make_plan((int)n3, &pl);
}

namespace {

// Smallest 5-smooth M >= 2 n - 1 (the Bluestein convolution length), 0 if above FFT_POINTS.
int bluestein_len(int n) {
  for (int m = 2 * n - 1; m <= FFT_POINTS; ++m) {
    FftPlan pl;
    if (make_plan(m, &pl)) return m;
  }
  return 0;
}

// Host mixed-radix (2, 3, 5) DFT in fp64, recursive decimation in time; sign -1 (forward).
void host_fft(std::vector<std::complex<double>>& a) {
  const int n = (int)a.size();
  if (n == 1) return;
  const int r = n % 2 == 0 ? 2 : n % 3 == 0 ? 3 : 5;
  const int m = n / r;
  std::vector<std::vector<std::complex<double>>> sub(r, std::vector<std::complex<double>>(m));
  for (int j = 0; j < m; ++j)
    for (int q = 0; q < r; ++q) sub[q][j] = a[j * r + q];
  for (int q = 0; q < r; ++q) host_fft(sub[q]);
  for (int k = 0; k < n; ++k) {
    std::complex<double> acc = 0.0;
    for (int q = 0; q < r; ++q) {
      const double ang = -2.0 * M_PI * (double)(((long long)q * k) % n) / (double)n;
      acc += sub[q][k % m] * std::complex<double>(cos(ang), sin(ang));
    }
    a[k] = acc;
  }
}

struct BlueTab {
  int M = 0;
  const float2* chirp = nullptr;   // c_k = e^{-pi i k^2 / N}, k < N
  const float2* bh = nullptr;      // FFT_M(b) / M, b the wrapped conj chirp
  const float2* st = nullptr;      // Stockham table of M
};

// Bluestein tables of length n (device copies, cached per device); false if n has no length-M plan.
bool get_bluestein(int n, BlueTab* out) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, BlueTab> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, n});
  if (it != cache.end()) { *out = it->second; return out->M > 0; }
  BlueTab t;
  t.M = bluestein_len(n);
  if (t.M) {
    const int M = t.M;
    std::vector<float2> chirp(n), bh(M);
    std::vector<std::complex<double>> b(M, 0.0);
    for (int k = 0; k < n; ++k) {
      const long long m = ((long long)k * k) % (2LL * n);     // exact: e^{-pi i k^2/n} has period 2n in k^2
      const double ang = M_PI * (double)m / (double)n;
      chirp[k] = make_float2((float)cos(ang), (float)-sin(ang));
      b[k] = std::complex<double>(cos(ang), sin(ang));
      if (k) b[M - k] = b[k];
    }
    host_fft(b);
    for (int k = 0; k < M; ++k) bh[k] = make_float2((float)(b[k].real() / M), (float)(b[k].imag() / M));
    std::vector<double> cs(2 * (size_t)M);
    host_twiddles(M, cs.data());
    std::vector<float2> st(stockham_table_len(M) + 1);
    host_stockham_table(M, cs.data(), st.data());
    void *dc = nullptr, *db = nullptr, *ds = nullptr;
    if (cudaMalloc(&dc, sizeof(float2) * n) != cudaSuccess || cudaMalloc(&db, sizeof(float2) * M) != cudaSuccess ||
        cudaMalloc(&ds, sizeof(float2) * st.size()) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaMemcpy(dc, chirp.data(), sizeof(float2) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(db, bh.data(), sizeof(float2) * M, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, st.data(), sizeof(float2) * st.size(), cudaMemcpyHostToDevice);
    t.chirp = (const float2*)dc;
    t.bh = (const float2*)db;
    t.st = (const float2*)ds;
  }
  cache[{dev, n}] = t;
  *out = t;
  return t.M > 0;
}

// The transform job of length n: the mixed-radix FFT for 5-smooth n (st = the handle's table), else
// Bluestein through a 5-smooth length M (its own tables).  L = the buffer length of a job.
bool fft_job(int64_t n3, const float2* st_n, FftPlan* pl, const float2** st, FftJob* job, int* L) {
  if (n3 <= 64 || n3 > FFT_POINTS) return false;
  if (make_plan((int)n3, pl)) {
    if (!st_n) return false;
    *st = st_n;
    *job = FftJob{0, nullptr, nullptr};
    *L = (int)n3;
    return true;
  }
  BlueTab t;
  if (!get_bluestein((int)n3, &t) || !make_plan(t.M, pl)) return false;
  *st = t.st;
  *job = FftJob{t.M, t.chirp, t.bh};
  *L = t.M;
  return true;
}

}  // namespace

bool bluestein_supported(int64_t n3) {
  FftPlan pl;
  return n3 > 64 && n3 <= FFT_POINTS && !make_plan((int)n3, &pl) && bluestein_len((int)n3) > 0;
}

bool launch_fwd_fft(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    const float2* st_n, __half* out, int64_t ld, float* unscale, cudaStream_t s) {
  FftPlan pl;
  const float2* st = nullptr;
  FftJob job;
  int L = 0;
  if (!fft_job(n3, st_n, &pl, &st, &job, &L)) return false;
  const int N = (int)n3, F = fft_F(L);
  const int TUB = 2 * F;
  const size_t smem = fft_smem_bytes(L);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  // vectorised loads need every block full and 16-byte aligned rows
  const int vec = (TUB % 4 == 0) && (P % TUB == 0) && (((uintptr_t)X) & 15) == 0;
  const void* k = role == 0 ? (const void*)fft_fwd_split_kernel<0> : (const void*)fft_fwd_split_kernel<1>;
  if (!fft_smem_ok(k, L)) return false;
  if (role == 0)
    fft_fwd_split_kernel<0><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, F, pl, maxbits, st, out, ld,
                                                                       unscale, vec, job);
  else
    fft_fwd_split_kernel<1><<<(unsigned)blocks, FFT_THREADS, smem, s>>>(X, P, Q, N, F, pl, maxbits, st, out, ld,
                                                                       unscale, vec, job);
  return cudaGetLastError() == cudaSuccess;
}

bool launch_inv_fft(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P, int64_t Q,
                    int64_t n3, const float2* st_n, OutUnscale u, float* X, cudaStream_t s) {
  FftPlan pl;
  const float2* st = nullptr;
  FftJob job;
  int L = 0;
  if (!fft_job(n3, st_n, &pl, &st, &job, &L)) return false;
  const int N = (int)n3, F = fft_F(L);
  const int TUB = 2 * F;
  const size_t smem = fft_smem_bytes(L);
  const int64_t blocks = (P + TUB - 1) / TUB * Q;
  // paired float2 loads of C-bar need both tubes of every pair in range and 8-byte alignment
  const int vec = (P % TUB == 0) && (ld % 2 == 0) && (fstride % 2 == 0) && (((uintptr_t)Cre) & 7) == 0 &&
                  (((uintptr_t)Cim) & 7) == 0;
  if (!fft_smem_ok((const void*)fft_inv_kernel, L)) return false;
  fft_inv_kernel<<<(unsigned)blocks, IFFT_THREADS, smem, s>>>(Cre, Cim, ld, fstride, P, Q, N, F, pl, st, u, X, vec,
                                                              job);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace tprod
