// Register-resident dense mode-3 DFT kernels for n3 <= 64 (the "small n3" path of the north star).
//
// K1 (forward, Alg. 1 step 1; Eq. (2)): one thread per tube x(0..N-1).
// For a real tube the Hermitian half X_f = sum_k x_k w^{fk}, w = e^{-2 pi i/N}, f < H = N/2+1
// (Eq. (8)), is evaluated with the conjugate-pair folding
//     u_k = x_k + x_{N-k},  v_k = x_k - x_{N-k}   (k = 1..(N-1)/2)
//     Re X_f = x_0 + sum_k u_k cos(2 pi f k/N) [+ (-1)^f x_{N/2}],   Im X_f = -sum_k v_k sin(2 pi f k/N)
// which halves the multiply-adds.  N is a template parameter, so every twiddle index (f k mod N)
// is a compile-time constant and the twiddles are read as constant-bank FFMA operands (no shared
// or global loads in the inner loop).  The output is scaled by 2^e (exact) and split into the
// fp16 hi/lo planes the tcgen05 GEMM consumes.
//
// K3 (inverse + fused conjugate fill, Alg. 1 step 2 second branch and step 3, L177-179):
//     C_t = (1/N) [R_0 + sum_{f=1}^{H-1} w_f (R_f cos(2 pi f t/N) - I_f sin(2 pi f t/N))],
//     w_f = 2 (f != N/2), 1 (f = N/2)
// with the pair folding C_t = a_t + b_t, C_{N-t} = a_t - b_t.
//
// Memory: every load/store is warp-coalesced along the contiguous dimension p (Matlab layout).
#include "internal.h"
#include "common.cuh"

#include <mutex>
#include <vector>

namespace tprod {

constexpr int DENSE_MAX = 64;
// c_tw[off(N) + m] = (cos, sin)(2 pi m / N), off(N) = N(N-1)/2
__constant__ float2 c_tw[DENSE_MAX * (DENSE_MAX + 1) / 2];

__host__ __device__ constexpr int tw_off(int N) { return N * (N - 1) / 2; }

// ---------------------------------------------------------------- register real FFT (N = 2^m >= 8)
// For power-of-two N the Hermitian half is computed in O(N log N) instead of the O(N^2/2) pair
// folding: pack z[n] = x[2n] + i x[2n+1] (n < M = N/2), Z = FFT_M(z) (radix-2 DIT
// in registers, twiddle indices compile-time), then
//   E_k = (Z_k + conj Z_{M-k})/2,  O_k = (Z_k - conj Z_{M-k})/(2i),  X_k = E_k + w^k O_k,  k = 0..M
// with w = e^{-2 pi i/N}.  The inverse reverses it: E_k = (X_k + conj X_{M-k})/2,
// O_k = w^{-k} (X_k - conj X_{M-k})/2, z = IFFT_M(E + i O), x[2n] = Re z, x[2n+1] = Im z.
__host__ __device__ constexpr bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
__host__ __device__ constexpr int bitrev(int v, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((v >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

// in-place forward DFT of a[0..M) (natural order in, natural order out), twiddles from table N
template <int N, int M>
__device__ __forceinline__ void cfft_reg(float2 (&a)[M]) {
  constexpr int LB = ilog2c(M);
  float2 b[M];
#pragma unroll
  for (int n = 0; n < M; ++n) b[bitrev(n, LB)] = a[n];
#pragma unroll
  for (int st = 0; st < LB; ++st) {
    const int len = 2 << st;
#pragma unroll
    for (int i = 0; i < M; i += len) {
#pragma unroll
      for (int j = 0; j < len / 2; ++j) {
        const float2 u = b[i + j];
        float2 v = b[i + j + len / 2];
        if (j != 0) {
          const float2 t = c_tw[tw_off(N) + j * (N / len)];     // w_len^j = (c, -s)
          v = make_float2(v.x * t.x + v.y * t.y, v.y * t.x - v.x * t.y);
        }
        b[i + j] = make_float2(u.x + v.x, u.y + v.y);
        b[i + j + len / 2] = make_float2(u.x - v.x, u.y - v.y);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < M; ++n) a[n] = b[n];
}

template <int N>
__device__ __forceinline__ void rfft_half(const float (&x)[N], float2 (&X)[N / 2 + 1]) {
  constexpr int M = N / 2;
  float2 z[M];
#pragma unroll
  for (int n = 0; n < M; ++n) z[n] = make_float2(x[2 * n], x[2 * n + 1]);
  cfft_reg<N, M>(z);
#pragma unroll
  for (int k = 0; k <= M; ++k) {
    const float2 zk = z[k % M], zm = z[(M - k) % M];
    const float2 E = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    const float2 O = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    if (k == 0 || k == M) {
      X[k] = make_float2(k == 0 ? E.x + O.x : E.x - O.x, k == 0 ? E.y + O.y : E.y - O.y);
    } else {
      const float2 t = c_tw[tw_off(N) + k];                        // w^k = (c, -s)
      X[k] = make_float2(E.x + O.x * t.x + O.y * t.y, E.y + O.y * t.x - O.x * t.y);
    }
  }
}

// C2R: X[0].y and X[N/2].y are ignored (Im of DC/Nyquist dropped); includes the 1/N scaling.
template <int N>
__device__ __forceinline__ void irfft_half(const float2 (&X)[N / 2 + 1], float (&x)[N]) {
  constexpr int M = N / 2;
  float2 z[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const float2 xk = (k == 0) ? make_float2(X[0].x, 0.f) : X[k];
    const float2 xm = (k == 0) ? make_float2(X[M].x, 0.f) : X[M - k];
    const float2 E = make_float2(0.5f * (xk.x + xm.x), 0.5f * (xk.y - xm.y));
    const float2 D = make_float2(0.5f * (xk.x - xm.x), 0.5f * (xk.y + xm.y));   // (X_k - conj X_{M-k})/2
    float2 O;
    if (k == 0) {
      O = D;
    } else {
      const float2 t = c_tw[tw_off(N) + k];                        // w^{-k} = (c, +s)
      O = make_float2(D.x * t.x - D.y * t.y, D.x * t.y + D.y * t.x);
    }
    // conj(E + i O) for the forward-FFT-based inverse
    z[k] = make_float2(E.x - O.y, -(E.y + O.x));
  }
  cfft_reg<N, M>(z);
  const float inv_m = 1.f / (float)M;
#pragma unroll
  for (int n = 0; n < M; ++n) {          // z = conj(FFT(conj Z)) / M
    x[2 * n] = z[n].x * inv_m;
    x[2 * n + 1] = -z[n].y * inv_m;
  }
}

template <int N, int ROLE>
__global__ void __launch_bounds__(128) fwd_dense_kernel(const float* __restrict__ X, int64_t P, int64_t Q,
                                                        const unsigned* __restrict__ maxbits,
                                                        __half* __restrict__ out, int64_t ld,
                                                        float* __restrict__ unscale) {
  constexpr int H = N / 2 + 1;
  constexpr int K2 = (N - 1) / 2;
  const int64_t pblocks = (P + 127) >> 7;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p = (blockIdx.x - q * pblocks) * 128 + threadIdx.x;
  if (p >= P) return;
  const int64_t PQ = P * Q;
  const float* x = X + p + P * q;
  float v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = __ldg(x + PQ * k);
  float2 Xf[H];
  if constexpr (is_pow2(N) && N >= 8) {
    rfft_half<N>(v, Xf);
  } else {
    float u[K2 + 1], w[K2 + 1];
#pragma unroll
    for (int k = 1; k <= K2; ++k) {
      u[k] = v[k] + v[N - k];
      w[k] = v[k] - v[N - k];
    }
#pragma unroll
    for (int f = 0; f < H; ++f) {
      float re = v[0], im = 0.f;
#pragma unroll
      for (int k = 1; k <= K2; ++k) {
        const float2 t = c_tw[tw_off(N) + (f * k) % N];
        re = fmaf(u[k], t.x, re);
        im = fmaf(-w[k], t.y, im);
      }
      if (N % 2 == 0) re += (f & 1) ? -v[N / 2] : v[N / 2];
      Xf[f] = make_float2(re, im);
    }
  }
  const unsigned mb = __ldg(maxbits + (ROLE == 0 ? p : q));
  const int e = scale_exp(mb, N);
  const float sc = pow2f(e);
  if (ROLE == 0 ? q == 0 : p == 0) unscale[ROLE == 0 ? p : q] = unscale_of(mb, e);
  const int64_t plane = Q * ld;
  __half* o = out + q * ld + p;
#pragma unroll
  for (int f = 0; f < H; ++f) {
    __half hi, lo;
    split_f16(Xf[f].x * sc, hi, lo);
    o[(int64_t)(4 * f + PL_RE_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_RE_LO) * plane] = lo;
    split_f16(Xf[f].y * sc, hi, lo);
    o[(int64_t)(4 * f + PL_IM_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_IM_LO) * plane] = lo;
  }
}

template <int N>
__global__ void __launch_bounds__(128) inv_dense_kernel(const float* __restrict__ Cre,
                                                        const float* __restrict__ Cim, int64_t ld,
                                                        int64_t fstride, int64_t P, int64_t Q,
                                                        OutUnscale u, float* __restrict__ X) {
  constexpr int H = N / 2 + 1;
  const int64_t pblocks = (P + 127) >> 7;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p = (blockIdx.x - q * pblocks) * 128 + threadIdx.x;
  if (p >= P) return;
  const float* cr = Cre + q * ld + p;
  const float* ci = Cim + q * ld + p;
  const int64_t PQ = P * Q;
  float* xo = X + p + P * q;
  if constexpr (is_pow2(N) && N >= 8) {
    const float2 sc = out_scale(u.row, p, u.col, q, 1.f);      // R18 (irfft_half applies 1/N)
    float2 Xf[H];
#pragma unroll
    for (int f = 0; f < H; ++f) {
      const bool self = (f == 0 || 2 * f == N);
      Xf[f] = make_float2(__ldg(cr + fstride * f), self ? 0.f : __ldg(ci + fstride * f));
    }
    float xt[N];
    irfft_half<N>(Xf, xt);
#pragma unroll
    for (int t = 0; t < N; ++t) xo[PQ * t] = apply_scale(xt[t], sc);
    return;
  }
  float R[H], I[H];
#pragma unroll
  for (int f = 0; f < H; ++f) {
    const float wf = (f == 0 || 2 * f == N) ? 1.f : 2.f;     // conjugate fill weight
    R[f] = wf * __ldg(cr + fstride * f);
    I[f] = (f == 0 || 2 * f == N) ? 0.f : wf * __ldg(ci + fstride * f);  // Im of DC/Nyquist dropped
  }
  const float2 sc = out_scale(u.row, p, u.col, q, 1.f / (float)N);   // 1/N and R18 unscale
#pragma unroll
  for (int t = 0; t <= N / 2; ++t) {
    float a = R[0], b = 0.f;
#pragma unroll
    for (int f = 1; f < H; ++f) {
      const float2 tw = c_tw[tw_off(N) + (f * t) % N];
      a = fmaf(R[f], tw.x, a);
      b = fmaf(-I[f], tw.y, b);
    }
    xo[PQ * t] = apply_scale(a + b, sc);
    if (t > 0 && 2 * t != N) xo[PQ * (N - t)] = apply_scale(a - b, sc);
  }
}

// Two adjacent tubes (p, p+1) per thread for N <= PAIR_MAX: float2 loads, half2 stores and paired
// fp16 conversions halve the per-tube instruction count of the memory-bound transforms.
// Requires P even (then every column start and every plane row stays 8-/4-byte aligned).
constexpr int PAIR_MAX = 32;

// ROLE 2 = B with its column scale computed here (K0 of B fused into K1 of B): the CTAs of one
// lateral slice q (its P / 256 blocks of 256 tubes) form one thread-block cluster; each CTA reduces
// max |B(:, q, :)| over its tubes, writes it into every peer's shared memory (DSMEM) and arrives on
// the cluster barrier, runs its DFTs, then waits and takes the max of the cluster's partial maxima --
// the exact K0 value (fmaxf of the same elements), so results are bitwise those of K0 + ROLE 1.
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <int N, int ROLE>
__global__ void __launch_bounds__(128) fwd_dense2_kernel(const float* __restrict__ X, int64_t P,
                                                         int64_t Q, const unsigned* __restrict__ maxbits,
                                                         __half* __restrict__ out, int64_t ld,
                                                         float* __restrict__ unscale) {
  constexpr int H = N / 2 + 1;
  constexpr int K2 = (N - 1) / 2;
  const int64_t pblocks = (P + 255) >> 8;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p = ((blockIdx.x - q * pblocks) * 128 + threadIdx.x) * 2;
  if (ROLE != 2 && p >= P) return;
  const bool act = p < P;                           // ROLE 2: every thread reaches the cluster barrier
  const int64_t PQh = (P * Q) >> 1;
  const float2* x = reinterpret_cast<const float2*>(X + (act ? p : 0) + P * q);
  float2 v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = act ? __ldg(x + PQh * k) : make_float2(0.f, 0.f);
  __shared__ float cmax[8];                         // ROLE 2: partial maxima of the cluster's CTAs
  uint32_t ncl = 1;
  if constexpr (ROLE == 2) {
    __shared__ float wmax[4];
    float m = 0.f;
#pragma unroll
    for (int k = 0; k < N; ++k) m = fmaxf(m, fmaxf(fabsf(v[k].x), fabsf(v[k].y)));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    __syncthreads();
    if (threadIdx.x == 0) {
      m = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]));
      uint32_t me;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(me));
      const uint32_t local = (uint32_t)__cvta_generic_to_shared(cmax + me);
      for (uint32_t r = 0; r < ncl; ++r) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(m) : "memory");
      }
    }
    cl_arrive();
  }
  float2 X0[H], X1[H];              // spectra of tube p (X0) and p+1 (X1)
  if constexpr (is_pow2(N) && N >= 8) {
    float t0[N], t1[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      t0[k] = v[k].x;
      t1[k] = v[k].y;
    }
    rfft_half<N>(t0, X0);
    rfft_half<N>(t1, X1);
  } else {
    float2 u[K2 + 1], w[K2 + 1];
#pragma unroll
    for (int k = 1; k <= K2; ++k) {
      u[k] = make_float2(v[k].x + v[N - k].x, v[k].y + v[N - k].y);
      w[k] = make_float2(v[k].x - v[N - k].x, v[k].y - v[N - k].y);
    }
#pragma unroll
    for (int f = 0; f < H; ++f) {
      float2 re = v[0], im = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 1; k <= K2; ++k) {
        const float2 t = c_tw[tw_off(N) + (f * k) % N];
        re.x = fmaf(u[k].x, t.x, re.x);
        re.y = fmaf(u[k].y, t.x, re.y);
        im.x = fmaf(-w[k].x, t.y, im.x);
        im.y = fmaf(-w[k].y, t.y, im.y);
      }
      if (N % 2 == 0) {
        const float sg = (f & 1) ? -1.f : 1.f;
        re.x = fmaf(sg, v[N / 2].x, re.x);
        re.y = fmaf(sg, v[N / 2].y, re.y);
      }
      X0[f] = make_float2(re.x, im.x);
      X1[f] = make_float2(re.y, im.y);
    }
  }
  int e0, e1;
  if (ROLE == 0) {
    const unsigned m0 = __ldg(maxbits + p), m1 = __ldg(maxbits + p + 1);
    e0 = scale_exp(m0, N);
    e1 = scale_exp(m1, N);
    if (q == 0) {
      unscale[p] = unscale_of(m0, e0);
      unscale[p + 1] = unscale_of(m1, e1);
    }
  } else {
    unsigned mq;
    if constexpr (ROLE == 2) {
      cl_wait();                                    // every CTA of the slice has written its maximum
      float m = cmax[0];
      for (uint32_t r = 1; r < ncl; ++r) m = fmaxf(m, cmax[r]);
      mq = __float_as_uint(m);
      if (!act) return;                             // no peer touches this CTA's shared memory now
    } else {
      mq = __ldg(maxbits + q);
    }
    e0 = e1 = scale_exp(mq, N);
    if (p == 0) unscale[q] = unscale_of(mq, e0);
  }
  const float s0 = pow2f(e0), s1 = pow2f(e1);
  const int64_t plane = Q * ld;
  __half* o = out + q * ld + p;
#pragma unroll
  for (int f = 0; f < H; ++f) {
    const float2 rs = make_float2(X0[f].x * s0, X1[f].x * s1), is = make_float2(X0[f].y * s0, X1[f].y * s1);
    const __half2 rh = __float22half2_rn(rs), ih = __float22half2_rn(is);
    const float2 rhf = __half22float2(rh), ihf = __half22float2(ih);
    const __half2 rl = __float22half2_rn(make_float2(rs.x - rhf.x, rs.y - rhf.y));
    const __half2 il = __float22half2_rn(make_float2(is.x - ihf.x, is.y - ihf.y));
    *reinterpret_cast<__half2*>(o + (int64_t)(4 * f + PL_RE_HI) * plane) = rh;
    *reinterpret_cast<__half2*>(o + (int64_t)(4 * f + PL_RE_LO) * plane) = rl;
    *reinterpret_cast<__half2*>(o + (int64_t)(4 * f + PL_IM_HI) * plane) = ih;
    *reinterpret_cast<__half2*>(o + (int64_t)(4 * f + PL_IM_LO) * plane) = il;
  }
}

// OverlapK3 (ov.done != nullptr): launched as a programmatic dependent of the GEMM; block b takes
// the (m, n) GEMM tile r = b / (128 pb_per_m) -- blocks ordered as the GEMM finishes its tiles --
// and waits until done[r] reaches the tile's count (ld.acquire.gpu by one
// thread, then a CTA barrier) before it reads C-bar through L2 (ld.global.cg: never a line an
// L1 might hold from before the GEMM wrote it).
struct OvArgs {
  const int* done;
  int target, pb_per_m, cols_per_n, nt;
};

template <int N>
__global__ void __launch_bounds__(128) inv_dense2_kernel(const float* __restrict__ Cre,
                                                         const float* __restrict__ Cim, int64_t ld,
                                                         int64_t fstride, int64_t P, int64_t Q,
                                                         OutUnscale u, float* __restrict__ X, OvArgs ov) {
  constexpr int H = N / 2 + 1;
  const int64_t pblocks = (P + 255) >> 8;
  int64_t q, pb;
  if (ov.done) {
    const int per = 128 * ov.pb_per_m;               // K3 blocks per (m, n) tile (cols_per_n = 128)
    const int r = (int)(blockIdx.x / per), j = (int)(blockIdx.x % per);
    q = (int64_t)(r % ov.nt) * ov.cols_per_n + (j % ov.cols_per_n);
    pb = (int64_t)(r / ov.nt) * ov.pb_per_m + j / ov.cols_per_n;
    if (q >= Q || pb >= pblocks) return;             // whole block: ragged edge of the tile grid
    if (threadIdx.x == 0) {
      const int* c = ov.done + r;
      int v;
      uint64_t t0, t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= ov.target) break;
        __nanosleep(500);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 4000000000ull) __trap();       // 4 s: a counter that never completes is a bug, not a wait
      }
    }
    __syncthreads();
  } else {
    q = blockIdx.x / pblocks;
    pb = blockIdx.x - q * pblocks;
  }
  const int64_t p = (pb * 128 + threadIdx.x) * 2;
  if (p >= P) return;
  const float2* cr = reinterpret_cast<const float2*>(Cre + q * ld + p);
  const float2* ci = reinterpret_cast<const float2*>(Cim + q * ld + p);
  const int64_t fs = fstride >> 1;
  const int64_t PQh = (P * Q) >> 1;
  float2* xo = reinterpret_cast<float2*>(X + p + P * q);
  if constexpr (is_pow2(N) && N >= 8) {
    const float2 s0 = out_scale(u.row, p, u.col, q, 1.f), s1 = out_scale(u.row, p + 1, u.col, q, 1.f);
    float2 X0[H], X1[H];
#pragma unroll
    for (int f = 0; f < H; ++f) {
      const bool self = (f == 0 || 2 * f == N);
      const float2 r = __ldcg(cr + fs * f);
      const float2 i = self ? make_float2(0.f, 0.f) : __ldcg(ci + fs * f);
      X0[f] = make_float2(r.x, i.x);
      X1[f] = make_float2(r.y, i.y);
    }
    float x0[N], x1[N];
    irfft_half<N>(X0, x0);
    irfft_half<N>(X1, x1);
#pragma unroll
    for (int t = 0; t < N; ++t) xo[PQh * t] = make_float2(apply_scale(x0[t], s0), apply_scale(x1[t], s1));
    return;
  }
  float2 R[H], I[H];
#pragma unroll
  for (int f = 0; f < H; ++f) {
    const bool self = (f == 0 || 2 * f == N);
    const float wf = self ? 1.f : 2.f;     // conjugate fill weight
    const float2 r = __ldcg(cr + fs * f);
    R[f] = make_float2(wf * r.x, wf * r.y);
    if (self) {
      I[f] = make_float2(0.f, 0.f);         // Im of DC/Nyquist dropped (C2R)
    } else {
      const float2 i = __ldcg(ci + fs * f);
      I[f] = make_float2(wf * i.x, wf * i.y);
    }
  }
  const float inv_n = 1.f / (float)N;
  const float2 s0 = out_scale(u.row, p, u.col, q, inv_n), s1 = out_scale(u.row, p + 1, u.col, q, inv_n);
#pragma unroll
  for (int t = 0; t <= N / 2; ++t) {
    float2 a = R[0], b = make_float2(0.f, 0.f);
#pragma unroll
    for (int f = 1; f < H; ++f) {
      const float2 tw = c_tw[tw_off(N) + (f * t) % N];
      a.x = fmaf(R[f].x, tw.x, a.x);
      a.y = fmaf(R[f].y, tw.x, a.y);
      b.x = fmaf(-I[f].x, tw.y, b.x);
      b.y = fmaf(-I[f].y, tw.y, b.y);
    }
    xo[PQh * t] = make_float2(apply_scale(a.x + b.x, s0), apply_scale(a.y + b.y, s1));
    if (t > 0 && 2 * t != N)
      xo[PQh * (N - t)] = make_float2(apply_scale(a.x - b.x, s0), apply_scale(a.y - b.y, s1));
  }
}

// ------------------------------------------------------------------------------ dispatch tables
using FwdFn = void (*)(const float*, int64_t, int64_t, const unsigned*, __half*, int64_t, float*);
using InvFn = void (*)(const float*, const float*, int64_t, int64_t, int64_t, int64_t, OutUnscale, float*);
using InvPFn = void (*)(const float*, const float*, int64_t, int64_t, int64_t, int64_t, OutUnscale, float*, OvArgs);

template <int N>
struct DenseTable {
  static void fill(FwdFn* f0, FwdFn* f1, InvFn* inv) {
    f0[N] = fwd_dense_kernel<N, 0>;
    f1[N] = fwd_dense_kernel<N, 1>;
    inv[N] = inv_dense_kernel<N>;
    DenseTable<N - 1>::fill(f0, f1, inv);
  }
};
template <>
struct DenseTable<0> {
  static void fill(FwdFn*, FwdFn*, InvFn*) {}
};

template <int N>
struct PairTable {
  static void fill(FwdFn* f0, FwdFn* f1, FwdFn* f2, InvPFn* inv) {
    f0[N] = fwd_dense2_kernel<N, 0>;
    f1[N] = fwd_dense2_kernel<N, 1>;
    f2[N] = fwd_dense2_kernel<N, 2>;
    inv[N] = inv_dense2_kernel<N>;
    PairTable<N - 1>::fill(f0, f1, f2, inv);
  }
};
template <>
struct PairTable<0> {
  static void fill(FwdFn*, FwdFn*, FwdFn*, InvPFn*) {}
};

struct DenseFns {
  FwdFn fwd0[DENSE_MAX + 1] = {};
  FwdFn fwd1[DENSE_MAX + 1] = {};
  InvFn inv[DENSE_MAX + 1] = {};
  FwdFn fwd0p[PAIR_MAX + 1] = {};
  FwdFn fwd1p[PAIR_MAX + 1] = {};
  FwdFn fwd2p[PAIR_MAX + 1] = {};
  InvPFn invp[PAIR_MAX + 1] = {};
  DenseFns() {
    DenseTable<DENSE_MAX>::fill(fwd0, fwd1, inv);
    PairTable<PAIR_MAX>::fill(fwd0p, fwd1p, fwd2p, invp);
  }
};

static const DenseFns& dense_fns() {
  static DenseFns t;
  return t;
}

static bool ensure_dense_twiddles() {
  static std::mutex mu;
  static uint64_t done_mask = 0;  // per device ordinal (< 64)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && (done_mask >> dev) & 1) return true;
  std::vector<float2> tab(DENSE_MAX * (DENSE_MAX + 1) / 2);
  std::vector<double> cs;
  for (int N = 1; N <= DENSE_MAX; ++N) {
    cs.assign(2 * N, 0.0);
    host_twiddles(N, cs.data());
    for (int m = 0; m < N; ++m) tab[tw_off(N) + m] = make_float2((float)cs[2 * m], (float)cs[2 * m + 1]);
  }
  if (cudaMemcpyToSymbol(c_tw, tab.data(), sizeof(float2) * tab.size()) != cudaSuccess) return false;
  if (dev < 64) done_mask |= 1ull << dev;
  return true;
}

bool dense_supported(int64_t n3) { return n3 >= 1 && n3 <= DENSE_MAX; }

bool launch_fwd_dense(const float* X, int64_t P, int64_t Q, int64_t n3, int role,
                      const unsigned* maxbits, __half* out, int64_t ld, float* unscale,
                      cudaStream_t s) {
  if (!dense_supported(n3) || !ensure_dense_twiddles()) return false;
  const DenseFns& t = dense_fns();
  const bool pair = n3 <= PAIR_MAX && P % 2 == 0 && ((uintptr_t)X & 7) == 0;
  FwdFn fn = pair ? (role == 0 ? t.fwd0p[n3] : t.fwd1p[n3]) : (role == 0 ? t.fwd0[n3] : t.fwd1[n3]);
  int64_t blocks = (P + (pair ? 255 : 127)) / (pair ? 256 : 128) * Q;
  void* args[] = {(void*)&X, (void*)&P, (void*)&Q, (void*)&maxbits, (void*)&out, (void*)&ld, (void*)&unscale};
  return cudaLaunchKernel((const void*)fn, dim3((unsigned)blocks), dim3(128), args, 0, s) == cudaSuccess;
}

bool fwd_colmax_ok(const float* X, int64_t P, int64_t n3) {
  return n3 >= 1 && n3 <= PAIR_MAX && P % 2 == 0 && P <= 8 * 256 && ((uintptr_t)X & 7) == 0;
}

bool launch_fwd_dense_colmax(const float* X, int64_t P, int64_t Q, int64_t n3, __half* out, int64_t ld,
                             float* unscale, cudaStream_t s) {
  if (!fwd_colmax_ok(X, P, n3) || !ensure_dense_twiddles()) return false;
  const int64_t pblocks = (P + 255) / 256;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pblocks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(pblocks * Q));
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  const unsigned* none = nullptr;
  return cudaLaunchKernelEx(&cfg, dense_fns().fwd2p[n3], X, P, Q, none, out, ld, unscale) == cudaSuccess;
}

bool inv_dense_pair_ok(int64_t n3) { return n3 >= 1 && n3 <= PAIR_MAX; }

bool launch_inv_dense(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P,
                      int64_t Q, int64_t n3, OutUnscale u, float* X, cudaStream_t s, OverlapK3* ov) {
  if (!dense_supported(n3) || !ensure_dense_twiddles()) return false;
  const bool pair = n3 <= PAIR_MAX && P % 2 == 0 && ld % 2 == 0 && fstride % 2 == 0 &&
                    ((uintptr_t)X & 7) == 0 && ((uintptr_t)Cre & 7) == 0 && ((uintptr_t)Cim & 7) == 0;
  int64_t blocks = (P + (pair ? 255 : 127)) / (pair ? 256 : 128) * Q;
  if (!pair) {
    InvFn fn = dense_fns().inv[n3];
    void* args[] = {(void*)&Cre, (void*)&Cim, (void*)&ld, (void*)&fstride, (void*)&P, (void*)&Q, (void*)&u, (void*)&X};
    return cudaLaunchKernel((const void*)fn, dim3((unsigned)blocks), dim3(128), args, 0, s) == cudaSuccess;
  }
  OvArgs oa = {nullptr, 0, 1, 128, 1};
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  if (ov && ov->done && ov->cols_per_n == 128) {
    // programmatic dependent of the GEMM just launched on `s`: blocks start as its CTAs free SMs
    oa = {ov->done, ov->target, ov->pb_per_m, ov->cols_per_n, ov->nt};
    const int64_t mt = ((P + 255) / 256 + ov->pb_per_m - 1) / ov->pb_per_m;
    blocks = mt * ov->nt * 128 * (int64_t)ov->pb_per_m;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ov->used = true;
  }
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  return cudaLaunchKernelEx(&cfg, dense_fns().invp[n3], Cre, Cim, ld, fstride, P, Q, u, X, oa) == cudaSuccess;
}

}  // namespace tprod
