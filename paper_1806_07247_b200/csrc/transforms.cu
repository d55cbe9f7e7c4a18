// Mode-3 transforms of the t-product hot path (Algorithm 1 steps 1 and 3).
//
//   K0 absmax      : per-row / per-column max |x|  -> exact power-of-two operand scales
//   K1 fwd_split   : X-bar_f(p,q) = sum_k X(p,q,k) w^{fk}, w = e^{-2 pi i/n3} (Eq. (2)),
//                    f = 0..h-1 only (Hermitian half, Eq. (8)), scaled by 2^e and split
//                    into fp16 hi/lo planes = the GEMM's operand format
//   K3 inv         : C(p,q,t) = (1/n3) [Re C-bar_0 + sum_{f=1}^{h-1} w_f Re(C-bar_f e^{+2 pi i f t/n3})]
//                    with w_f = 2, except w = 1 for f = n3/2 (even n3): the conjugate fill of
//                    Alg. 1 step 2 (L177) fused into the inverse DFT (L126); slices h..n3-1 are
//                    never materialised, the DC/Nyquist imaginary parts are discarded (C2R).
//
// Layout of X: element (p,q,k) at p + P*q + P*Q*k (Matlab layout); consecutive
// threads take consecutive p, so every global access is coalesced along the contiguous dim.
#include "internal.h"
#include "common.cuh"

#include <math.h>

namespace tprod {

// ------------------------------------------------------------------------------------ twiddles
void host_twiddles(int n, double* cs) {
  // angle = 2 pi m / n.  Reduce m to the first octant exactly with integer arithmetic so that
  // the symmetric values are bit-identical and the axis values are exact.
  for (int m = 0; m < n; ++m) {
    // use 8m/n to find the octant without rounding: work with r = m (mod n) scaled by 8
    long long num = 8LL * m;           // angle / (pi/4) = 8m/n
    int oct = (int)(num / n);          // 0..7
    long long rem = num - (long long)oct * n;  // remainder in [0, n): angle within octant = rem/n * pi/4
    double a = (M_PI / 4.0) * ((double)rem / (double)n);
    double c, s;
    // base angle phi = oct*pi/4 + a
    switch (oct) {
      case 0: c = cos(a);                        s = sin(a); break;
      case 1: c = sin(M_PI / 4.0 - a);           s = cos(M_PI / 4.0 - a); break;
      case 2: c = -sin(a);                       s = cos(a); break;
      case 3: c = -cos(M_PI / 4.0 - a);          s = sin(M_PI / 4.0 - a); break;
      case 4: c = -cos(a);                       s = -sin(a); break;
      case 5: c = -sin(M_PI / 4.0 - a);          s = -cos(M_PI / 4.0 - a); break;
      case 6: c = sin(a);                        s = -cos(a); break;
      default: c = cos(M_PI / 4.0 - a);          s = -sin(M_PI / 4.0 - a); break;
    }
    cs[2 * m] = c;
    cs[2 * m + 1] = s;
  }
}

// ------------------------------------------------------------------------------------ K0
// role 0: max over (q,k) for each p  (A rows i);  role 1: max over (p,k) for each q (B cols j)
__global__ void absmax_p_kernel(const float* __restrict__ X, int64_t P, int64_t ncols,
                                unsigned* __restrict__ maxbits) {
  // blockDim = (32, 8): x -> p within a 32-chunk, y -> columns (q,k) flattened
  __shared__ float red[8][33];
  int64_t p = (int64_t)blockIdx.x * 32 + threadIdx.x;
  float m = 0.f;
  if (p < P) {
    for (int64_t c = (int64_t)blockIdx.y * 8 + threadIdx.y; c < ncols; c += (int64_t)gridDim.y * 8)
      m = fmaxf(m, fabsf(__ldg(X + p + P * c)));
  }
  red[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && p < P) {
    for (int r = 1; r < 8; ++r) m = fmaxf(m, red[r][threadIdx.x]);
    atomicMax(maxbits + p, __float_as_uint(m));
  }
}

__global__ void absmax_q_kernel(const float* __restrict__ X, int64_t P, int64_t Q, int64_t n3,
                                unsigned* __restrict__ maxbits) {
  // one warp per run (q,k): the contiguous P elements X(:, q, k)
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < Q * n3; r += nwarps) {
    int64_t q = r % Q, k = r / Q;
    const float* x = X + P * q + P * Q * k;
    float m = 0.f;
    for (int64_t p = lane; p < P; p += 32) m = fmaxf(m, fabsf(__ldg(x + p)));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) atomicMax(maxbits + q, __float_as_uint(m));
  }
}

// Fused, vectorised K0 for both operands in one launch (requires 16-byte aligned bases and
// n1 % 4 == 0, n2 % 4 == 0).  Blocks [0, nbA) reduce A's rows: a 256-float strip of p times a
// strided set of columns (q,k), float4 loads, smem reduction over the 4 column lanes, one atomic
// per p per block.  Blocks [nbA, nbA+nbB) reduce B's columns: one warp per contiguous run
// B(:, j, k) (float4 loads), one atomic per run.
__global__ void __launch_bounds__(256) absmax2_kernel(const float* __restrict__ A, int64_t n1,
                                                      int64_t colsA, int gyA, int gxA, int txv,
                                                      const float* __restrict__ B, int64_t n2,
                                                      int64_t n4, int64_t n3,
                                                      unsigned* __restrict__ maxA,
                                                      unsigned* __restrict__ maxB) {
  const int nbA = gxA * gyA;
  if ((int)blockIdx.x < nbA) {
    // A rows: a strip of 4*txv consecutive p (txv float4 lanes) x ty = 256/txv column lanes
    __shared__ float red[256 * 4 + 256];
    const int ty_n = 256 / txv, W = 4 * txv + 1;
    const int bx = blockIdx.x % gxA, by = blockIdx.x / gxA;
    const int tx = threadIdx.x % txv, ty = threadIdx.x / txv;
    const int64_t p = (int64_t)bx * 4 * txv + 4 * tx;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p < n1) {
      const float4* base = reinterpret_cast<const float4*>(A + p);
      const int64_t step = (int64_t)gyA * ty_n;
      // batches of U independent loads in flight per thread (latency-bound otherwise on narrow A)
      constexpr int U = 8;
      for (int64_t c0 = (int64_t)by * ty_n + ty; c0 < colsA; c0 += U * step) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t c = c0 + u * step;
          v[u] = c < colsA ? __ldg(base + (c * n1 >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          m.x = fmaxf(m.x, fabsf(v[u].x));
          m.y = fmaxf(m.y, fabsf(v[u].y));
          m.z = fmaxf(m.z, fabsf(v[u].z));
          m.w = fmaxf(m.w, fabsf(v[u].w));
        }
      }
    }
    red[ty * W + 4 * tx] = m.x;
    red[ty * W + 4 * tx + 1] = m.y;
    red[ty * W + 4 * tx + 2] = m.z;
    red[ty * W + 4 * tx + 3] = m.w;
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t pt = (int64_t)bx * 4 * txv + t;
    if (t < 4 * txv && pt < n1) {
      float r = 0.f;
      for (int y = 0; y < ty_n; ++y) r = fmaxf(r, red[y * W + t]);
      atomicMax(maxA + pt, __float_as_uint(r));
    }
  } else {
    // B columns: warp w owns column j = w mod n4 and the runs B(:, j, k) for k = w / n4 + i * wpc
    // (wpc warps per column), one atomic per warp
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)(blockIdx.x - nbA) * 256 + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)(gridDim.x - nbA) * 256) >> 5;
    const int64_t wpc = nwarps >= n4 ? nwarps / n4 : 1;
    for (int64_t w = warp; w < n4 * wpc; w += nwarps) {
      const int64_t j = w % n4, k0 = w / n4;
      float m = 0.f;
      const int64_t r4 = n2 >> 2;                      // float4 per run B(:, j, k)
      if (r4 >= 128) {
        for (int64_t k = k0; k < n3; k += wpc) {
          const float4* x = reinterpret_cast<const float4*>(B + n2 * (j + n4 * k));   // run (j,k)
#pragma unroll 4
          for (int64_t l4 = lane; l4 < r4; l4 += 32) {
            float4 v = __ldg(x + l4);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
          }
        }
      } else if (r4 >= 32) {
        // runs of 128..508 floats (config 2): KU runs of the column at a time, two float4 per run
        // and lane, 8 loads in flight per lane (one run at a time measured 17.4 us for config 2's
        // K0, this 13.5 us; long runs keep the loop above, which measured faster on config 3)
        constexpr int KU = 4;
        for (int64_t kb = k0; kb < n3; kb += KU * wpc) {
          for (int64_t l4 = lane; l4 < r4; l4 += 64) {
            float4 v[KU][2];
#pragma unroll
            for (int u = 0; u < KU; ++u) {
              const int64_t k = kb + u * wpc;
              const float4* x = reinterpret_cast<const float4*>(B + n2 * (j + n4 * k));   // run (j,k)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
                v[u][hh] = (k < n3 && l4 + 32 * hh < r4) ? __ldg(x + l4 + 32 * hh) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < KU; ++u)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u][hh].x), fabsf(v[u][hh].y)), fmaxf(fabsf(v[u][hh].z), fabsf(v[u][hh].w))));
          }
        }
      } else {
        // short runs: the warp splits into G = 32 / r4 lane groups, each on its own run (j, k) of
        // column j (r4 float4 lanes per run), U loads per lane in flight per batch
        constexpr int U = 8;
        const int G = 32 / (int)r4, g = lane / (int)r4, l4 = lane - g * (int)r4;
        for (int64_t kb = k0; kb < n3; kb += (int64_t)U * G * wpc) {
          float4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t k = kb + (int64_t)(u * G + g) * wpc;
            v[u] = (g < G && k < n3) ? __ldg(reinterpret_cast<const float4*>(B + n2 * (j + n4 * k)) + l4)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
        }
      }
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(maxB + j, __float_as_uint(m));
    }
  }
}

void launch_absmax2(const float* A, const float* B, int64_t n1, int64_t n2, int64_t n3, int64_t n4,
                    unsigned* maxA, unsigned* maxB, int num_sms, cudaStream_t s) {
  // A or B may be null (prepared-operand calls): that operand's part is skipped
  const bool vec = (!A || (n1 % 4 == 0 && ((uintptr_t)A & 15) == 0)) && n2 % 4 == 0 &&
                   (!B || ((uintptr_t)B & 15) == 0);
  if (!vec) {
    if (A) launch_absmax(A, n1, n2, n3, 0, maxA, s);
    if (B) launch_absmax(B, n2, n4, n3, 1, maxB, s);
    return;
  }
  // split ~8 CTAs per SM between the two tensors in proportion to their sizes
  const double szA = A ? (double)n1 * n2 * n3 : 0.0, szB = B ? (double)n2 * n4 * n3 : 0.0;
  const int64_t total = (int64_t)num_sms * 8;
  int64_t nbA_target = (int64_t)(total * szA / (szA + szB));
  // small operands: >= 64 KB per CTA (config 2's 8 MB A took 592 CTAs of 14 KB each, and their
  // 592 x n1 same-address atomicMax updates cost more than the loads: 13.5 us for 16.8 MB)
  const int64_t capA = (int64_t)(szA * 4.0 / 65536.0) + 1, capB = (int64_t)(szB * 4.0 / 65536.0) + 1;
  if (nbA_target > capA) nbA_target = capA;
  if (nbA_target < 1) nbA_target = 1;
  int txv = 1;
  while (txv < 64 && 4 * txv < n1) txv <<= 1;       // float4 lanes across p (narrow A: more column lanes)
  const int64_t gxA = (n1 + 4 * txv - 1) / (4 * txv);
  const int64_t colsA = n2 * n3;
  int64_t gyA = (nbA_target + gxA - 1) / gxA;
  const int64_t maxgy = (colsA + 256 / txv - 1) / (256 / txv);
  if (gyA > maxgy) gyA = maxgy;
  if (gyA < 1) gyA = 1;
  if (!A) gyA = 0;
  int64_t nbB = total - gxA * gyA;
  const int64_t runsB = n4 * n3;
  if (nbB > (runsB + 7) / 8) nbB = (runsB + 7) / 8;      // at most one run per warp
  if (nbB > capB) nbB = capB;
  if (nbB < 1) nbB = 1;
  if (!B) nbB = 0;
  absmax2_kernel<<<(unsigned)(gxA * gyA + nbB), 256, 0, s>>>(A, n1, colsA, (int)gyA, (int)gxA, txv, B, n2,
                                                             n4, n3, maxA, maxB);
}

void launch_absmax(const float* X, int64_t P, int64_t Q, int64_t n3, int role, unsigned* maxbits,
                   cudaStream_t s) {
  if (role == 0) {
    int64_t ncols = Q * n3;
    int64_t gx = (P + 31) / 32;
    int64_t gy = (ncols + 7) / 8;
    int64_t target = 148 * 16;  // enough CTAs to saturate HBM
    int64_t cap = (target + gx - 1) / gx;
    if (gy > cap) gy = cap;
    if (gy > 65535) gy = 65535;
    if (gy < 1) gy = 1;
    absmax_p_kernel<<<dim3((unsigned)gx, (unsigned)gy), dim3(32, 8), 0, s>>>(X, P, ncols, maxbits);
  } else {
    int64_t runs = Q * n3;
    int64_t blocks = (runs * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    absmax_q_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, P, Q, n3, maxbits);
  }
}

// Dynamic shared memory for a kernel's staged twiddle table of `bytes`: the table size when the
// kernel can be opted in to it (up to 96 KB, leaving room for co-resident CTAs), else 0 (the
// kernel then reads the table from global memory).
static size_t tw_smem_bytes(const void* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return bytes;
  if (bytes > 96 * 1024) return 0;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return bytes;
}

// ------------------------------------------------------------------------------------ K1 (fp32)
// Generic fallback (any n3; O(n3^2) per tube).  n3 <= 64 runs transforms_dense.cu instead.
// The twiddle table is staged in shared memory when it fits (tw_smem = 1), else read through L1/L2.
template <int ROLE>
__global__ void fwd_split_kernel(const float* __restrict__ X, int64_t P, int64_t Q, int n3, int h,
                                 const unsigned* __restrict__ maxbits,
                                 const float2* __restrict__ tw, int tw_smem, __half* __restrict__ out,
                                 int64_t ld, float* __restrict__ unscale) {
  extern __shared__ float2 stw_buf[];
  const float2* stw = tw;
  if (tw_smem) {
    for (int m = threadIdx.x; m < n3; m += blockDim.x) stw_buf[m] = tw[m];
    __syncthreads();
    stw = stw_buf;
  }
  int64_t pblocks = (P + blockDim.x - 1) / blockDim.x;
  int64_t q = blockIdx.x / pblocks;
  int64_t p = (blockIdx.x % pblocks) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t PQ = P * Q;
  const float* x = X + p + P * q;
  const unsigned mb = __ldg(maxbits + (ROLE == 0 ? p : q));
  const int e = scale_exp(mb, n3);
  const float sc = pow2f(e);
  if (ROLE == 0 ? q == 0 : p == 0) unscale[ROLE == 0 ? p : q] = unscale_of(mb, e);
  const int64_t plane = Q * ld;
  __half* o = out + q * ld + p;
  for (int f = 0; f < h; ++f) {
    float re = 0.f, im = 0.f;
    int m = 0;
    for (int k = 0; k < n3; ++k) {
      float v = __ldg(x + PQ * k);
      float2 w = stw[m];
      re = fmaf(v, w.x, re);
      im = fmaf(-v, w.y, im);       // w^{fk} = cos - i sin
      m += f;
      if (m >= n3) m -= n3;
    }
    __half hi, lo;
    split_f16(re * sc, hi, lo);
    o[(int64_t)(4 * f + PL_RE_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_RE_LO) * plane] = lo;
    split_f16(im * sc, hi, lo);
    o[(int64_t)(4 * f + PL_IM_HI) * plane] = hi;
    o[(int64_t)(4 * f + PL_IM_LO) * plane] = lo;
  }
}

void launch_fwd_split(const float* X, int64_t P, int64_t Q, int64_t n3, int role,
                      const unsigned* maxbits, Twiddles32 tw, __half* out, int64_t ld,
                      float* unscale, int num_sms, cudaStream_t s) {
  if (tw.staged && tw.tc && launch_fwd_dft_tc(X, P, Q, n3, role, maxbits, out, ld, unscale, num_sms, s)) return;
  cudaGetLastError();
  if (tw.staged) {
    if (launch_fwd_tma(X, P, Q, n3, role, maxbits, out, ld, unscale, num_sms, s)) return;
    cudaGetLastError();
    if (launch_fwd_tube(X, P, Q, n3, role, maxbits, tw.st, out, ld, unscale, num_sms, s)) return;
    cudaGetLastError();
  }
  if (launch_fwd_dense(X, P, Q, n3, role, maxbits, out, ld, unscale, s)) return;
  if (tw.staged && tw.cluster && launch_fwd_cluster(X, P, Q, n3, role, maxbits, tw.tw, out, ld, unscale, num_sms, s)) return;
  cudaGetLastError();
  if (tw.staged && launch_fwd_4step(X, P, Q, n3, role, maxbits, tw, out, ld, unscale, num_sms, s)) return;
  cudaGetLastError();
  // 5-smooth n3 > 64: mixed-radix FFT (the handle's Stockham table); otherwise Bluestein's chirp-z
  // through a 5-smooth length (its own tables); both return false for n3 <= 64
  if (launch_fwd_fft(X, P, Q, n3, role, maxbits, tw.st, out, ld, unscale, s)) return;
  cudaGetLastError();
  const int threads = 128;
  int64_t blocks = (P + threads - 1) / threads * Q;
  int h = (int)h_slices(n3);
  const void* k = role == 0 ? (const void*)fwd_split_kernel<0> : (const void*)fwd_split_kernel<1>;
  const size_t smem = tw_smem_bytes(k, sizeof(float2) * (size_t)n3);
  const int ts = smem > 0;
  if (role == 0)
    fwd_split_kernel<0><<<(unsigned)blocks, threads, smem, s>>>(X, P, Q, (int)n3, h, maxbits, tw.tw, ts, out, ld, unscale);
  else
    fwd_split_kernel<1><<<(unsigned)blocks, threads, smem, s>>>(X, P, Q, (int)n3, h, maxbits, tw.tw, ts, out, ld, unscale);
}

__global__ void decode_split_kernel(const __half* __restrict__ in, int64_t ld, int64_t P, int64_t Q,
                                    int h, int role, const float* __restrict__ unscale,
                                    float* __restrict__ re, float* __restrict__ im) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)h * P * Q;
  if (idx >= total) return;
  int64_t p = idx % P, q = (idx / P) % Q, f = idx / (P * Q);
  const float u = unscale[role == 0 ? p : q];
  const int64_t plane = Q * ld;
  const __half* b = in + q * ld + p;
  float r = __half2float(b[(4 * f + PL_RE_HI) * plane]) + __half2float(b[(4 * f + PL_RE_LO) * plane]);
  float i = __half2float(b[(4 * f + PL_IM_HI) * plane]) + __half2float(b[(4 * f + PL_IM_LO) * plane]);
  re[idx] = r * u;
  im[idx] = i * u;
}

void launch_decode_split(const __half* in, int64_t ld, int64_t P, int64_t Q, int64_t n3, int role,
                         const float* unscale, float* re, float* im, cudaStream_t s) {
  int64_t total = h_slices(n3) * P * Q;
  decode_split_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      in, ld, P, Q, (int)h_slices(n3), role, unscale, re, im);
}

// ------------------------------------------------------------------------------------ K3 (fp32)
template <typename T, typename T2>
__global__ void inv_kernel(const T* __restrict__ Cre, const T* __restrict__ Cim, int64_t ld,
                           int64_t fstride, int64_t P, int64_t Q, int n3, int h,
                           const T2* __restrict__ tw, int tw_smem, OutUnscale u, T* __restrict__ X) {
  extern __shared__ unsigned char smem_raw[];
  const T2* stw = tw;
  if (tw_smem) {
    T2* b = reinterpret_cast<T2*>(smem_raw);
    for (int m = threadIdx.x; m < n3; m += blockDim.x) b[m] = tw[m];
    __syncthreads();
    stw = b;
  }
  int64_t pblocks = (P + blockDim.x - 1) / blockDim.x;
  int64_t q = blockIdx.x / pblocks;
  int64_t p = (blockIdx.x % pblocks) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const T* cr = Cre + q * ld + p;
  const T* ci = Cim + q * ld + p;
  const T inv_n = T(1) / T(n3);
  const float2 sc = out_scale(u.row, p, u.col, q, 1.f);      // R18 (fp64 path: nullptr, exactly 1)
  for (int t = 0; t < n3; ++t) {
    T acc = cr[0];                      // Re C-bar_0 (Im of DC discarded)
    int m = 0;
    for (int f = 1; f < h; ++f) {
      m += t;
      if (m >= n3) m -= n3;             // m = f t mod n3
      T2 w = stw[m];
      T r = cr[(int64_t)f * fstride], i = ci[(int64_t)f * fstride];
      T v = r * w.x - i * w.y;          // Re(C-bar_f e^{+i theta})
      acc += (2 * f == n3) ? v : T(2) * v;
    }
    X[p + P * q + P * Q * (int64_t)t] = ((acc * inv_n) * (T)sc.x) * (T)sc.y;
  }
}

void launch_inv_f32(const float* Cre, const float* Cim, int64_t ld, int64_t fstride, int64_t P,
                    int64_t Q, int64_t n3, Twiddles32 tw, OutUnscale u, float* X, int num_sms, cudaStream_t s,
                    OverlapK3* ov) {
  const bool prod_layout = tw.staged && Cim == Cre + Q * ld && fstride == 2 * Q * ld;
  if (prod_layout && tw.tc && launch_inv_dft_tc(Cre, ld, P, Q, n3, u, X, num_sms, s)) return;
  cudaGetLastError();
  if (prod_layout && launch_inv_tube(Cre, ld, P, Q, n3, tw.st, u, X, num_sms, s, ov)) return;
  cudaGetLastError();
  if (prod_layout && tw.cluster && launch_inv_cluster(Cre, ld, P, Q, n3, tw.tw, u, X, num_sms, s)) return;
  cudaGetLastError();
  if (prod_layout && launch_inv_4step(Cre, ld, P, Q, n3, tw, u, X, num_sms, s)) return;
  cudaGetLastError();
  if (launch_inv_dense(Cre, Cim, ld, fstride, P, Q, n3, u, X, s, ov)) return;
  if (launch_inv_fft(Cre, Cim, ld, fstride, P, Q, n3, tw.st, u, X, s)) return;
  cudaGetLastError();
  const int threads = 128;
  int64_t blocks = (P + threads - 1) / threads * Q;
  const size_t smem = tw_smem_bytes((const void*)inv_kernel<float, float2>, sizeof(float2) * (size_t)n3);
  inv_kernel<float, float2><<<(unsigned)blocks, threads, smem, s>>>(
      Cre, Cim, ld, fstride, P, Q, (int)n3, (int)h_slices(n3), tw.tw, smem > 0, u, X);
}

// ------------------------------------------------------------------------------------ fp64 path
__global__ void fwd_f64_kernel(const double* __restrict__ X, int64_t P, int64_t Q, int n3, int h,
                               const double2* __restrict__ tw, int tw_smem, double* __restrict__ out,
                               int64_t ld) {
  extern __shared__ double2 stw64_buf[];
  const double2* stw64 = tw;
  if (tw_smem) {
    for (int m = threadIdx.x; m < n3; m += blockDim.x) stw64_buf[m] = tw[m];
    __syncthreads();
    stw64 = stw64_buf;
  }
  int64_t pblocks = (P + blockDim.x - 1) / blockDim.x;
  int64_t q = blockIdx.x / pblocks;
  int64_t p = (blockIdx.x % pblocks) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t PQ = P * Q;
  const double* x = X + p + P * q;
  const int64_t plane = Q * ld;
  double* o = out + q * ld + p;
  for (int f = 0; f < h; ++f) {
    double re = 0.0, im = 0.0;
    int m = 0;
    for (int k = 0; k < n3; ++k) {
      double v = x[PQ * k];
      double2 w = stw64[m];
      re = fma(v, w.x, re);
      im = fma(-v, w.y, im);
      m += f;
      if (m >= n3) m -= n3;
    }
    o[(int64_t)(2 * f) * plane] = re;
    o[(int64_t)(2 * f + 1) * plane] = im;
  }
}

void launch_fwd_f64(const double* X, int64_t P, int64_t Q, int64_t n3, Twiddles64 tw, double* out,
                    int64_t ld, cudaStream_t s) {
  if (launch_fwd_fft64(X, P, Q, n3, out, ld, s)) return;
  cudaGetLastError();
  const int threads = 128;
  int64_t blocks = (P + threads - 1) / threads * Q;
  const size_t smem = tw_smem_bytes((const void*)fwd_f64_kernel, sizeof(double2) * (size_t)n3);
  fwd_f64_kernel<<<(unsigned)blocks, threads, smem, s>>>(X, P, Q, (int)n3, (int)h_slices(n3), tw.tw, smem > 0, out,
                                                         ld);
}

void launch_inv_f64(const double* Cb, int64_t ld, int64_t P, int64_t Q, int64_t n3, Twiddles64 tw,
                    double* X, cudaStream_t s) {
  if (launch_inv_fft64(Cb, ld, P, Q, n3, X, s)) return;
  cudaGetLastError();
  const int threads = 128;
  int64_t blocks = (P + threads - 1) / threads * Q;
  const size_t smem = tw_smem_bytes((const void*)inv_kernel<double, double2>, sizeof(double2) * (size_t)n3);
  inv_kernel<double, double2><<<(unsigned)blocks, threads, smem, s>>>(
      Cb, Cb + Q * ld, ld, 2 * Q * ld, P, Q, (int)n3, (int)h_slices(n3), tw.tw, smem > 0, OutUnscale{}, X);
}

}  // namespace tprod
