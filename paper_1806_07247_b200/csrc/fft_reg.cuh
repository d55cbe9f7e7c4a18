// In-register FFT building blocks shared by the Stockham transform kernels (transforms_fft.cu,
// transforms_tma.cu).  Complex numbers are float2 (x = Re, y = Im); DIR = -1 forward
// (w = e^{-2 pi i/n}, Eq. (1)-(2)), +1 inverse.
#pragma once
#include <cuda_runtime.h>

namespace tprod {
namespace fftreg {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 mul_i(float2 a) { return make_float2(-a.y, a.x); }   // i * a

// w_M^i = exp(DIR * 2 pi i * i / M) for M | 16, DIR = -1 forward / +1 inverse
template <int DIR>
__device__ __forceinline__ float2 wconst(int M, int i) {
  constexpr double C16[16] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
                              0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
                              -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
                              0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};
  const int m = i * (16 / M);
  const float c = (float)C16[m & 15];
  const float s = (float)C16[(m + 12) & 15];      // sin(x) = cos(x - pi/2)
  return make_float2(c, DIR < 0 ? -s : s);
}

// In-register DFT of R points, natural order in and out.
template <int R, int DIR>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
  if constexpr (R == 3) {
    const float c = -0.5f, s = (float)(DIR * 0.86602540378443865);      // w_3 = c + i s
    const float2 t1 = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    const float2 m = make_float2(v[0].x + c * t1.x, v[0].y + c * t1.y);
    const float2 id = mul_i(cscale(d, s));
    v[0] = cadd(v[0], t1);
    v[1] = cadd(m, id);
    v[2] = csub(m, id);
  } else if constexpr (R == 5) {
    const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
    const float s1 = (float)(DIR * 0.95105651629515357), s2 = (float)(DIR * 0.58778525229247313);
    const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    const float2 m1 = make_float2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
    const float2 m2 = make_float2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
    const float2 n1 = mul_i(make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
    const float2 n2 = mul_i(make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
    v[0] = cadd(v[0], cadd(a1, a2));
    v[1] = cadd(m1, n1);
    v[4] = csub(m1, n1);
    v[2] = cadd(m2, n2);
    v[3] = csub(m2, n2);
  } else {
    // R = 2^m: radix-2 DIF, bit-reversed result reordered by renaming
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
}

// table twiddle (cos, DIR*sin)
template <int DIR>
__device__ __forceinline__ float2 twN(const float2* __restrict__ tw, int m) {
  const float2 t = __ldg(tw + m);
  return make_float2(t.x, DIR < 0 ? -t.y : t.y);
}

}  // namespace fftreg
}  // namespace tprod
