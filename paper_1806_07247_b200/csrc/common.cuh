// Device helpers shared by the kernels of libtprod.so.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace tprod {

// Exponent e of the exact power-of-two operand scale 2^e.
// |X-bar_f(p,q)| = |sum_k x_k w^{fk}| <= n3 * max|x| (Eq. (2), |w| = 1), so with
// b = n3 * max|x| < 2^E we take e = 15 - E and every scaled spectral value is < 2^15 < 65504.
// Clamped to [-126, 126] so that 2^e and 2^-e are normal fp32 numbers: full accuracy for every
// row / column with n3 * max|x| >= 2^-111 (smaller ones land in fp16 subnormals) and no fp16
// overflow while n3 * max|x| < 2^141.
__device__ __forceinline__ int scale_exp(unsigned maxbits, int64_t n3) {
  float mx = __uint_as_float(maxbits);
  if (!(mx > 0.f)) return 0;
  double b = (double)mx * (double)n3;
  int E;
  frexp(b, &E);
  int e = 15 - E;
  return e < -126 ? -126 : (e > 126 ? 126 : e);
}

// 2^e as an fp32 for e in [-126, 127] (exact).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }

// 2^e for any e: exact for e in [-149, 127] (subnormal below -126), 0 below, +inf above.
__device__ __forceinline__ float pow2f_ext(int e) {
  if (e > 127) return __int_as_float(0x7f800000);
  if (e >= -126) return pow2f(e);
  if (e < -149) return 0.f;
  return __int_as_float(1 << (e + 149));
}

// Unscale factor K1 writes for an index whose max |x| is `maxbits`: 2^-e, or exactly 0 for an
// all-zero row / column (its part of C is exactly zero, so the factor that restores it is 0).
__device__ __forceinline__ float unscale_of(unsigned maxbits, int e) {
  return maxbits == 0u ? 0.f : pow2f(-e);
}

// Output scale of the inverse transform (R18).  C-bar leaves the GEMM at the operands'
// exact power-of-two scales, so the two real tubes that share one complex inverse FFT are of
// comparable magnitude; each output tube (p, q) is then brought back to its own scale:
//   out = (x * s.x) * s.y = x * c * urow[p] * ucol[q]
// with c the transform's own factor (e.g. 1/n3).  urow / ucol hold 2^-e or 0 (nullptr = 1).  The
// exponent sum is split in two multipliers so that neither leaves the fp32 range and the
// intermediate lies between x and the result (no spurious overflow / underflow).
__device__ __forceinline__ float2 out_scale(const float* urow, int64_t p, const float* ucol, int64_t q, float c,
                                            int extra_exp = 0) {
  int F = extra_exp;                   // an additional exact 2^extra_exp (the tensor-core inverse's own scale)
  if (urow) {
    const float u = __ldg(urow + p);
    if (u == 0.f) return make_float2(0.f, 0.f);
    F += ((__float_as_int(u) >> 23) & 0xff) - 127;
  }
  if (ucol) {
    const float u = __ldg(ucol + q);
    if (u == 0.f) return make_float2(0.f, 0.f);
    F += ((__float_as_int(u) >> 23) & 0xff) - 127;
  }
  const int F1 = F < -100 ? -100 : (F > 100 ? 100 : F);
  return make_float2(c * pow2f(F1), pow2f_ext(F - F1));
}
// out_scale from already-loaded factors ua = urow[p], ub = ucol[q] (1 where there is none).
__device__ __forceinline__ float2 out_scale_of(float ua, float ub, float c, int extra_exp = 0) {
  if (ua == 0.f || ub == 0.f) return make_float2(0.f, 0.f);
  const int F = extra_exp + ((__float_as_int(ua) >> 23) & 0xff) - 127 + ((__float_as_int(ub) >> 23) & 0xff) - 127;
  const int F1 = F < -100 ? -100 : (F > 100 ? 100 : F);
  return make_float2(c * pow2f(F1), pow2f_ext(F - F1));
}
__device__ __forceinline__ float apply_scale(float x, float2 s) { return (x * s.x) * s.y; }

// hi/lo split of an fp32 value into two fp16 terms: v = hi + lo + r, |r| <= 2^-11 |lo| + 2^-25.
__device__ __forceinline__ void split_f16(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

}  // namespace tprod
