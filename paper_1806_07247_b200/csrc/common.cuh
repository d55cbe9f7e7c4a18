// Device helpers shared by the kernels of libtprod.so.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace tprod {

// Exponent e of the exact power-of-two operand scale 2^e.
// |X-bar_f(p,q)| = |sum_k x_k w^{fk}| <= n3 * max|x| (Eq. (2), |w| = 1), so with
// b = n3 * max|x| < 2^E we take e = 15 - E and every scaled spectral value is < 2^15 < 65504.
// Clamped to [-100, 100] so that 2^e and 2^-e are normal fp32 numbers.
__device__ __forceinline__ int scale_exp(unsigned maxbits, int64_t n3) {
  float mx = __uint_as_float(maxbits);
  if (!(mx > 0.f)) return 0;
  double b = (double)mx * (double)n3;
  int E;
  frexp(b, &E);
  int e = 15 - E;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}

// 2^e as an fp32 for e in [-126, 127] (exact).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }

// hi/lo split of an fp32 value into two fp16 terms: v = hi + lo + r, |r| <= 2^-11 |lo| + 2^-25.
__device__ __forceinline__ void split_f16(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

}  // namespace tprod
