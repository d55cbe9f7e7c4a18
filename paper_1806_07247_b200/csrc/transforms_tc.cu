// K1 / K3 for n3 <= 64 as dense DFT-matrix contractions on the tcgen05 tensor cores (the north
// star's "small n3 (<= 64) is done as a dense DFT-matrix contraction").
//
// Eq. (2) is a matrix product: the Hermitian half of the DFT of a block of 128
// real tubes x_m (m = tube, k = 0..N-1) is
//   Y = X W,   X: 128 x N,   W: N x 2H with columns  W[k, 2f] = cos(2 pi f k / N),
//                                                     W[k, 2f+1] = -sin(2 pi f k / N)   (f < H)
// so Re X_f = Y[:, 2f], Im X_f = Y[:, 2f+1] (Alg. 1 step 1; only f < H = N/2 + 1 by
// Eq. (8)).  The inverse with the fused conjugate fill (Alg. 1 step 2 second branch +
// step 3, L177-179) is the same kind of product with K = 2H rows of C-bar (re, im interleaved):
//   x_t = (2/N) sum_f (w_f/2) (Re C_f cos(2 pi f t/N) - Im C_f sin(2 pi f t/N)),  w_f = 1 (f = 0, N/2)
// or 2, the imaginary parts of the DC / Nyquist slices dropped (C2R).
//
// Precision (3xTF32): the tensor core reads 32-bit operands as tf32 (10-bit mantissa).  Each fp32
// operand is split exactly into hi = x with the low 13 mantissa bits cleared and lo = x - hi, and
// Y = Xlo Whi + Xhi Wlo + Xhi Whi (Xlo Wlo is below fp32 rounding; the two small terms are
// accumulated first so the rounding of the tensor-core accumulation is relative to the small
// partial sums), fp32 accumulation in TMEM.  No operand scaling is needed (tf32 has fp32's
// exponent range); K1's epilogue applies the exact power-of-two operand scale of the main GEMM and
// splits into its fp16 hi/lo planes, K3's the 2/N and the per-tube unscale of DESIGN.md R18.
//
// The operand X is the TMA-loaded tile itself: four boxes of 32 tubes x rows, loaded with TMA's
// 128-byte swizzle of 32-byte atoms (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: the 32-byte chunk index
// of row k XORed with k mod 4), are exactly the MN-major tf32 operand layout tcgen05 accepts
// (descriptor layout type SWIZZLE_128B_BASE32B: M atoms of 32 elements LBO apart, 4-row K groups
// SBO = 512 B apart -- the only MN-major layout for tf32; the plain 128B swizzle reads as zeros,
// measured), so the only SIMT pass over the input is the in-place hi / lo split.
//
// Warp-specialised persistent CTA (one per SM, 18 warps), work item = 128 consecutive tubes of one q:
//   warp 0       TMA producer: X tiles into an S-slot ring (S = 2..6, the deepest that fits)
//   warp 1       MMA issuer: 3 (K/8) tcgen05.mma.kind::tf32 (M = 128) into a double-buffered TMEM
//                accumulator; the commits free the ring slot and fill the accumulator
//   warps 2-9    split: X -> (hi in place, lo)
//   warps 10-17  epilogue: TMEM -> registers (lane = tube, half the columns per warp) -> scale /
//                split -> warp-coalesced global stores (K1: the 4 fp16 planes of the GEMM operand
//                format; K3: the fp32 output rows X(p0:p0+128, q, 0:N))
// The W tables (hi and lo planes, already in the swizzled shared-memory image) are copied into
// shared memory once per CTA.
#include "internal.h"
#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.h"

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace tprod {

namespace {

using namespace ptx;

constexpr int TM = 128;            // tubes per work item = MMA M
constexpr int NTHR = 576;          // 18 warps: producer, MMA, 8 split, 8 epilogue
constexpr uint32_t TF32_MASK = 0xFFFFE000u;

__host__ __device__ constexpr int rup(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// explicit shared-memory accesses by 32-bit shared address (the aligned dynamic-smem pointer is
// derived through integer arithmetic, so plain C++ accesses compile to generic LD/ST)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ float4 tf32_hi(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & TF32_MASK), __uint_as_float(__float_as_uint(v.y) & TF32_MASK),
                     __uint_as_float(__float_as_uint(v.z) & TF32_MASK), __uint_as_float(__float_as_uint(v.w) & TF32_MASK));
}

// Shared-memory regions (byte offsets, 1024-aligned): W image, then the ring of S slots, each an X
// tile (4 M-atoms x nk rows x 128 B) followed by its lo tile.  S (2..SMAX) is the deepest ring
// that fits: S - 1 TMA loads stay in flight while one item is split / multiplied, which is what
// keeps HBM busy (one 16 KB tile in flight per SM was measured to cap the kernel near 3 TB/s).
constexpr int SMAX = 6;
__host__ __device__ inline uint32_t al1k(uint32_t x) { return (x + 1023u) & ~1023u; }
__host__ __device__ inline uint32_t slot_bytes_of(int nk) { return (uint32_t)(4 * nk * 128); }
__host__ __device__ inline uint32_t ring_off(uint32_t w_bytes) { return al1k(w_bytes); }
constexpr uint32_t SMEM_BUDGET = 225 * 1024;        // dynamic shared memory per CTA (+1 KB alignment)
inline int ring_slots(int nk, uint32_t w_bytes) {
  const int s = (int)((SMEM_BUDGET - ring_off(w_bytes)) / (2 * slot_bytes_of(nk)));
  return s < SMAX ? s : SMAX;
}
constexpr int SPLIT0 = 2, NSPLIT = 8;       // split warps 2..9
constexpr int EPI0 = 10, NEPI = 8;          // epilogue warps 10..17: lane group warp & 3, column half (warp-10)/4

struct Bars {
  uint64_t x_full[SMAX], x_empty[SMAX], lo_full[SMAX], acc_full[2], acc_empty[2];
};

// Common skeleton of K1 and K3: setup and the producer / MMA / split / epilogue roles.  The
// epilogue's arithmetic and its (warp-coalesced, direct) global stores are the caller's
// `epi(q, p0, m, half, acc, v)` (m = tube = TMEM lane, acc = its NO/2 accumulator columns
// half * NO/2 ...), where v = `pre(q, p0, m)` holds the item's per-tube scale data, loaded one item
// ahead (software-pipelined: a global load's latency per item would otherwise serialise the
// epilogue, measured ~2x slower).  rows = TMA box rows (N for K1, 2H for K3), nk = rup(rows, 8) K rows, NO = MMA N
// (template), S = ring depth, zero_row(ar) = ring rows (atom * nk + row) whose value must be dropped
// (K3: Im of DC / Nyquist).  X slot s (and its lo tile) is refilled only after the MMAs of the item that used it
// have completed (x_empty[s], committed by the MMA warp).
template <int NO, class ZeroRow, class Pre, class Epi>
__device__ __forceinline__ void dft_tc_body(const CUtensorMap* mIn, int64_t P, int64_t Q, int rows, int S,
                                            const uint4* __restrict__ wimg, int w_bytes, ZeroRow zero_row,
                                            Pre&& pre, Epi&& epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ Bars bar;
  __shared__ uint32_t tmem_slot;
  const int nk = rup(rows, 8);
  const uint32_t slot_bytes = slot_bytes_of(nk), ring = ring_off((uint32_t)w_bytes);
  // (slot addresses computed arithmetically: a dynamically indexed pointer array would live in local
  // memory and turn every shared access into a generic one)
  auto xs = [&](int s) { return smem + ring + (uint32_t)(2 * s) * slot_bytes; };
  auto los = [&](int s) { return smem + ring + (uint32_t)(2 * s + 1) * slot_bytes; };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t pblocks = (P + TM - 1) / TM, items = pblocks * Q;
  constexpr int NOA = tmem_cols(NO);
  constexpr int CH = NO / 2;                         // accumulator columns per epilogue warp

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&bar.x_full[i], 1);
      mbar_init(&bar.x_empty[i], 1);
      mbar_init(&bar.lo_full[i], NSPLIT);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.acc_full[i], 1);
      mbar_init(&bar.acc_empty[i], NEPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(2 * NOA));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < w_bytes / 16; i += NTHR) reinterpret_cast<uint4*>(smem)[i] = __ldg(wimg + i);
  // the K padding rows (nk > rows) of the X and lo tiles are never written by TMA: zero the ring once
  for (int i = tid; i < (int)(2 * S * slot_bytes / 16); i += NTHR)
    reinterpret_cast<uint4*>(smem + ring)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (whole warp, lane 0 issues)
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int64_t q = it / pblocks, p0 = (it - q * pblocks) * TM;
      mbar_wait_sleep(&bar.x_empty[s], ph ^ 1, 2000);
      if (lane == 0) {
        expect_tx(&bar.x_full[s], (uint32_t)(4 * rows * 128));
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
          tma_load3(xs(s) + mb * nk * 128, mIn, &bar.x_full[s], (int)(p0 + 32 * mb), (int)q, 0);
      }
      __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, elected lane)
    constexpr uint32_t IDESC = idesc_tf32(TM, NO);
    const uint32_t wh = smem_u32(smem), wl = wh + (uint32_t)(w_bytes / 2);
    int s = 0, n = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ++n) {
      const int d = n & 1;
      mbar_wait(&bar.lo_full[s], ph);
      mbar_wait(&bar.acc_empty[d], ((n >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t xb = smem_u32(xs(s)), lob = smem_u32(los(s)), acc = tmem + (uint32_t)(d * NOA);
      for (int ks = 0; ks < nk / 8; ++ks) {            // small terms first: Xlo Whi + Xhi Wlo
        const uint32_t wo = (uint32_t)((ks >> 2) * NO * 128 + (ks & 3) * 32);
        const uint64_t ah = sdesc(xb + ks * 1024, nk * 128, 512, 1), al = sdesc(lob + ks * 1024, nk * 128, 512, 1);
        mma_tf32(acc, al, sdesc(wh + wo, 16, 1024, 2), IDESC, ks > 0 ? 1u : 0u);
        mma_tf32(acc, ah, sdesc(wl + wo, 16, 1024, 2), IDESC, 1u);
      }
      for (int ks = 0; ks < nk / 8; ++ks) {            // then Xhi Whi
        const uint32_t wo = (uint32_t)((ks >> 2) * NO * 128 + (ks & 3) * 32);
        mma_tf32(acc, sdesc(xb + ks * 1024, nk * 128, 512, 1), sdesc(wh + wo, 16, 1024, 2), IDESC, 1u);
      }
      mma_commit(&bar.x_empty[s]);                     // X tile s and its lo tile free
      mma_commit(&bar.acc_full[d]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp < EPI0) {
    // ------------------------------------------------------------ split: x = hi (in place) + lo
    const int t = tid - 32 * SPLIT0;
    const int nv = (int)(slot_bytes / 16);
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      mbar_wait_sleep(&bar.x_full[s], ph, 1000);
      const uint32_t x = smem_u32(xs(s)), l = smem_u32(los(s));
#pragma unroll 4
      for (int i = t; i < nv; i += 32 * NSPLIT) {
        float4 v = lds128(x + 16 * i);
        if (zero_row(i >> 3)) v = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 h = tf32_hi(v);
        sts128(x + 16 * i, h);
        sts128(l + 16 * i, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) arrive(&bar.lo_full[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3, half = (warp - EPI0) >> 2;
    const int m = lg * 32 + lane;                      // tube of this thread = TMEM lane
    int n = 0;
    auto vnext = pre(blockIdx.x / pblocks, (blockIdx.x % pblocks) * TM, m);
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ++n) {
      const int d = n & 1;
      const int64_t q = it / pblocks, p0 = (it - q * pblocks) * TM;
      const auto v = vnext;
      if (it + gridDim.x < items) {
        const int64_t nx = it + gridDim.x;
        vnext = pre(nx / pblocks, (nx % pblocks) * TM, m);
      }
      mbar_wait_sleep(&bar.acc_full[d], (n >> 1) & 1, 1000);
      tc_fence_after();
      uint32_t r[CH];
#pragma unroll
      for (int c = 0; c < CH; c += 8) {
        uint32_t v[8];
        tmem_ld8(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(d * NOA + half * CH + c), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) r[c + j] = v[j];
      }
      tmem_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive(&bar.acc_empty[d]);
      epi(q, p0, m, half, r, v);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * NOA));
  }
}

// ------------------------------------------------------------------------------ K1 (forward)
// Accumulator columns (compact, NO = rup(2 ceil(N/2), 16)): 0 = Re X_0, 1 = Re X_{N/2} (even N;
// zero column for odd N), (2f, 2f+1) = (Re, Im) X_f for 1 <= f < ceil(N/2).  The imaginary parts of
// the real DC / Nyquist slices are written as exact zeros.  ROLE 0: A (row scale per tube p), ROLE 1:
// B (column scale per q); the scales are K0's exact powers of two.  Output: the fp16
// split planes [f][Re_hi, Re_lo, Im_hi, Im_lo][q][ld], each warp store 32 consecutive p.
template <int NO, int ROLE>
__global__ void __launch_bounds__(NTHR, 1) fwd_dft_tc_kernel(const __grid_constant__ CUtensorMap mX, int64_t P,
                                                             int64_t Q, int N, int S, const uint4* __restrict__ wimg,
                                                             int w_bytes, const unsigned* __restrict__ maxbits,
                                                             __half* __restrict__ out, int64_t ld,
                                                             float* __restrict__ unscale) {
  const int HC = (N + 1) / 2;
  const int64_t plane = Q * ld;
  dft_tc_body<NO>(
      &mX, P, Q, N, S, wimg, w_bytes, [](int) { return false; },
      [&](int64_t q, int64_t p0, int m) -> unsigned {    // K0's max of this tube's row (A) / column (B)
        const int64_t p = p0 + m;
        if (ROLE == 0) return p < P ? __ldg(maxbits + p) : 0u;
        return q < Q ? __ldg(maxbits + q) : 0u;
      },
      [&](int64_t q, int64_t p0, int m, int half, const uint32_t (&r)[NO / 2], unsigned mb) {
        const int64_t p = p0 + m;
        if (p >= P) return;
        const int e = scale_exp(mb, N);
        if (half == 0 && (ROLE == 0 ? q == 0 : (p0 == 0 && m == 0))) unscale[ROLE == 0 ? p : q] = unscale_of(mb, e);
        const float sc = pow2f(e);
        __half* o = out + q * ld + p;
        auto put = [&](int f, float re, float im) {
          const __half2 h = __float22half2_rn(make_float2(re, im));
          const float2 hf = __half22float2(h);
          const __half2 l = __float22half2_rn(make_float2(re - hf.x, im - hf.y));
          __half* of = o + (int64_t)(4 * f) * plane;
          of[PL_RE_HI * plane] = __low2half(h);
          of[PL_RE_LO * plane] = __low2half(l);
          of[PL_IM_HI * plane] = __high2half(h);
          of[PL_IM_LO * plane] = __high2half(l);
        };
#pragma unroll
        for (int j = 0; j < NO / 2; j += 2) {
          const int f = (half * (NO / 2) + j) >> 1;        // column pair (2f, 2f+1)
          if (f == 0) {
            put(0, __uint_as_float(r[j]) * sc, 0.f);       // DC: real
            if (N % 2 == 0) put(N / 2, __uint_as_float(r[j + 1]) * sc, 0.f);   // Nyquist: real
          } else if (f < HC) {
            put(f, __uint_as_float(r[j]) * sc, __uint_as_float(r[j + 1]) * sc);
          }
        }
      });
}

// ------------------------------------------------------------------------------ K3 (inverse)
// NO = rup(N, 16) accumulator columns (output points t), K = 2H rows of C-bar (re, im of f < H).
// Output: X(p, q, t), each warp store 32 consecutive p (128 bytes).
template <int NO>
__global__ void __launch_bounds__(NTHR, 1) inv_dft_tc_kernel(const __grid_constant__ CUtensorMap mC, int64_t P,
                                                             int64_t Q, int N, int S, const uint4* __restrict__ wimg,
                                                             int w_bytes, OutUnscale u, float* __restrict__ X) {
  const int H = N / 2 + 1;
  const int nyq = (N % 2 == 0) ? N + 1 : -1;         // row of Im C_{N/2}; row 1 = Im C_0 (both dropped)
  const float c = 2.f / (float)N;
  const int64_t PQ = P * Q;
  const int nk = rup(2 * H, 8);
  // rows of the 4 M-atoms (atom-major): row r of atom a is ring row a * nk + r
  auto drop = [=](int ar) {
    const int r = ar - nk * (ar >= nk) - nk * (ar >= 2 * nk) - nk * (ar >= 3 * nk);   // row within its atom
    return r == 1 || r == nyq;
  };
  dft_tc_body<NO>(
      &mC, P, Q, 2 * H, S, wimg, w_bytes, drop,
      [&](int64_t q, int64_t p0, int m) -> float2 {      // the tube's unscale factors (R18), one item ahead
        const int64_t p = p0 + m;
        const bool in = p < P && q < Q;
        return make_float2(u.row && in ? __ldg(u.row + p) : 1.f, u.col && in ? __ldg(u.col + q) : 1.f);
      },
      [&](int64_t q, int64_t p0, int m, int half, const uint32_t (&r)[NO / 2], float2 uu) {
        const int64_t p = p0 + m;
        if (p >= P) return;
        const float2 sc = out_scale_of(uu.x, uu.y, c);
        float* xo = X + p + P * q;
#pragma unroll
        for (int j = 0; j < NO / 2; ++j) {
          const int t = half * (NO / 2) + j;
          if (t < N) xo[PQ * t] = apply_scale(__uint_as_float(r[j]), sc);
        }
      });
}

// ------------------------------------------------------------------------------ W tables (host)
// Shared-memory image of a tf32 B operand: two planes (hi, lo) of `rows` K-major rows, K split in
// 32-element atoms of 128-byte rows (atom stride rows * 128 bytes), 128B swizzle (16-byte chunk c of
// row n stored at chunk c ^ (n mod 8)).  hi = value with the low 13 mantissa bits cleared (exactly
// what the tensor core reads), lo = value - hi.  value(n, k) from fn; k >= K is zero.
template <class Fn>
std::vector<float> w_image(int rows, int K, Fn fn) {
  const int atoms = (K + 31) / 32;
  const size_t plane = (size_t)atoms * rows * 32;        // floats per plane
  std::vector<float> img(2 * plane, 0.f);
  for (int nr = 0; nr < rows; ++nr)
    for (int k = 0; k < atoms * 32; ++k) {
      const double v = k < K ? fn(nr, k) : 0.0;
      const float vf = (float)v;
      uint32_t bits;
      std::memcpy(&bits, &vf, 4);
      bits &= TF32_MASK;
      float hi;
      std::memcpy(&hi, &bits, 4);
      const float lo = (float)(v - (double)hi);
      const int a = k / 32, kk = k % 32, chunk = kk / 4, within = kk % 4;
      const size_t idx = (size_t)a * rows * 32 + (size_t)nr * 32 + (size_t)((chunk ^ (nr & 7)) * 4 + within);
      img[idx] = hi;
      img[plane + idx] = lo;
    }
  return img;
}

struct WKey {
  int dev, n, dir;
  bool operator<(const WKey& o) const { return dev != o.dev ? dev < o.dev : n != o.n ? n < o.n : dir < o.dir; }
};
struct WTab {
  const uint4* img = nullptr;
  int bytes = 0;
};

// Device copy of the W image of size n, direction dir (0: forward, 1: inverse), cached per device.
bool get_w(int n, int dir, WTab* out) {
  static std::mutex mu;
  static std::map<WKey, WTab> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  auto itc = cache.find(WKey{dev, n, dir});
  if (itc != cache.end()) { *out = itc->second; return true; }
  std::vector<double> cs(2 * (size_t)n);
  host_twiddles(n, cs.data());                         // (cos, sin)(2 pi m / n), exact octant reduction
  const int H = n / 2 + 1;
  std::vector<float> img;
  if (dir == 0) {
    // compact rows (see fwd_dft_tc_kernel): 0 = cos(0) = 1, 1 = cos(pi k) (even n) or 0,
    // 2f + c = (cos | -sin)(2 pi f k / n) for 1 <= f < ceil(n/2); K = n input points
    const int HC = (n + 1) / 2;
    img = w_image(rup(2 * HC, 16), n, [&](int r, int k) -> double {
      const int f = r >> 1, c = r & 1;
      if (f == 0) return c == 0 ? 1.0 : (n % 2 == 0 ? ((k & 1) ? -1.0 : 1.0) : 0.0);
      if (f >= HC) return 0.0;
      const int m = (int)(((long long)f * k) % n);
      return c == 0 ? cs[2 * m] : -cs[2 * m + 1];
    });
  } else {
    // rows t (output points), K = 2H: (w_f / 2)(cos | -sin)(2 pi f t / n); the 2/n is applied in fp32
    img = w_image(rup(n, 16), 2 * H, [&](int t, int k) -> double {
      const int f = k >> 1, c = k & 1;
      if (t >= n) return 0.0;
      const bool self = (f == 0 || 2 * f == n);
      if (c == 1 && self) return 0.0;
      const double w = self ? 0.5 : 1.0;
      const int m = (int)(((long long)f * t) % n);
      return w * (c == 0 ? cs[2 * m] : -cs[2 * m + 1]);
    });
  }
  void* d = nullptr;
  const size_t bytes = img.size() * sizeof(float);
  if (cudaMalloc(&d, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
  if (cudaMemcpy(d, img.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) { cudaFree(d); return false; }
  WTab t{(const uint4*)d, (int)bytes};
  cache[WKey{dev, n, dir}] = t;
  *out = t;
  return true;
}

int persistent_grid(int64_t items, int num_sms) { return (int)(items < num_sms ? items : num_sms); }

template <int NO, int ROLE>
bool launch_fwd_t(const CUtensorMap& mx, int64_t P, int64_t Q, int N, const WTab& w, const unsigned* maxbits,
                  __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  const int nk = rup(N, 8);
  int S = ring_slots(nk, (uint32_t)w.bytes);
  if (S < 2) return false;
  const size_t smem = ring_off((uint32_t)w.bytes) + (size_t)2 * S * slot_bytes_of(nk) + 1024;
  const void* fn = (const void*)fwd_dft_tc_kernel<NO, ROLE>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  const int64_t items = (P + TM - 1) / TM * Q;
  const uint4* img = w.img;
  int wb = w.bytes;
  void* args[] = {(void*)&mx, (void*)&P, (void*)&Q, (void*)&N, (void*)&S, (void*)&img, (void*)&wb,
                  (void*)&maxbits, (void*)&out, (void*)&ld, (void*)&unscale};
  return cudaLaunchKernel(fn, dim3(persistent_grid(items, num_sms)), dim3(NTHR), args, smem, s) == cudaSuccess;
}

template <int NO>
bool launch_inv_t(const CUtensorMap& mc, int64_t P, int64_t Q, int N, const WTab& w, OutUnscale u, float* X,
                  int num_sms, cudaStream_t s) {
  const int nk = rup(2 * (N / 2 + 1), 8);
  int S = ring_slots(nk, (uint32_t)w.bytes);
  if (S < 2) return false;
  const size_t smem = ring_off((uint32_t)w.bytes) + (size_t)2 * S * slot_bytes_of(nk) + 1024;
  const void* fn = (const void*)inv_dft_tc_kernel<NO>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  const int64_t items = (P + TM - 1) / TM * Q;
  const uint4* img = w.img;
  int wb = w.bytes;
  void* args[] = {(void*)&mc, (void*)&P, (void*)&Q, (void*)&N, (void*)&S, (void*)&img, (void*)&wb, (void*)&u,
                  (void*)&X};
  return cudaLaunchKernel(fn, dim3(persistent_grid(items, num_sms)), dim3(NTHR), args, smem, s) == cudaSuccess;
}

}  // namespace

bool dft_tc_supported(int64_t n3) { return n3 >= 2 && n3 <= 64; }

bool launch_fwd_dft_tc(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                       __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  if (!dft_tc_supported(n3) || P % 4 != 0 || ((uintptr_t)X & 15)) return false;
  const int N = (int)n3;
  WTab w;
  if (!get_w(N, 0, &w)) return false;
  CUtensorMap mx;
  if (!tmap_3d(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, (uint64_t)P, (uint64_t)P, (uint64_t)Q, (uint64_t)N, 32, 1,
               (uint32_t)N, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return false;
  switch (rup(2 * ((N + 1) / 2), 16)) {
    case 16: return role == 0 ? launch_fwd_t<16, 0>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s)
                              : launch_fwd_t<16, 1>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s);
    case 32: return role == 0 ? launch_fwd_t<32, 0>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s)
                              : launch_fwd_t<32, 1>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s);
    case 48: return role == 0 ? launch_fwd_t<48, 0>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s)
                              : launch_fwd_t<48, 1>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s);
    case 64: return role == 0 ? launch_fwd_t<64, 0>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s)
                              : launch_fwd_t<64, 1>(mx, P, Q, N, w, maxbits, out, ld, unscale, num_sms, s);
    default: return false;
  }
}

bool launch_inv_dft_tc(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, OutUnscale u, float* X,
                       int num_sms, cudaStream_t s) {
  if (!dft_tc_supported(n3) || P % 4 != 0 || ld % 4 != 0 || ((uintptr_t)Cre & 15)) return false;
  const int N = (int)n3, H = N / 2 + 1;
  WTab w;
  if (!get_w(N, 1, &w)) return false;
  CUtensorMap mc;
  if (!tmap_3d(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Cre, (uint64_t)P, (uint64_t)ld, (uint64_t)Q,
               (uint64_t)(2 * H), 32, 1, (uint32_t)(2 * H), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return false;
  switch (rup(N, 16)) {
    case 16: return launch_inv_t<16>(mc, P, Q, N, w, u, X, num_sms, s);
    case 32: return launch_inv_t<32>(mc, P, Q, N, w, u, X, num_sms, s);
    case 48: return launch_inv_t<48>(mc, P, Q, N, w, u, X, num_sms, s);
    case 64: return launch_inv_t<64>(mc, P, Q, N, w, u, X, num_sms, s);
    default: return false;
  }
}

}  // namespace tprod
