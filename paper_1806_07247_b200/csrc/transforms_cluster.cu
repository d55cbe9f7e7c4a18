// One-pass long-tube transforms for n3 = 4096 on 8-CTA thread-block clusters (config 4).
//
// K1: Alg. 1 step 1, Eq. (2), Hermitian half only (Eq. (8)),
//     exact 2^e operand scaling and the fp16 hi/lo split.
// K3: Alg. 1 step 2 second branch + step 3 (L177-179): conjugate fill, inverse FFT, 1/N, per-tube
//     unscale (R18).
//
// The four-step form of the FFT, N = 64 * 64, k = k1 + 64 k2, f = f2 + 64 f1:
//   step A:  Y[k1, f2] = w_N^{k1 f2} sum_{k2} x[k1 + 64 k2] w_64^{k2 f2}
//   step B:  X[f2 + 64 f1] = sum_{k1} Y[k1, f2] w_64^{k1 f1}
// The two-pass kernels of transforms_tma.cu run the steps as two launches and move the whole
// intermediate Y through HBM.  Here one cluster of 8 CTAs owns a block of 32 consecutive tubes
// (two real tubes per complex FFT: 16 FFTs) and keeps Y on chip: CTA r TMA-loads the 512 rows
// k1 in [8r, 8r+8) x all k2 (128-byte rows), runs step A on them, multiplies by the twiddle and
// stores each result straight into the shared memory of the CTA that owns its f2 (distributed
// shared memory, st.async counted on the owner's mbarrier); once its 64 KB have arrived a CTA holds
// all k1 of its 8 f2 values and runs step B.  Each operand moves through HBM once (read x, write the split
// spectrum), half the traffic of the two-pass form.
//
// f2 ownership is mirror-closed (f2 and 64 - f2 in the same CTA), so the real-pair separation
// X_f = (Z_f + conj Z_{N-f}) / 2 (N - f = (64 - f2) + 64 (63 - f1)) needs no second exchange:
//   CTA 0:  f2 in {0, 32, 1, 63, 2, 62, 3, 61};   CTA r >= 1:  f2 in {j, 64 - j}, j = 4r .. 4r + 3.
// The inverse runs the same steps backwards (conjugate fill built from the CTA's own Hermitian
// rows, inverse step B over f1, twiddle, exchange by k1, inverse step A over f2, TMA store).
//
// Per CTA: a 64 KB TMA buffer (the next item's load is issued as soon as step A has read it),
// two 64 KB exchange buffers (alternating items), a 4 KB table of the step twiddles; 512 threads; 64-point FFTs as two
// in-place radix-8 Stockham passes over 128 columns (every shared access of a warp is 32
// consecutive float2).
#include "internal.h"
#include "common.cuh"
#include "fft_reg.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>

namespace tprod {

namespace {

using namespace fftreg;

constexpr int CN = 4096, CR = 64;           // N = CR * CR
constexpr int CS = 8;                       // CTAs per cluster
#ifndef TPROD_CL_TUB
#define TPROD_CL_TUB 32
#endif
constexpr int CTUB = TPROD_CL_TUB, CPAIR = CTUB / 2;   // tubes per work item, complex FFTs per item
constexpr int CK = CR / CS;                 // k1 rows (forward input) / f2 slots per CTA
constexpr int COLS = CK * CPAIR;            // FFT columns per CTA (128)
constexpr int CNT = CTUB == 32 ? 512 : 256; // threads per CTA
constexpr int CPS = CTUB == 32 ? 1 : 2;     // CTAs per SM
constexpr int JB = CNT / COLS;              // butterfly rows per column handled side by side (4)
constexpr int BPT = 8 / JB;                 // radix-8 butterflies per thread per pass (2)
constexpr int ZF2 = CR * COLS;              // float2 per buffer (64 KB)
constexpr int SMEM_CL = 3 * ZF2 * 8 + CK * CR * 8 + 256;   // load + 2 exchange buffers, twiddles, f = N/2 rows

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cl(uint32_t a, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void load4(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(s32(dst)), "l"(m), "r"(s32(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void load5(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2, int c3,
                                      int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      ::"r"(s32(dst)), "l"(m), "r"(s32(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void load3(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(s32(dst)), "l"(m), "r"(s32(b)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void store3(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
               "r"(s32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void store4(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
               "r"(s32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void store5(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(m),
               "r"(s32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}

// ---- f2 ownership: mirror pairs {j, 64 - j} stay in one CTA
__device__ __forceinline__ int f2_owner(int f2) {
  if (f2 == 0 || f2 == 32) return 0;
  const int j = f2 < 32 ? f2 : 64 - f2;
  return j >> 2;
}
__device__ __forceinline__ int f2_slot(int f2) {
  if (f2 == 0) return 0;
  if (f2 == 32) return 1;
  const int j = f2 < 32 ? f2 : 64 - f2;
  return (j < 4 ? 2 * j : 2 * (j & 3)) + (f2 > 32 ? 1 : 0);
}
__device__ __forceinline__ int slot_f2(int r, int s) {
  if (r == 0 && s < 2) return s == 0 ? 0 : 32;
  const int j = (r == 0 ? 0 : 4 * r) + s / 2;
  return (s & 1) ? 64 - j : j;
}
// slot holding 64 - f2 (the partner of the real-pair separation / conjugate fill)
__device__ __forceinline__ int mirror_slot(int r, int s) { return (r == 0 && s < 2) ? s : (s ^ 1); }

// ---- 64-point FFTs down the rows of z[64][COLS] (float2), one column per FFT.  Thread t owns
// column t % COLS and butterflies j = t / COLS + JB u, u < BPT (radix 8: 8 butterflies per column).
// Pass 1 (Ns = 1): rows j + 8r -> DFT_8 -> rows 8j + r (in place; all reads before any write).
template <int DIR, bool PRE>
__device__ __forceinline__ void col_pass1(float2* z, float2 pre) {
  const int col = threadIdx.x % COLS, jb = threadIdx.x / COLS;
  float2 v[BPT][8];
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int j = jb + JB * u;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      v[u][r] = z[(j + 8 * r) * COLS + col];
      if (PRE) v[u][r] = make_float2(v[u][r].x * pre.x, v[u][r].y * pre.y);
    }
    dft_reg<8, DIR>(v[u]);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int j = jb + JB * u;
#pragma unroll
    for (int r = 0; r < 8; ++r) z[(8 * j + r) * COLS + col] = v[u][r];
  }
  __syncthreads();
}
// Pass 2 (Ns = 8): rows j + 8r times w_64^{r j} -> DFT_8 -> output index j + 8r (natural order).
// Results stay in v for the caller: v[u][r] is output j + 8r of this thread's column.
template <int DIR>
__device__ __forceinline__ void col_pass2(const float2* z, const float2* __restrict__ tw, float2 (&v)[BPT][8]) {
  const int col = threadIdx.x % COLS, jb = threadIdx.x / COLS;
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int j = jb + JB * u;
#pragma unroll
    for (int r = 0; r < 8; ++r) v[u][r] = z[(j + 8 * r) * COLS + col];
#pragma unroll
    for (int r = 1; r < 8; ++r) v[u][r] = cmul(v[u][r], twN<DIR>(tw, 64 * r * j));   // w_N^{64 rj} = w_64^{rj}
    dft_reg<8, DIR>(v[u]);
  }
}

// Exchange: st.async of each value into the owning CTA's buffer, counted on that CTA's receive
// mbarrier (complete_tx bytes), so a CTA waits only for its own 64 KB, with no cluster-wide barrier
// per item.  The exchange buffers alternate between items: a peer can write buffer b again only at
// item n + 2, which needs this CTA's item-n+1 data, sent after this CTA has finished item n.
__device__ __forceinline__ void st_async(uint32_t a, float2 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(a),
               "f"(v.x), "f"(v.y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cl_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;\nbarrier.cluster.wait;" ::: "memory");
}

// K1: ROLE 0 = A (row scales per tube, applied before the shared FFT), 1 = B (column scale per q).
// Output: split planes [f][plane][q][ld] written directly from registers (64-byte rows per half warp).
template <int ROLE>
__global__ void __launch_bounds__(CNT, CPS) cl_fwd_kernel(const __grid_constant__ CUtensorMap mX, int64_t P, int64_t Q,
                                                        const unsigned* __restrict__ maxbits,
                                                        const float2* __restrict__ tw, __half* __restrict__ out,
                                                        int64_t ld, float* __restrict__ unscale) {
  extern __shared__ __align__(1024) unsigned char smc[];
  float2* X = reinterpret_cast<float2*>(smc);                 // [k2][k1 local][c]   (TMA load)
  float2* W0 = X + ZF2;                                       // [k1][slot][c] -> [f1][slot][c], 2 buffers
  float2* tws = W0 + 2 * ZF2;                                 // w_N^{k1 f2}: [k1 local][f2]
  __shared__ uint64_t full, recv[2];
  const int tid = threadIdx.x;
  const int rank = (int)cl_rank();
  const int col = tid % COLS, c = col % CPAIR, k1l = col / CPAIR, k1 = CK * rank + k1l, jb = tid / COLS;
  const int64_t pblocks = (P + CTUB - 1) / CTUB, items = pblocks * Q;
  const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  if (tid == 0) {
    mb_init(&full, 1);
    mb_init(&recv[0], 1);
    mb_init(&recv[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < CK * CR; i += CNT) tws[i] = twN<-1>(tw, (CK * rank + i / CR) * (i % CR));
  __syncthreads();
  cl_sync_relaxed();                                          // every CTA's barriers initialised
  if (tid == 0 && cid < items) {
    const int64_t q = cid / pblocks, p0 = (cid - q * pblocks) * CTUB;
    mb_expect(&full, ZF2 * 8);
    load4(X, &mX, &full, (int)p0, (int)q, CK * rank, 0);
  }
  const int64_t plane = Q * ld;
  uint32_t n = 0;
  for (int64_t it = cid; it < items; it += ncl, ++n) {
    const int b = n & 1;
    float2* W = W0 + b * ZF2;
    const int64_t q = it / pblocks, p0 = (it - q * pblocks) * CTUB;
    const int64_t p = p0 + 2 * c;
    const bool in0 = p < P, in1 = p + 1 < P;
    float2 pre = make_float2(1.f, 1.f), post = make_float2(1.f, 1.f);
    if (ROLE == 0) {
      const int e0 = in0 ? scale_exp(__ldg(maxbits + p), CN) : 0;
      const int e1 = in1 ? scale_exp(__ldg(maxbits + p + 1), CN) : 0;
      pre = make_float2(pow2f(e0), pow2f(e1));
      if (q == 0 && rank == 0 && tid < CPAIR) {
        if (in0) unscale[p] = unscale_of(__ldg(maxbits + p), e0);
        if (in1) unscale[p + 1] = unscale_of(__ldg(maxbits + p + 1), e1);
      }
    } else {
      const int e = scale_exp(__ldg(maxbits + q), CN);
      post = make_float2(pow2f(e), pow2f(e));
      if (p0 == 0 && rank == 0 && tid == 0) unscale[q] = unscale_of(__ldg(maxbits + q), e);
    }
    mb_wait(&full, n & 1);
    // ---- step A: FFT over k2 for the CTA's 8 k1 rows x 16 pairs
    col_pass1<-1, ROLE == 0>(X, pre);
    float2 v[BPT][8];
    col_pass2<-1>(X, tw, v);
    __syncthreads();                                          // X fully read: refill it
    if (tid == 0) {
      if (it + ncl < items) {
        const int64_t it2 = it + ncl;
        const int64_t q2 = it2 / pblocks, p2 = (it2 - q2 * pblocks) * CTUB;
        fence_async();
        mb_expect(&full, ZF2 * 8);
        load4(X, &mX, &full, (int)p2, (int)q2, CK * rank, 0);
      }
      mb_expect(&recv[b], ZF2 * 8);                           // this item's 64 KB from the cluster
    }
    {
      const uint32_t wa = s32(W) + (uint32_t)((k1 * CK * CPAIR + c) * 8), ra = s32(&recv[b]);
#pragma unroll
      for (int u = 0; u < BPT; ++u) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int f2 = jb + JB * u + 8 * r;
          const uint32_t dst = (uint32_t)f2_owner(f2);
          st_async(cl_mapa(wa + (uint32_t)(f2_slot(f2) * CPAIR * 8), dst), cmul(v[u][r], tws[k1l * CR + f2]),
                   cl_mapa(ra, dst));
        }
      }
    }
    mb_wait(&recv[b], (n >> 1) & 1);                          // all k1 of this CTA's f2 slots
    // ---- step B: FFT over k1 for the CTA's 8 f2 slots x 16 pairs (columns (slot, c))
    col_pass1<-1, false>(W, pre);
    col_pass2<-1>(W, tw, v);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < BPT; ++u)
#pragma unroll
      for (int r = 0; r < 8; ++r) W[(jb + JB * u + 8 * r) * COLS + col] = v[u][r];   // [f1][slot][c]
    __syncthreads();
    // ---- Hermitian half: real-pair separation, 2^e scaling (B), fp16 hi/lo split, stored as
    // half2 (tubes 2c', 2c'+1) into the four planes of row f (CPAIR % ... : c' fixed per thread)
    const int cc = tid % CPAIR;
    const bool st_ok = p0 + 2 * cc < P;                       // P even: both tubes in range
    __half* ob = out + q * ld + p0 + 2 * cc;
    for (int idx = tid; idx < CK * 32 * CPAIR + CPAIR; idx += CNT) {
      int s, f1;
      if (idx < CK * 32 * CPAIR) {
        f1 = (idx / CPAIR) % 32;
        s = idx / (32 * CPAIR);
      } else {                                                // f = N/2: slot 0 of CTA 0, f1 = 32
        if (rank != 0) break;
        f1 = 32;
        s = 0;
      }
      const int f2 = slot_f2(rank, s);
      const float2 zf = W[(f1 * CK + s) * CPAIR + cc];
      const float2 zm = f2 == 0 ? W[(((64 - f1) & 63) * CK + s) * CPAIR + cc]
                                : W[((63 - f1) * CK + mirror_slot(rank, s)) * CPAIR + cc];
      const float2 sc = ROLE == 0 ? make_float2(1.f, 1.f) : post;
      // X_f = (Z_f + conj Z_{N-f}) / 2 ;  Y_f = (Z_f - conj Z_{N-f}) / (2i)
      const float2 re = make_float2(0.5f * (zf.x + zm.x) * sc.x, 0.5f * (zf.y + zm.y) * sc.y);
      const float2 im = make_float2(0.5f * (zf.y - zm.y) * sc.x, -0.5f * (zf.x - zm.x) * sc.y);
      const __half2 rh = __float22half2_rn(re), ih = __float22half2_rn(im);
      const float2 rhf = __half22float2(rh), ihf = __half22float2(ih);
      if (st_ok) {
        __half2* o = reinterpret_cast<__half2*>(ob + (int64_t)(4 * (f2 + CR * f1)) * plane);
        o[0] = rh;                                                                   // PL_RE_HI
        *reinterpret_cast<__half2*>(reinterpret_cast<__half*>(o) + plane) =
            __float22half2_rn(make_float2(re.x - rhf.x, re.y - rhf.y));              // PL_RE_LO
        *reinterpret_cast<__half2*>(reinterpret_cast<__half*>(o) + 2 * plane) = ih;   // PL_IM_HI
        *reinterpret_cast<__half2*>(reinterpret_cast<__half*>(o) + 3 * plane) =
            __float22half2_rn(make_float2(im.x - ihf.x, im.y - ihf.y));              // PL_IM_LO
      }
    }
  }
  cl_sync_relaxed();                                          // no peer still writes this CTA's smem
}

// K3 (same work items): load the CTA's Hermitian C-bar rows f = f2 + 64 f1 (f2 in its slots),
// build Z with the conjugate fill in place, inverse step B over f1, twiddle w_N^{-f2 k1}, exchange by
// k1, inverse step A over f2, 1/N and the per-tube unscale, one TMA store of the rows
// k1 in [8r, 8r+8) x all k2.
__global__ void __launch_bounds__(CNT, CPS) cl_inv_kernel(const __grid_constant__ CUtensorMap mC5,
                                                        const __grid_constant__ CUtensorMap mC3,
                                                        const __grid_constant__ CUtensorMap mXo, int64_t P,
                                                        int64_t Q, const float2* __restrict__ tw, OutUnscale u) {
  extern __shared__ __align__(1024) unsigned char smc[];
  float* L = reinterpret_cast<float*>(smc);                   // [slot][f1 < 32][re|im][32 tubes] -> Z [f1][slot][c]
  float2* Z = reinterpret_cast<float2*>(L);
  float2* Xb0 = Z + ZF2;                                      // [f2][k1 local][c] -> [k2][k1 local][c], 2 buffers
  float2* tws = Xb0 + 2 * ZF2;                                // w_N^{-f2 k1}: [slot][k1]
  float* Lx = reinterpret_cast<float*>(tws + CK * CR);        // [re|im][32 tubes] of f = N/2
  __shared__ uint64_t full, recv[2];
  const int tid = threadIdx.x;
  const int rank = (int)cl_rank();
  const int col = tid % COLS, c = col % CPAIR, jb = tid / COLS;
  const int64_t pblocks = (P + CTUB - 1) / CTUB, items = pblocks * Q;
  const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  const uint32_t lbytes = CK * 32 * 2 * CTUB * 4 + (rank == 0 ? 2 * CTUB * 4 : 0);
  auto issue = [&](int64_t itn) {
    const int64_t q = itn / pblocks, p0 = (itn - q * pblocks) * CTUB;
    mb_expect(&full, lbytes);
#pragma unroll 1
    for (int s = 0; s < CK; ++s) load5(L + s * 32 * 2 * CTUB, &mC5, &full, (int)p0, (int)q, 0, slot_f2(rank, s), 0);
    if (rank == 0) load3(Lx, &mC3, &full, (int)p0, (int)q, 2 * (CN / 2));
  };
  if (tid == 0) {
    mb_init(&full, 1);
    mb_init(&recv[0], 1);
    mb_init(&recv[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < CK * CR; i += CNT) tws[i] = twN<+1>(tw, slot_f2(rank, i / CR) * (i % CR));
  __syncthreads();
  cl_sync_relaxed();
  if (tid == 0 && cid < items) issue(cid);
  uint32_t n = 0;
  for (int64_t it = cid; it < items; it += ncl, ++n) {
    const int b = n & 1;
    float2* Xb = Xb0 + b * ZF2;
    const int64_t q = it / pblocks, p0 = (it - q * pblocks) * CTUB;
    mb_wait(&full, n & 1);
    // ---- Z_f = X_f + i Y_f, f = f2 + 64 f1, with the conjugate fill (Im of DC / N/2 dropped), built in
    // place: Hermitian row (s, f1 < 32) of pair c gives Z[f1][s][c] and, conjugated, the fill
    // Z[63 - f1][s^1][c] (Z[64 - f1][0][c] for f2 = 0); f = N/2 (CTA 0) gives Z[32][0][c].
    constexpr int PER = CK * 32 * CPAIR / CNT;                // Hermitian entries per thread (8)
    float4 e[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = tid + k * CNT;
      const int cc = idx % CPAIR, f1 = (idx / CPAIR) % 32, s = idx / (32 * CPAIR);
      const float* src = L + (s * 32 + f1) * 2 * CTUB;
      const float2 re = reinterpret_cast<const float2*>(src)[cc];
      const float2 im = reinterpret_cast<const float2*>(src + CTUB)[cc];
      e[k] = make_float4(re.x, re.y, im.x, im.y);             // (x_r, y_r, x_i, y_i)
    }
    float4 ex = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rank == 0 && tid < CPAIR) {
      const float2 re = reinterpret_cast<const float2*>(Lx)[tid];
      ex = make_float4(re.x, re.y, 0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = tid + k * CNT;
      const int cc = idx % CPAIR, f1 = (idx / CPAIR) % 32, s = idx / (32 * CPAIR);
      const int f2 = slot_f2(rank, s);
      float4 x = e[k];
      if (f2 == 0 && f1 == 0) x.z = x.w = 0.f;                // DC: Im dropped
      Z[(f1 * CK + s) * CPAIR + cc] = make_float2(x.x - x.w, x.z + x.y);                    // X_f + i Y_f
      if (f2 != 0 || f1 != 0) {
        const int g1 = f2 == 0 ? 64 - f1 : 63 - f1;
        const int sg = f2 == 0 ? s : mirror_slot(rank, s);
        Z[(g1 * CK + sg) * CPAIR + cc] = make_float2(x.x + x.w, x.y - x.z);                 // conj fill
      }
    }
    if (rank == 0 && tid < CPAIR) Z[(32 * CK + 0) * CPAIR + tid] = make_float2(ex.x, ex.y);  // f = N/2 (self)
    __syncthreads();
    // ---- inverse step B: over f1 (columns (slot, c)) -> U[k1][slot][c]
    col_pass1<+1, false>(Z, make_float2(1.f, 1.f));
    float2 v[BPT][8];
    col_pass2<+1>(Z, tw, v);
    __syncthreads();                                          // Z fully read: refill L
    if (tid == 0) {
      if (it + ncl < items) {
        fence_async();
        issue(it + ncl);
      }
      wait_read();            // the previous item's store has read Xb[b ^ 1] (peers refill it at item n + 1)
      mb_expect(&recv[b], ZF2 * 8);
    }
    __syncthreads();
    {
      const int s = col / CPAIR, f2 = slot_f2(rank, s);
      const uint32_t xa = s32(Xb) + (uint32_t)((f2 * CK * CPAIR + c) * 8), ra = s32(&recv[b]);
#pragma unroll
      for (int uu = 0; uu < BPT; ++uu) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int k1 = jb + JB * uu + 8 * r;
          const uint32_t dst = (uint32_t)(k1 / CK);
          st_async(cl_mapa(xa + (uint32_t)((k1 % CK) * CPAIR * 8), dst), cmul(v[uu][r], tws[s * CR + k1]),
                   cl_mapa(ra, dst));
        }
      }
    }
    mb_wait(&recv[b], (n >> 1) & 1);                          // all f2 of this CTA's k1 rows
    // ---- inverse step A: over f2 (columns (k1 local, c)) -> x[k1 + 64 k2]
    col_pass1<+1, false>(Xb, make_float2(1.f, 1.f));
    col_pass2<+1>(Xb, tw, v);
    __syncthreads();
    {
      // 1/N and the per-tube unscale (R18): tubes 2c, 2c + 1 of this column
      const int64_t p = p0 + 2 * c;
      const float2 a = p < P ? out_scale(u.row, p, u.col, q, 1.f / (float)CN) : make_float2(0.f, 0.f);
      const float2 bb = p + 1 < P ? out_scale(u.row, p + 1, u.col, q, 1.f / (float)CN) : make_float2(0.f, 0.f);
#pragma unroll
      for (int uu = 0; uu < BPT; ++uu)
#pragma unroll
        for (int r = 0; r < 8; ++r)
          Xb[(jb + JB * uu + 8 * r) * COLS + col] =
              make_float2((v[uu][r].x * a.x) * a.y, (v[uu][r].y * bb.x) * bb.y);   // [k2][k1 local][c]
    }
    fence_async();
    __syncthreads();
    if (tid == 0) {
      store4(&mXo, Xb, (int)p0, (int)q, CK * rank, 0);
      commit();
    }
  }
  if (tid == 0) wait_all();
  cl_sync_relaxed();
}

// ---- host
PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    else
      cudaGetLastError();
  });
  return fn;
}

// rank-D map; dims / byte strides (D - 1 of them) / box given innermost first
bool make_map(CUtensorMap* m, CUtensorMapDataType t, int D, const void* base, const cuuint64_t* dims,
              const cuuint64_t* strides, const cuuint32_t* box) {
  auto fn = enc();
  if (!fn || ((uintptr_t)base & 15) != 0) return false;
  for (int i = 0; i < D - 1; ++i)
    if (strides[i] % 16 != 0) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, t, (cuuint32_t)D, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <typename K>
bool launch_cluster(K kern, int64_t items, int num_sms, cudaStream_t s, void** args) {
  if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_CL) != cudaSuccess)
    return false;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(CNT);
  cfg.dynamicSmemBytes = SMEM_CL;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_cl = num_sms / CS;
  {
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3((unsigned)(CS * max_cl));
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)kern, &q) == cudaSuccess && ncl > 0)
      max_cl = std::min(max_cl, ncl);
    else
      cudaGetLastError();
  }
  const int64_t ncl = std::min<int64_t>(items, max_cl);
  cfg.gridDim = dim3((unsigned)(ncl * CS));
  return cudaLaunchKernelExC(&cfg, (const void*)kern, args) == cudaSuccess;
}

}  // namespace

bool cluster_fft_supported(int64_t n3) { return n3 == CN; }

bool launch_fwd_cluster(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                        const float2* tw, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  if (!cluster_fft_supported(n3) || !tw || P % 4 != 0 || ld % 2 != 0) return false;
  CUtensorMap mx;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)P, (cuuint64_t)Q, CR, CR};
    const cuuint64_t st[3] = {(cuuint64_t)P * 4, (cuuint64_t)(P * Q) * 4, (cuuint64_t)(P * Q) * CR * 4};
    const cuuint32_t box[4] = {CTUB, 1, CK, CR};
    if (!make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, dims, st, box)) return false;
  }
  const int64_t items = (P + CTUB - 1) / CTUB * Q;
  void* args[] = {(void*)&mx, (void*)&P, (void*)&Q, (void*)&maxbits, (void*)&tw, (void*)&out, (void*)&ld,
                  (void*)&unscale};
  return role == 0 ? launch_cluster(cl_fwd_kernel<0>, items, num_sms, s, args)
                   : launch_cluster(cl_fwd_kernel<1>, items, num_sms, s, args);
}

bool launch_inv_cluster(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const float2* tw,
                        OutUnscale u, float* X, int num_sms, cudaStream_t s) {
  if (!cluster_fft_supported(n3) || !tw || P % 4 != 0 || ld % 4 != 0) return false;
  CUtensorMap mc5, mc3, mxo;
  {   // C-bar planes [f][re|im][q][ld] fp32, row 2 f + ri, f = f2 + 64 f1 (f1 < 32)
    const cuuint64_t row = (cuuint64_t)(Q * ld) * 4;
    const cuuint64_t dims[5] = {(cuuint64_t)P, (cuuint64_t)Q, 2, CR, 32};
    const cuuint64_t st[4] = {(cuuint64_t)ld * 4, row, 2 * row, 2 * CR * row};
    const cuuint32_t box[5] = {CTUB, 1, 2, 1, 32};
    if (!make_map(&mc5, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, Cre, dims, st, box)) return false;
    const cuuint64_t d3[3] = {(cuuint64_t)P, (cuuint64_t)Q, (cuuint64_t)(2 * h_slices(n3))};
    const cuuint64_t s3[2] = {(cuuint64_t)ld * 4, row};
    const cuuint32_t b3[3] = {CTUB, 1, 2};
    if (!make_map(&mc3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Cre, d3, s3, b3)) return false;
  }
  {
    const cuuint64_t dims[4] = {(cuuint64_t)P, (cuuint64_t)Q, CR, CR};
    const cuuint64_t st[3] = {(cuuint64_t)P * 4, (cuuint64_t)(P * Q) * 4, (cuuint64_t)(P * Q) * CR * 4};
    const cuuint32_t box[4] = {CTUB, 1, CK, CR};
    if (!make_map(&mxo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, dims, st, box)) return false;
  }
  const int64_t items = (P + CTUB - 1) / CTUB * Q;
  void* args[] = {(void*)&mc5, (void*)&mc3, (void*)&mxo, (void*)&P, (void*)&Q, (void*)&tw, (void*)&u};
  return launch_cluster(cl_inv_kernel, items, num_sms, s, args);
}

}  // namespace tprod
