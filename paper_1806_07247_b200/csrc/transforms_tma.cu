// TMA-staged mode-3 transforms.  (1) Persistent dense forward DFT for non-power-of-two
// 32 < n3 <= 64 (fwd_tma_kernel; the inverse of those sizes runs the register kernels of
// transforms_dense.cu, measured faster).  Same arithmetic as transforms_dense.cu (conjugate-pair
// folding, compile-time twiddle indices into a constant-bank table), different data movement:
//
//   * a work item is 256 consecutive tubes p0..p0+255 of one q;
//   * one thread TMA-loads the item's whole tile  X(p0:p0+256, q, 0:n3)  (a 3-D box, the
//     out-of-range tail zero-filled) into a shared-memory buffer, double-buffered across the
//     persistent loop, so HBM latency overlaps the arithmetic of the previous item without
//     holding the tile in registers;
//   * each thread reads its TPT adjacent tubes from smem (conflict-free) and writes half2/__half
//     results, warp-coalesced along p.  TPT = 2 for n3 <= 32, else 1 (register budget).
// (2) Tube-parallel Stockham FFTs for power-of-two n3 (K1 and K3) and (3) the four-step long-tube
// transforms, described at their kernels below.
//
// K1: Alg. 1 step 1, Eq. (2), Hermitian half (Eq. (8)).
// K3: Alg. 1 step 2 second branch + step 3 (L177-179): fused conjugate fill + inverse DFT.
#include "internal.h"
#include "common.cuh"
#include "fft_reg.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <mutex>
#include <algorithm>
#include <vector>

namespace tprod {

namespace {

constexpr int TMAX = 64;
constexpr int TP = 256;          // tubes per work item
__constant__ float2 c_tw2[TMAX * (TMAX + 1) / 2];
__host__ __device__ constexpr int toff(int N) { return N * (N - 1) / 2; }
__host__ __device__ constexpr int tpt_of(int N) { return N <= 32 ? 2 : 1; }

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(su32(dst)), "l"(m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// bulk tensor store smem -> global (async proxy); completion tracked by bulk groups
__device__ __forceinline__ void tma_store3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct Item {
  int64_t q, p0;
};
template <int TPI = TP>
__device__ __forceinline__ Item item_of(int64_t it, int64_t pblocks) {
  Item r;
  r.q = it / pblocks;
  r.p0 = (it - r.q * pblocks) * TPI;
  return r;
}

// Persistent double-buffered TMA pipeline shared by K1 and K3: calls body(item, smem buffer) for
// every work item of this CTA.  BUF = floats per buffer; box = {TPI, 1, rows} (TPI tubes per item).
template <int BUF, int TPI = TP, typename Body>
__device__ __forceinline__ void tma_pipeline(const CUtensorMap* m, int64_t P, int64_t Q, float* smem,
                                             uint64_t* full, Body&& body) {
  const int tid = threadIdx.x;
  const int64_t pblocks = (P + TPI - 1) / TPI;
  const int64_t items = pblocks * Q;
  if (tid == 0) {
    bar_init(&full[0], 1);
    bar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t it0 = blockIdx.x;
  if (tid == 0 && it0 < items) {
    const Item nx = item_of<TPI>(it0, pblocks);
    bar_expect(&full[0], BUF * 4);
    tma3d(smem, m, &full[0], (int)nx.p0, (int)nx.q, 0);
  }
  int n = 0;
  for (int64_t it = it0; it < items; it += gridDim.x, ++n) {
    const int b = n & 1;
    if (tid == 0 && it + gridDim.x < items) {       // prefetch the next item into the other buffer
      const Item nx = item_of<TPI>(it + gridDim.x, pblocks);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_expect(&full[b ^ 1], BUF * 4);
      tma3d(smem + (b ^ 1) * BUF, m, &full[b ^ 1], (int)nx.p0, (int)nx.q, 0);
    }
    bar_wait(&full[b], (n >> 1) & 1);
    body(item_of<TPI>(it, pblocks), smem + b * BUF);
    __syncthreads();      // buffer b fully consumed before it is refilled (two iterations on)
  }
}

// K2 -> K3 overlap, streaming consumer (internal.h OverlapK3::stream): the items are numbered in the
// GEMM's tile-completion order -- (m, n) tile r = m * nt + n slowest, inside a tile the 128 lateral
// slices of each of its `ppm` tube blocks -- and handed out by the device counter `work`; thread 0
// waits (acquire, bounded: a counter that never completes traps) for the tile's counter before it
// issues the TMA load (fence.proxy.async: the GEMM's generic-proxy stores, acquired by this thread,
// ordered before the async-proxy read).  CTAs resident while the GEMM still runs (on the SMs its
// cluster grid leaves idle) thus invert finished m-rows; the rest join when the GEMM's CTAs exit.
struct TubeOv {
  const int* done;
  int* work;
  int target, ppm, nt;
};
template <int BUF, int TPI, typename Body>
__device__ __forceinline__ void tma_pipeline_ov(const CUtensorMap* m, int64_t P, int64_t Q, float* smem,
                                                uint64_t* full, const TubeOv& ov, Body&& body) {
  __shared__ long long s_item[2];                    // (q << 32) | p0 of the item in buffer b, -1 = none
  const int tid = threadIdx.x;
  const int64_t pblocks = (P + TPI - 1) / TPI;
  const int per = 128 * ov.ppm;                      // items per (m, n) tile (GEMM N tile = 128)
  const int64_t total = ((pblocks + ov.ppm - 1) / ov.ppm) * ov.nt * per;
  if (tid == 0) {
    bar_init(&full[0], 1);
    bar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int ready = -1;                                    // last tile seen complete (thread 0)
  auto fetch = [&](int slot) {                       // thread 0: next item into buffer `slot`
    for (;;) {
      const int64_t i = atomicAdd(ov.work, 1);
      if (i >= total) {
        s_item[slot] = -1;
        return;
      }
      const int r = (int)(i / per), j = (int)(i - (int64_t)r * per);
      const int64_t q = (int64_t)(r % ov.nt) * 128 + (j & 127);
      const int64_t pb = (int64_t)(r / ov.nt) * ov.ppm + (j >> 7);
      if (q >= Q || pb >= pblocks) continue;         // ragged edge of the tile grid
      if (r != ready) {
        const int* c = ov.done + r;
        int v;
        uint64_t t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
          if (v >= ov.target) break;
          __nanosleep(1000);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > 8000000000ull) __trap();
        }
        ready = r;
      }
      asm volatile("fence.proxy.async;" ::: "memory");
      bar_expect(&full[slot], BUF * 4);
      tma3d(smem + slot * BUF, m, &full[slot], (int)(pb * TPI), (int)q, 0);
      s_item[slot] = (long long)((q << 32) | (pb * TPI));
      return;
    }
  };
  if (tid == 0) fetch(0);
  __syncthreads();
  for (int n = 0;; ++n) {
    const int b = n & 1;
    const long long cur = s_item[b];
    if (cur < 0) break;
    if (tid == 0) fetch(b ^ 1);                      // prefetch (buffer b ^ 1 was released by the last barrier)
    bar_wait(&full[b], (n >> 1) & 1);
    Item it;
    it.q = cur >> 32;
    it.p0 = cur & 0xffffffffll;
    body(it, smem + b * BUF);
    __syncthreads();
  }
}

// load TPT adjacent floats of row r of a [rows][TP] smem tile
template <int TPT>
__device__ __forceinline__ void lds(const float* s, int r, int tid, float (&o)[TPT]) {
  if constexpr (TPT == 2) {
    const float2 v = reinterpret_cast<const float2*>(s + r * TP)[tid];
    o[0] = v.x;
    o[1] = v.y;
  } else {
    o[0] = s[r * TP + tid];
  }
}

template <int TPT>
__device__ __forceinline__ void store_split(__half* dst_hi, __half* dst_lo, const float (&v)[TPT], bool full_pair) {
  if constexpr (TPT == 2) {
    const float2 x = make_float2(v[0], v[1]);
    const __half2 h = __float22half2_rn(x);
    const float2 hf = __half22float2(h);
    const __half2 l = __float22half2_rn(make_float2(x.x - hf.x, x.y - hf.y));
    if (full_pair) {
      *reinterpret_cast<__half2*>(dst_hi) = h;
      *reinterpret_cast<__half2*>(dst_lo) = l;
    } else {
      *dst_hi = __low2half(h);
      *dst_lo = __low2half(l);
    }
  } else {
    __half h, l;
    split_f16(v[0], h, l);
    *dst_hi = h;
    *dst_lo = l;
  }
}

template <int N, int ROLE>
__global__ void __launch_bounds__(TP / tpt_of(N)) fwd_tma_kernel(const __grid_constant__ CUtensorMap mX,
                                                                int64_t P, int64_t Q,
                                                                const unsigned* __restrict__ maxbits,
                                                                __half* __restrict__ out, int64_t ld,
                                                                float* __restrict__ unscale) {
  constexpr int H = N / 2 + 1;
  constexpr int K2 = (N - 1) / 2;
  constexpr int TPT = tpt_of(N);
  constexpr int BUF = TP * N;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const int64_t plane = Q * ld;
  tma_pipeline<BUF>(&mX, P, Q, smem, full, [&](const Item& cur, const float* s) {
    const int64_t p = cur.p0 + TPT * tid;
    if (p >= P) return;
    const bool pair = (TPT == 2) && (p + 1 < P);
    float v[N][TPT];
#pragma unroll
    for (int k = 0; k < N; ++k) lds<TPT>(s, k, tid, v[k]);
    float u[K2 + 1][TPT], w[K2 + 1][TPT];
#pragma unroll
    for (int k = 1; k <= K2; ++k)
#pragma unroll
      for (int t = 0; t < TPT; ++t) {
        u[k][t] = v[k][t] + v[N - k][t];
        w[k][t] = v[k][t] - v[N - k][t];
      }
    const int64_t q = cur.q;
    float sc[TPT];
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      int e = 0;
      if (ROLE == 0) {
        if (p + t < P) e = scale_exp(__ldg(maxbits + p + t), N);
        if (q == 0 && p + t < P) unscale[p + t] = unscale_of(__ldg(maxbits + p + t), e);
      } else {
        e = scale_exp(__ldg(maxbits + q), N);
        if (p == 0 && t == 0) unscale[q] = unscale_of(__ldg(maxbits + q), e);
      }
      sc[t] = pow2f(e);
    }
    __half* o = out + q * ld + p;
#pragma unroll
    for (int f = 0; f < H; ++f) {
      float re[TPT], im[TPT];
#pragma unroll
      for (int t = 0; t < TPT; ++t) {
        re[t] = v[0][t];
        im[t] = 0.f;
      }
#pragma unroll
      for (int k = 1; k <= K2; ++k) {
        const float2 tw = c_tw2[toff(N) + (f * k) % N];
#pragma unroll
        for (int t = 0; t < TPT; ++t) {
          re[t] = fmaf(u[k][t], tw.x, re[t]);
          im[t] = fmaf(-w[k][t], tw.y, im[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < TPT; ++t) {
        if (N % 2 == 0) re[t] += (f & 1) ? -v[N / 2][t] : v[N / 2][t];
        re[t] *= sc[t];
        im[t] *= sc[t];
      }
      __half* of = o + (int64_t)(4 * f) * plane;
      store_split<TPT>(of + PL_RE_HI * plane, of + PL_RE_LO * plane, re, pair);
      store_split<TPT>(of + PL_IM_HI * plane, of + PL_IM_LO * plane, im, pair);
    }
  });
}

// ------------------------------------------------------------------------------ tube-parallel FFT
// Power-of-two 32 <= n3 <= 256 (configs 2 and 5): a work item is TUB = 2F consecutive tubes of
// one q (F = min(4096 / N, 128) complex FFTs, two real tubes packed per FFT as in
// transforms_fft.cu), TMA-loaded as the tile X(p0:p0+TUB, q, 0:N).  Read as float2 that tile IS
// the point-major layout z[k][c] (c = tube pair), so the radix-16 (+ 8/4/2) Stockham passes run
// in place on the TMA buffer with the F FFTs of a warp side by side: every shared access of a warp
// is 32 consecutive float2 (conflict-free) and every twiddle w_{Ns R}^{r k} is warp-uniform (one
// broadcast load from the handle's per-pass table).  Outputs are 128-byte warp rows (half2 planes
// for K1, float2 rows for K3).
//   K1: Alg. 1 step 1, Hermitian half (Eq. (8)), 2^e scale, fp16 split.
//   K3: Alg. 1 step 2 second branch + step 3 (L177-179): conjugate fill, inverse FFT, 1/N.
using namespace fftreg;

constexpr int TUBE_NT = 256;
// rows per TMA store box for R output rows: R / k for the smallest k with R / k <= 256, k | R
__host__ __device__ constexpr int store_rows(int R, int k = 1) {
  return (R % k == 0 && R / k <= 256) ? R / k : store_rows(R, k + 1);
}

template <int N>
struct TubeCfg {
  static constexpr int F = (4096 / N) > 128 ? 128 : 4096 / N;   // complex FFTs per item
  static constexpr int TUB = 2 * F;                              // tubes per item (TMA box <= 256)
  static constexpr int LOG = N == 32 ? 5 : N == 64 ? 6 : N == 128 ? 7 : 8;
  static constexpr int NP = LOG / 4 + (LOG % 4 ? 1 : 0);         // passes: radix 16, then 2^(LOG%4)
};
__host__ __device__ constexpr int tube_R(int log, int i) { return i < log / 4 ? 16 : 1 << (log % 4); }
__host__ __device__ constexpr int tube_Ns(int i) { return i == 0 ? 1 : 16 << (4 * (i - 1)); }
// twiddle-table offset of pass i (make_plan layout of transforms_fft.cu: (R - 1) Ns entries per
// pass with Ns > 1)
__host__ __device__ constexpr int tube_toff(int log, int i) {
  return i <= 1 ? 0 : tube_toff(log, i - 1) + (tube_R(log, i - 1) - 1) * tube_Ns(i - 1);
}

// PRE: multiply the loaded values by `pre` (the thread's column c = threadIdx.x % F is the same for
// all its butterflies since NT % F == 0): per-tube exact scales applied before two real tubes share
// one complex FFT, so neither tube's rounding error is large relative to the other's scale.
// POST: multiply the results by post1 then post2 (per tube of the pair, same fixed column) before
// they are stored: the inverse's per-output-tube unscale of DESIGN.md R18.
template <int N, int F, int R, int Ns, int DIR, int NT = TUBE_NT, bool PRE = false, bool POST = false>
__device__ __forceinline__ void tube_pass(float2* z, const float2* __restrict__ tp, float2 pre = make_float2(1.f, 1.f),
                                          float2 post1 = make_float2(1.f, 1.f), float2 post2 = make_float2(1.f, 1.f)) {
  constexpr int NB = N / R;
  constexpr int BPT = F * NB / NT;
  static_assert(F * NB % NT == 0, "butterflies must divide evenly");
  static_assert(!PRE || NT % F == 0, "pre-scale needs a fixed column per thread");
  float2 v[BPT][R];
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int b = threadIdx.x + u * NT;
    const int c = b % F, j = b / F, k = j % Ns;
#pragma unroll
    for (int r = 0; r < R; ++r) v[u][r] = z[(j + r * NB) * F + c];
    if (PRE) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = make_float2(v[u][r].x * pre.x, v[u][r].y * pre.y);
    }
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[u][r] = cmul(v[u][r], twN<DIR>(tp, (r - 1) * Ns + k));
    }
    dft_reg<R, DIR>(v[u]);
    if (POST) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        v[u][r] = make_float2((v[u][r].x * post1.x) * post2.x, (v[u][r].y * post1.y) * post2.y);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int b = threadIdx.x + u * NT;
    const int c = b % F, j = b / F, k = j % Ns, g = j / Ns;
#pragma unroll
    for (int r = 0; r < R; ++r) z[(g * Ns * R + k + r * Ns) * F + c] = v[u][r];
  }
  __syncthreads();
}

template <int N, int DIR, int F = TubeCfg<N>::F, int NT = TUBE_NT, bool PRE = false, bool POST = false>
__device__ __forceinline__ void tube_fft(float2* z, const float2* __restrict__ st, float2 pre = make_float2(1.f, 1.f),
                                         float2 post1 = make_float2(1.f, 1.f), float2 post2 = make_float2(1.f, 1.f)) {
  using C = TubeCfg<N>;
  static_assert(C::NP <= 2, "tube FFTs have at most two passes");
  if constexpr (C::NP == 1) {
    tube_pass<N, F, tube_R(C::LOG, 0), tube_Ns(0), DIR, NT, PRE, POST>(z, st, pre, post1, post2);
  } else {
    tube_pass<N, F, tube_R(C::LOG, 0), tube_Ns(0), DIR, NT, PRE>(z, st, pre);
    tube_pass<N, F, tube_R(C::LOG, 1), tube_Ns(1), DIR, NT, false, POST>(z, st + tube_toff(C::LOG, 1),
                                                                          make_float2(1.f, 1.f), post1, post2);
  }
}

// K1 epilogue staged in shared memory: the item's 4h output rows (f, plane) of TUB halves are
// written with 32-bit shared stores and leave as TMA bulk tensor stores (<= 256 rows per box), so
// the SM issues no 64-bit global address arithmetic and HBM sees whole 256-byte rows.
template <int N, int ROLE>
__global__ void __launch_bounds__(TUBE_NT) fwd_tube_kernel(const __grid_constant__ CUtensorMap mX,
                                                          const __grid_constant__ CUtensorMap mO, int64_t P,
                                                          int64_t Q, const unsigned* __restrict__ maxbits,
                                                          const float2* __restrict__ st, float* __restrict__ unscale) {
  using C = TubeCfg<N>;
  constexpr int F = C::F, TUB = C::TUB, H = N / 2 + 1;
  constexpr int BUF = TUB * N;                      // floats per input buffer
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full[2];
  __half2* stg = reinterpret_cast<__half2*>(smem + 2 * BUF);   // [4h][TUB / 2] output rows
  const int c = threadIdx.x % F;                    // TUBE_NT % F == 0: fixed tube pair per thread
  tma_pipeline<BUF, TUB>(&mX, P, Q, smem, full, [&](const Item& cur, float* s) {
    float2* z = reinterpret_cast<float2*>(s);       // z[k][c] = (x_{2c}[k], x_{2c+1}[k])
    const int64_t q = cur.q, p = cur.p0 + 2 * c;
    const bool in0 = p < P, in1 = p + 1 < P;
    int e0 = 0, e1 = 0;
    if (ROLE == 0) {
      if (in0) e0 = scale_exp(__ldg(maxbits + p), N);
      if (in1) e1 = scale_exp(__ldg(maxbits + p + 1), N);
      if (q == 0 && threadIdx.x < F) {
        if (in0) unscale[p] = unscale_of(__ldg(maxbits + p), e0);
        if (in1) unscale[p + 1] = unscale_of(__ldg(maxbits + p + 1), e1);
      }
    } else {
      e0 = e1 = scale_exp(__ldg(maxbits + q), N);
      if (cur.p0 == 0 && threadIdx.x == 0) unscale[q] = unscale_of(__ldg(maxbits + q), e0);
    }
    // A's two tubes of a pair have their own row scales: applied before the shared FFT (exact
    // powers of two); B's pair shares its column scale, applied after
    const float s0 = ROLE == 0 ? 1.f : pow2f(e0), s1 = ROLE == 0 ? 1.f : pow2f(e1);
    if (ROLE == 0)
      tube_fft<N, -1, F, TUBE_NT, true>(z, st, make_float2(pow2f(e0), pow2f(e1)));
    else
      tube_fft<N, -1>(z, st);
    if (threadIdx.x == 0) bulk_wait_read();         // the previous item's stores have read stg
    __syncthreads();
#pragma unroll 4
    for (int f = threadIdx.x / F; f < H; f += TUBE_NT / F) {
      const float2 zf = z[f * F + c], zm = z[((N - f) % N) * F + c];
      // X_f = (Z_f + conj Z_{N-f}) / 2 ;  Y_f = (Z_f - conj Z_{N-f}) / (2i)
      const float2 re = make_float2(0.5f * (zf.x + zm.x) * s0, 0.5f * (zf.y + zm.y) * s1);
      const float2 im = make_float2(0.5f * (zf.y - zm.y) * s0, -0.5f * (zf.x - zm.x) * s1);
      const __half2 rh = __float22half2_rn(re), ih = __float22half2_rn(im);
      const float2 rhf = __half22float2(rh), ihf = __half22float2(ih);
      __half2* row = stg + (4 * f) * (TUB / 2) + c;
      row[PL_RE_HI * (TUB / 2)] = rh;
      row[PL_RE_LO * (TUB / 2)] = __float22half2_rn(make_float2(re.x - rhf.x, re.y - rhf.y));
      row[PL_IM_HI * (TUB / 2)] = ih;
      row[PL_IM_LO * (TUB / 2)] = __float22half2_rn(make_float2(im.x - ihf.x, im.y - ihf.y));
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      constexpr int RB = store_rows(4 * H);
#pragma unroll
      for (int r0 = 0; r0 < 4 * H; r0 += RB) tma_store3d(&mO, stg + r0 * (TUB / 2), (int)cur.p0, (int)q, r0);
      bulk_commit();
    }
  });
  if (threadIdx.x == 0) bulk_wait_all();
}

// K3: the 1/N of the inverse is applied while Z is built (a power of two: exact), the per-tube
// unscale (R18) by the last FFT pass, and the transformed tile z[k][c] -- which read as floats IS
// the output rows X(p0:p0+TUB, q, k) -- leaves by one TMA bulk tensor store.
template <int N>
__global__ void __launch_bounds__(TUBE_NT) inv_tube_kernel(const __grid_constant__ CUtensorMap mC,
                                                          const __grid_constant__ CUtensorMap mXo, int64_t P,
                                                          int64_t Q, const float2* __restrict__ st, OutUnscale u,
                                                          TubeOv ov) {
  using C = TubeCfg<N>;
  constexpr int F = C::F, TUB = C::TUB, H = N / 2 + 1;
  constexpr int BUF = TUB * 2 * H;                  // C-bar tile: rows [f][re|im], TUB floats each
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full[2];
  float2* z = reinterpret_cast<float2*>(smem + 2 * BUF);     // z[k][c], separate from the TMA buffers
  const float inv_n = 1.f / (float)N;
  auto body = [&](const Item& cur, const float* s) {
    if (threadIdx.x == 0) bulk_wait_read();                  // the previous item's store has read z
    __syncthreads();
    // Z / N = (X + i Y) / N with the conjugate fill (Im of DC / Nyquist dropped: C2R)
    for (int idx = threadIdx.x; idx < H * F; idx += TUBE_NT) {
      const int c = idx % F, f = idx / F;
      const bool self = (f == 0 || 2 * f == N);
      const float2 re = reinterpret_cast<const float2*>(s + (2 * f) * TUB)[c];       // (x_r, y_r)
      const float2 im = self ? make_float2(0.f, 0.f)
                             : reinterpret_cast<const float2*>(s + (2 * f + 1) * TUB)[c];  // (x_i, y_i)
      z[f * F + c] = make_float2((re.x - im.y) * inv_n, (im.x + re.y) * inv_n);        // X_f + i Y_f
      if (!self) z[(N - f) * F + c] = make_float2((re.x + im.y) * inv_n, (re.y - im.x) * inv_n);
    }
    __syncthreads();
    {
      const int64_t p = cur.p0 + 2 * (threadIdx.x % F);         // this thread's tube pair (TUBE_NT % F == 0)
      const float2 a = p < P ? out_scale(u.row, p, u.col, cur.q, 1.f) : make_float2(0.f, 0.f);
      const float2 b = p + 1 < P ? out_scale(u.row, p + 1, u.col, cur.q, 1.f) : make_float2(0.f, 0.f);
      tube_fft<N, +1, F, TUBE_NT, false, true>(z, st, make_float2(1.f, 1.f), make_float2(a.x, b.x),
                                               make_float2(a.y, b.y));
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store3d(&mXo, z, (int)cur.p0, (int)cur.q, 0);
      bulk_commit();
    }
  };
  if (ov.done) tma_pipeline_ov<BUF, TUB>(&mC, P, Q, smem, full, ov, body);
  else tma_pipeline<BUF, TUB>(&mC, P, Q, smem, full, body);
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------ four-step K1
// Long power-of-two tubes, N = N1 * N2 (N1, N2 in {64, 128}: n3 = 4096, 8192, 16384).  With
// k = k1 + N1 k2 and f = N2 f1 + f2 (Eq. (2) split into two short DFTs, the four-step form of the
// FFT of PAPER.md:L102):
//   pass 1:  Y[k1, f2] = w_N^{k1 f2} sum_{k2} x[k1 + N1 k2] w_{N2}^{k2 f2}      (stored at row k1 + N1 f2)
//   pass 2:  X[N2 f1 + f2] = sum_{k1} Y[k1, f2] w_{N1}^{k1 f1}
// Both passes are tube-parallel (TUB consecutive tubes side by side, two real tubes per complex
// FFT): TMA gathers the N2 rows k1 + N1 k2 (pass 1) or the N1 rows k1 + N1 f2 (pass 2) of a 4-D view
// {p, q, k1, k2} of the tensor, so every row moved is TUB*4 contiguous bytes (vs 32 bytes for the
// one-pass kernel, whose 8 tubes x N points fill a CTA's shared memory).  The intermediate Y has
// the input's shape (W, a workspace the size of the larger operand).  Pass 2 handles f2 together
// with N2 - f2, so both X_f and X_{N-f} of the real-pair separation are in shared memory.
template <int N2, int TUB>
__global__ void __launch_bounds__(2 * TUB) fwd4_pass1_kernel(const __grid_constant__ CUtensorMap mX4,
                                                            const __grid_constant__ CUtensorMap mW4, int64_t P,
                                                            int64_t Q, int N1, const float2* __restrict__ st2,
                                                            const float2* __restrict__ twN,
                                                            const unsigned* __restrict__ rowmax) {
  constexpr int F = TUB / 2, NT = 2 * TUB;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full;
  float2* z = reinterpret_cast<float2*>(smem);      // z[k2][c]
  if (threadIdx.x == 0) {
    bar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t items = pblocks * Q * N1;
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1) {
    const int k1 = (int)(it % N1);
    const int64_t r = it / N1;
    const int64_t q = r / pblocks, p0 = (r - q * pblocks) * TUB;
    if (threadIdx.x == 0) {
      bulk_wait_read();                             // the previous item's store has read z
      fence_async_smem();
      bar_expect(&full, TUB * N2 * 4);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
          ::"r"(su32(smem)), "l"(&mX4), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(k1), "r"(0)
          : "memory");
    }
    bar_wait(&full, ph);
    if (rowmax) {
      // A (row scales): the pair's own exact scales before the shared FFT (pass 2 then skips them)
      const int64_t p = p0 + 2 * (threadIdx.x % F);
      const int N = N1 * N2;
      const float s0 = p < P ? pow2f(scale_exp(__ldg(rowmax + p), N)) : 1.f;
      const float s1 = p + 1 < P ? pow2f(scale_exp(__ldg(rowmax + p + 1), N)) : 1.f;
      tube_fft<N2, -1, F, NT, true>(z, st2, make_float2(s0, s1));   // over k2 -> z[f2][c]
    } else {
      tube_fft<N2, -1, F, NT>(z, st2);
    }
    for (int idx = threadIdx.x; idx < N2 * F; idx += NT) {
      const int f2 = idx / F;
      const float2 t = __ldg(twN + k1 * f2);          // w_N^{k1 f2} = (cos, -sin), k1 f2 < N
      z[idx] = cmul(z[idx], make_float2(t.x, -t.y));
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
                   ::"l"(&mW4), "r"(su32(smem)), "r"((int)p0), "r"((int)q), "r"(k1), "r"(0)
                   : "memory");
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

template <int N1, int TUB, int ROLE>
__global__ void __launch_bounds__(2 * TUB) fwd4_pass2_kernel(const __grid_constant__ CUtensorMap mW4, int64_t P,
                                                            int64_t Q, int N2, const unsigned* __restrict__ maxbits,
                                                            const float2* __restrict__ st1, __half* __restrict__ out,
                                                            int64_t ld, int64_t plane, float* __restrict__ unscale) {
  constexpr int F = TUB / 2, NT = 2 * TUB;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full;
  float2* za = reinterpret_cast<float2*>(smem);               // [f1][c] of column f2
  float2* zb = za + N1 * F;                                   // [f1][c] of column N2 - f2
  const int N = N1 * N2;
  if (threadIdx.x == 0) {
    bar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int half = N2 / 2;
  const int64_t items = pblocks * Q * (half + 1);
  const int c = threadIdx.x % F;                                // NT % F == 0
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1) {
    const int f2 = (int)(it % (half + 1));
    const int64_t r = it / (half + 1);
    const int64_t q = r / pblocks, p0 = (r - q * pblocks) * TUB;
    const int f2b = (N2 - f2) % N2;
    const bool two = f2b != f2;
    if (threadIdx.x == 0) {
      bar_expect(&full, (two ? 2 : 1) * TUB * N1 * 4);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
          ::"r"(su32(za)), "l"(&mW4), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(0), "r"(f2)
          : "memory");
      if (two)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
            ::"r"(su32(zb)), "l"(&mW4), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(0), "r"(f2b)
            : "memory");
    }
    bar_wait(&full, ph);
    tube_fft<N1, -1, F, NT>(za, st1);                           // over k1 -> X[N2 f1 + f2]
    if (two) tube_fft<N1, -1, F, NT>(zb, st1);
    // ---- Hermitian half, real-pair separation, 2^e scaling, fp16 hi/lo split
    const int64_t p = p0 + 2 * c;
    if (p < P) {
      const bool in1 = p + 1 < P;
      int e0 = 0, e1 = 0;
      if (ROLE == 0) {
        e0 = scale_exp(__ldg(maxbits + p), N);
        if (in1) e1 = scale_exp(__ldg(maxbits + p + 1), N);
        if (q == 0 && f2 == 0 && threadIdx.x < F) {
          unscale[p] = unscale_of(__ldg(maxbits + p), e0);
          if (in1) unscale[p + 1] = unscale_of(__ldg(maxbits + p + 1), e1);
        }
      } else {
        e0 = e1 = scale_exp(__ldg(maxbits + q), N);
        if (p0 == 0 && f2 == 0 && threadIdx.x == 0) unscale[q] = unscale_of(__ldg(maxbits + q), e0);
      }
      const float s0 = ROLE == 0 ? 1.f : pow2f(e0), s1 = ROLE == 0 ? 1.f : pow2f(e1);   // A: applied in pass 1
      __half* o = out + q * ld + p;
      for (int t = 0; t < (two ? 2 : 1); ++t) {
        const float2* zt = t == 0 ? za : zb;
        const float2* zo = t == 0 ? zb : za;                    // tile holding the partners
        const int fc = t == 0 ? f2 : f2b;
        for (int f1 = threadIdx.x / F; f1 < N1; f1 += NT / F) {
          const int f = N2 * f1 + fc;
          if (2 * f > N) continue;
          const float2 zf = zt[f1 * F + c];
          // X_{N-f}: f2 = 0 -> row (N1 - f1) mod N1 of the same column, else row N1-1-f1 of N2 - f2
          const float2 zm = fc == 0 ? zt[((N1 - f1) % N1) * F + c] : (two ? zo : zt)[(N1 - 1 - f1) * F + c];
          const float2 re = make_float2(0.5f * (zf.x + zm.x) * s0, 0.5f * (zf.y + zm.y) * s1);
          const float2 im = make_float2(0.5f * (zf.y - zm.y) * s0, -0.5f * (zf.x - zm.x) * s1);
          const __half2 rh = __float22half2_rn(re), ih = __float22half2_rn(im);
          const float2 rhf = __half22float2(rh), ihf = __half22float2(ih);
          const __half2 rl = __float22half2_rn(make_float2(re.x - rhf.x, re.y - rhf.y));
          const __half2 il = __float22half2_rn(make_float2(im.x - ihf.x, im.y - ihf.y));
          __half* of = o + (int64_t)(4 * f) * plane;
          if (in1) {
            *reinterpret_cast<__half2*>(of + PL_RE_HI * plane) = rh;
            *reinterpret_cast<__half2*>(of + PL_RE_LO * plane) = rl;
            *reinterpret_cast<__half2*>(of + PL_IM_HI * plane) = ih;
            *reinterpret_cast<__half2*>(of + PL_IM_LO * plane) = il;
          } else {
            of[PL_RE_HI * plane] = __low2half(rh);
            of[PL_RE_LO * plane] = __low2half(rl);
            of[PL_IM_HI * plane] = __low2half(ih);
            of[PL_IM_LO * plane] = __low2half(il);
          }
        }
      }
    }
    __syncthreads();                                            // tiles consumed before the next loads
  }
}

// ------------------------------------------------------------------------------ four-step K3
// Inverse (Alg. 1 step 2b + 3, L177-179) for the same long tubes, f = f1 + N1 f2, k = N2 k1 + k2:
//   pass 1:  U[f1, k2] = w_N^{-f1 k2} sum_{f2} Z[f1 + N1 f2] w_{N2}^{-f2 k2}     (stored at row f1 + N1 k2)
//   pass 2:  z[N2 k1 + k2] = (1/N) sum_{f1} U[f1, k2] w_{N1}^{-f1 k1}
// with Z_f = X_f + i Y_f of two real tubes and the conjugate fill Z_f = conj X_{N-f} + i conj Y_{N-f}
// for f > N/2 (Im of DC / Nyquist dropped).  Pass 1 reads C-bar through a 5-D view
// {p, q, re|im, f1, f2} (row 2f + re|im, f = f1 + N1 f2, f2 <= N2/2) and handles column f1 together
// with its mirror N1 - f1, whose rows hold X_{N-f}.
template <int N2, int TUB>
__global__ void __launch_bounds__(2 * TUB) inv4_pass1_kernel(const __grid_constant__ CUtensorMap mC5,
                                                            const __grid_constant__ CUtensorMap mW4, int64_t P,
                                                            int64_t Q, int N1, const float2* __restrict__ st2,
                                                            const float2* __restrict__ twN) {
  constexpr int F = TUB / 2, NT = 2 * TUB;
  constexpr int RB = N2 / 2 + 1;                              // f2 rows per column tile
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full;
  float* ca = smem;                                           // [f2][re|im][TUB] of column f1
  float* cb = ca + RB * 2 * TUB;                              // ... of column N1 - f1
  float2* za = reinterpret_cast<float2*>(cb + RB * 2 * TUB);  // Z / U of column f1: [f2|k2][c]
  float2* zb = za + N2 * F;                                   // ... of column N1 - f1
  const int N = N1 * N2;
  if (threadIdx.x == 0) {
    bar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int hc = N1 / 2;
  const int64_t items = pblocks * Q * (hc + 1);
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1) {
    const int f1 = (int)(it % (hc + 1));
    const int64_t r = it / (hc + 1);
    const int64_t q = r / pblocks, p0 = (r - q * pblocks) * TUB;
    const int f1b = (N1 - f1) % N1;
    const bool two = f1b != f1;
    if (threadIdx.x == 0) {
      bulk_wait_read();                                       // previous item's stores have read za/zb
      fence_async_smem();
      bar_expect(&full, (two ? 2 : 1) * RB * 2 * TUB * 4);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
          ::"r"(su32(ca)), "l"(&mC5), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(0), "r"(f1), "r"(0)
          : "memory");
      if (two)
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            ::"r"(su32(cb)), "l"(&mC5), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(0), "r"(f1b), "r"(0)
            : "memory");
    }
    bar_wait(&full, ph);
    // Z of column fc (t = 0: f1, t = 1: f1b), f = fc + N1 f2: own rows for f <= N/2, the other
    // column's mirrored rows otherwise
    for (int t = 0; t < (two ? 2 : 1); ++t) {
      const int fc = t == 0 ? f1 : f1b;
      const float* own = t == 0 ? ca : cb;
      const float* oth = two ? (t == 0 ? cb : ca) : ca;
      float2* z = t == 0 ? za : zb;
      for (int idx = threadIdx.x; idx < N2 * F; idx += NT) {
        const int f2 = idx / F, c = idx % F;
        const int f = fc + N1 * f2;
        float2 v;
        if (2 * f <= N) {
          const bool self = (f == 0 || 2 * f == N);
          const float2 re = reinterpret_cast<const float2*>(own + (f2 * 2) * TUB)[c];
          const float2 im = self ? make_float2(0.f, 0.f) : reinterpret_cast<const float2*>(own + (f2 * 2 + 1) * TUB)[c];
          v = make_float2(re.x - im.y, im.x + re.y);            // X_f + i Y_f
        } else {
          const int g2 = fc == 0 ? N2 - f2 : N2 - 1 - f2;        // row of g = N - f in column (N1 - fc) mod N1
          const float* src = fc == 0 ? own : oth;
          const float2 re = reinterpret_cast<const float2*>(src + (g2 * 2) * TUB)[c];
          const float2 im = reinterpret_cast<const float2*>(src + (g2 * 2 + 1) * TUB)[c];
          v = make_float2(re.x + im.y, re.y - im.x);            // conj X_g + i conj Y_g
        }
        z[idx] = v;
      }
    }
    __syncthreads();
    tube_fft<N2, +1, F, NT>(za, st2);                         // over f2 -> [k2][c]
    if (two) tube_fft<N2, +1, F, NT>(zb, st2);
    for (int t = 0; t < (two ? 2 : 1); ++t) {
      const int fc = t == 0 ? f1 : f1b;
      float2* z = t == 0 ? za : zb;
      for (int idx = threadIdx.x; idx < N2 * F; idx += NT) {
        const int k2 = idx / F;
        const float2 w = __ldg(twN + fc * k2);                // w_N^{-fc k2} = (cos, +sin)
        z[idx] = cmul(z[idx], w);
      }
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
                   ::"l"(&mW4), "r"(su32(za)), "r"((int)p0), "r"((int)q), "r"(f1), "r"(0)
                   : "memory");
      if (two)
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
                     ::"l"(&mW4), "r"(su32(zb)), "r"((int)p0), "r"((int)q), "r"(f1b), "r"(0)
                     : "memory");
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

template <int N1, int TUB>
__global__ void __launch_bounds__(2 * TUB) inv4_pass2_kernel(const __grid_constant__ CUtensorMap mW4,
                                                            const __grid_constant__ CUtensorMap mX4t, int64_t P,
                                                            int64_t Q, int N2, const float2* __restrict__ st1,
                                                            OutUnscale u) {
  constexpr int F = TUB / 2, NT = 2 * TUB;
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t full;
  float2* z = reinterpret_cast<float2*>(smem);                // [f1 -> k1][c]
  const float inv_n = 1.f / (float)(N1 * N2);
  if (threadIdx.x == 0) {
    bar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t items = pblocks * Q * N2;
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1) {
    const int k2 = (int)(it % N2);
    const int64_t r = it / N2;
    const int64_t q = r / pblocks, p0 = (r - q * pblocks) * TUB;
    if (threadIdx.x == 0) {
      bulk_wait_read();
      fence_async_smem();
      bar_expect(&full, TUB * N1 * 4);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
          ::"r"(su32(smem)), "l"(&mW4), "r"(su32(&full)), "r"((int)p0), "r"((int)q), "r"(0), "r"(k2)
          : "memory");
    }
    bar_wait(&full, ph);
    {
      // 1/N and the per-tube unscale (R18), folded into the last pass; NT % F == 0: fixed pair
      const int64_t p = p0 + 2 * (threadIdx.x % F);
      const float2 a = p < P ? out_scale(u.row, p, u.col, q, inv_n) : make_float2(0.f, 0.f);
      const float2 b = p + 1 < P ? out_scale(u.row, p + 1, u.col, q, inv_n) : make_float2(0.f, 0.f);
      tube_fft<N1, +1, F, NT, false, true>(z, st1, make_float2(1.f, 1.f), make_float2(a.x, b.x),
                                           make_float2(a.y, b.y));   // over f1 -> z[k1][c]
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      // rows k = k2 + N2 k1 of X through the view {p, q, k2, k1}
      asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
                   ::"l"(&mX4t), "r"(su32(smem)), "r"((int)p0), "r"((int)q), "r"(k2), "r"(0)
                   : "memory");
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------ tables / launch
using FwdFn = void (*)(CUtensorMap, int64_t, int64_t, const unsigned*, __half*, int64_t, float*);

// Measured (config 3, n3 = 31): the register kernels of transforms_dense.cu (direct warp-coalesced
// loads, ~14 warps/SM) already run K1 at ~5.5 TB/s and K3 faster than the TMA-staged variants, so
// the TMA path is instantiated only where it wins: the forward transform for 32 < n3 <= 64
// (config 5: 18.9 -> 13.9 ms).  TMIN..TMAX bound the instantiated range.
constexpr int TMIN = 33;

template <int N>
struct Tab {
  static void fill(FwdFn* f0, FwdFn* f1) {
    f0[N] = fwd_tma_kernel<N, 0>;
    f1[N] = fwd_tma_kernel<N, 1>;
    Tab<N - 1>::fill(f0, f1);
  }
};
template <>
struct Tab<TMIN - 1> {
  static void fill(FwdFn*, FwdFn*) {}
};

struct Fns {
  FwdFn f0[TMAX + 1] = {}, f1[TMAX + 1] = {};
  Fns() { Tab<TMAX>::fill(f0, f1); }
};
const Fns& fns() {
  static Fns t;
  return t;
}

bool ensure_tw() {
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && (done >> dev) & 1) return true;
  std::vector<float2> tab(TMAX * (TMAX + 1) / 2);
  std::vector<double> cs;
  for (int N = 1; N <= TMAX; ++N) {
    cs.assign(2 * N, 0.0);
    host_twiddles(N, cs.data());
    for (int m = 0; m < N; ++m) tab[toff(N) + m] = make_float2((float)cs[2 * m], (float)cs[2 * m + 1]);
  }
  if (cudaMemcpyToSymbol(c_tw2, tab.data(), sizeof(float2) * tab.size()) != cudaSuccess) return false;
  if (dev < 64) done |= 1ull << dev;
  return true;
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
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

// fp32 3-D map {d0 (contiguous, pitch ld0), d1, d2 (pitch ld0*d1)}, box {TP, 1, b2}
bool map_f32(CUtensorMap* m, const void* base, uint64_t d0, uint64_t ld0, uint64_t d1, uint64_t d2,
             uint32_t b2, uint32_t b0 = TP) {
  auto fn = encode();
  if (!fn || (ld0 * 4) % 16 != 0 || ((uintptr_t)base & 15) != 0 || b2 > 256) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld0 * 4, ld0 * d1 * 4};
  cuuint32_t box[3] = {b0, 1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp16 3-D map {d0 (contiguous, pitch ld0), d1, d2 (pitch ld0*d1)}, box {b0, 1, b2} (TMA stores)
bool map_f16_out(CUtensorMap* m, void* base, uint64_t d0, uint64_t ld0, uint64_t d1, uint64_t d2, uint32_t b0,
                 uint32_t b2) {
  auto fn = encode();
  if (!fn || (ld0 * 2) % 16 != 0 || ((uintptr_t)base & 15) != 0 || b0 > 256 || b2 > 256) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld0 * 2, ld0 * d1 * 2};
  cuuint32_t box[3] = {b0, 1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int grid_for(int64_t items, size_t smem_bytes, int threads, int num_sms) {
  int per_sm = (int)((220 * 1024) / (smem_bytes + 1024));
  const int per_sm_thr = 2048 / threads;
  if (per_sm > per_sm_thr) per_sm = per_sm_thr;
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  int64_t g = (int64_t)num_sms * per_sm;
  return (int)(items < g ? items : g);
}

int threads_of(int64_t n3) { return TP / (n3 <= 32 ? 2 : 1); }


// Persistent grid: the CTAs that are co-resident on an SM (registers, smem, threads), times the SMs.
int grid_occ(const void* fn, int64_t items, size_t smem, int num_sms) {
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TUBE_NT, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int64_t g = (int64_t)num_sms * per_sm;
  return (int)(items < g ? items : g);
}

// Tube-parallel Stockham transforms (power-of-two 32 <= n3 <= 256); false = not handled.
template <int N>
bool launch_fwd_tube_n(const float* X, int64_t P, int64_t Q, int role, const unsigned* maxbits, const float2* st,
                       __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  using C = TubeCfg<N>;
  CUtensorMap m;
  if (!map_f32(&m, X, (uint64_t)P, (uint64_t)P, (uint64_t)Q, (uint64_t)N, (uint32_t)N, (uint32_t)C::TUB))
    return false;
  constexpr int H = N / 2 + 1;
  CUtensorMap mo;   // split planes [f][4][q][ld] as {P (pitch ld), Q, 4h}, fp16, box {TUB, 1, <=256}
  if (!map_f16_out(&mo, out, (uint64_t)P, (uint64_t)ld, (uint64_t)Q, (uint64_t)(4 * H), (uint32_t)C::TUB,
                   (uint32_t)store_rows(4 * H)))
    return false;
  const void* fn = role == 0 ? (const void*)fwd_tube_kernel<N, 0> : (const void*)fwd_tube_kernel<N, 1>;
  const size_t smem = 2 * sizeof(float) * C::TUB * (size_t)N + sizeof(__half) * 4 * H * C::TUB;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  const int64_t items = (P + C::TUB - 1) / C::TUB * Q;
  const int grid = grid_occ(fn, items, smem, num_sms);
  void* args[] = {(void*)&m, (void*)&mo, (void*)&P, (void*)&Q, (void*)&maxbits, (void*)&st, (void*)&unscale};
  return cudaLaunchKernel(fn, dim3(grid), dim3(TUBE_NT), args, smem, s) == cudaSuccess;
}

template <int N>
bool launch_inv_tube_n(const float* Cre, int64_t ld, int64_t P, int64_t Q, const float2* st, OutUnscale u, float* X,
                       int num_sms, cudaStream_t s, OverlapK3* ov) {
  using C = TubeCfg<N>;
  constexpr int H = N / 2 + 1;
  CUtensorMap m, mo;
  if (!map_f32(&m, Cre, (uint64_t)P, (uint64_t)ld, (uint64_t)Q, (uint64_t)(2 * H), (uint32_t)(2 * H),
               (uint32_t)C::TUB) ||
      !map_f32(&mo, X, (uint64_t)P, (uint64_t)P, (uint64_t)Q, (uint64_t)N, (uint32_t)N, (uint32_t)C::TUB))
    return false;
  const void* fn = (const void*)inv_tube_kernel<N>;
  const size_t smem = 2 * sizeof(float) * C::TUB * 2 * H + sizeof(float2) * (size_t)C::F * N;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  const int64_t items = (P + C::TUB - 1) / C::TUB * Q;
  const int grid = grid_occ(fn, items, smem, num_sms);
  TubeOv to = {nullptr, nullptr, 0, 1, 1};
  void* args[] = {(void*)&m, (void*)&mo, (void*)&P, (void*)&Q, (void*)&st, (void*)&u, (void*)&to};
  if (ov && ov->done && ov->stream && ov->work && ov->cols_per_n == 128 && (256 * ov->pb_per_m) % C::TUB == 0) {
    // programmatic dependent of the GEMM just launched on `s` (internal.h OverlapK3): its CTAs start
    // once every GEMM CTA is resident, on the SMs the GEMM's cluster grid leaves free
    to = {ov->done, ov->work, ov->target, 256 * ov->pb_per_m / C::TUB, ov->nt};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TUBE_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    ov->used = true;
    return cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess;
  }
  return cudaLaunchKernel(fn, dim3(grid), dim3(TUBE_NT), args, smem, s) == cudaSuccess;
}


// 4-D fp32 view {P, Q, N1, N2} of a Matlab-layout P x Q x (N1 N2) tensor (row k1 + N1 k2), box
// {TUB, 1, b2, b3}
// (Qs = the tensor's full lateral size for the strides, Q = the lateral slices of this view)
bool map_f32_4d(CUtensorMap* m, const void* base, uint64_t P, uint64_t Q, uint64_t N1, uint64_t N2, uint32_t tub,
                uint32_t b2, uint32_t b3, uint64_t Qs = 0) {
  auto fn = encode();
  if (!Qs) Qs = Q;
  if (!fn || (P * 4) % 16 != 0 || ((uintptr_t)base & 15) != 0) return false;
  cuuint64_t dims[4] = {P, Q, N1, N2};
  cuuint64_t strides[3] = {P * 4, P * Qs * 4, P * Qs * N1 * 4};
  cuuint32_t box[4] = {tub, 1, b2, b3};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Lateral-slice chunks of a four-step transform (measurement knob): with TPROD_4STEP_L2_MB = m > 0
// the passes run chunk by chunk so that a chunk's intermediate (4 P Qc n3 bytes <= m MB) could stay
// in L2 until pass 2 reads it.  Measured on config 4 (K1 + K3): one chunk 0.203 ms, 40 MB chunks
// 0.240 ms, 24 MB chunks 0.275 ms -- the smaller grids per launch cost more than the DRAM re-read of
// the intermediate saves -- so the default is one chunk.
int64_t fourstep_chunk(int64_t P, int64_t Q, int64_t n3) {
  static const int64_t budget = [] {
    const char* e = getenv("TPROD_4STEP_L2_MB");
    return (int64_t)(e ? atoi(e) : 0) << 20;
  }();
  if (budget <= 0) return Q;
  const int64_t per_q = 4 * P * n3;
  const int64_t qmax = std::max<int64_t>(1, budget / per_q);
  const int64_t nch = (Q + qmax - 1) / qmax;
  return (Q + nch - 1) / nch;
}

template <int N1, int N2, int TUB>
bool launch_fwd4_t(const float* X, int64_t P, int64_t Q, int role, const unsigned* maxbits, const Twiddles32& tw,
                   __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  const void* k1 = (const void*)fwd4_pass1_kernel<N2, TUB>;
  const void* k2 = role == 0 ? (const void*)fwd4_pass2_kernel<N1, TUB, 0> : (const void*)fwd4_pass2_kernel<N1, TUB, 1>;
  const size_t sm1 = sizeof(float) * TUB * N2, sm2 = 2 * sizeof(float) * TUB * N1;
  if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1) != cudaSuccess ||
      cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2) != cudaSuccess)
    return false;
  const int64_t pblocks = (P + TUB - 1) / TUB;
  int per1 = 1, per2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k1, 2 * TUB, sm1);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k2, 2 * TUB, sm2);
  const int64_t Qc = fourstep_chunk(P, Q, (int64_t)N1 * N2);
  const int64_t plane = Q * ld;
  for (int64_t q0 = 0; q0 < Q; q0 += Qc) {
    int64_t Qi = std::min(Qc, Q - q0);
    CUtensorMap mx, mw1, mw2;
    if (!map_f32_4d(&mx, X + P * q0, P, Qi, N1, N2, TUB, 1, N2, Q) ||
        !map_f32_4d(&mw1, tw.scratch, P, Qi, N1, N2, TUB, 1, N2) || !map_f32_4d(&mw2, tw.scratch, P, Qi, N1, N2, TUB, N1, 1))
      return false;
    const int64_t it1 = pblocks * Qi * N1, it2 = pblocks * Qi * (N2 / 2 + 1);
    const int g1 = (int)std::min<int64_t>(it1, (int64_t)num_sms * std::max(per1, 1));
    const int g2 = (int)std::min<int64_t>(it2, (int64_t)num_sms * std::max(per2, 1));
    int n1i = N1, n2i = N2;
    const float2* st1 = tw.st_n1;
    const float2* st2 = tw.st_n2;
    const float2* twn = tw.tw;
    const unsigned* rowmax = role == 0 ? maxbits : nullptr;   // A: row scales applied in pass 1
    // B (role 1): the column maxima / unscale factors of this chunk's lateral slices
    const unsigned* mb = role == 0 ? maxbits : maxbits + q0;
    float* us = role == 0 ? unscale : unscale + q0;
    __half* o = out + q0 * ld;
    void* a1[] = {(void*)&mx, (void*)&mw1, (void*)&P, (void*)&Qi, (void*)&n1i, (void*)&st2, (void*)&twn, (void*)&rowmax};
    if (cudaLaunchKernel(k1, dim3(g1), dim3(2 * TUB), a1, sm1, s) != cudaSuccess) return false;
    void* a2[] = {(void*)&mw2, (void*)&P, (void*)&Qi, (void*)&n2i, (void*)&mb, (void*)&st1, (void*)&o, (void*)&ld,
                  (void*)&plane, (void*)&us};
    if (cudaLaunchKernel(k2, dim3(g2), dim3(2 * TUB), a2, sm2, s) != cudaSuccess) return false;
  }
  return true;
}

// 5-D fp32 view {P (pitch ld), Q, 2, N1, R2} of C-bar planes [f][re|im][q][ld] with f = f1 + N1 f2,
// box {tub, 1, 2, 1, R2}
bool map_cbar_5d(CUtensorMap* m, const void* base, uint64_t P, uint64_t ld, uint64_t Q, uint64_t N1, uint64_t R2,
                 uint32_t tub, uint64_t Qs = 0) {
  auto fn = encode();
  if (!Qs) Qs = Q;
  if (!fn || (ld * 4) % 16 != 0 || ((uintptr_t)base & 15) != 0) return false;
  cuuint64_t dims[5] = {P, Q, 2, N1, R2};
  cuuint64_t strides[4] = {ld * 4, ld * Qs * 4, 2 * ld * Qs * 4, 2 * N1 * ld * Qs * 4};
  cuuint32_t box[5] = {tub, 1, 2, 1, (cuuint32_t)R2};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N1, int N2, int TUB>
bool launch_inv4_t(const float* Cre, int64_t ld, int64_t P, int64_t Q, const Twiddles32& tw, OutUnscale u, float* X,
                   int num_sms, cudaStream_t s) {
  const void* k1 = (const void*)inv4_pass1_kernel<N2, TUB>;
  const void* k2 = (const void*)inv4_pass2_kernel<N1, TUB>;
  const size_t sm1 = sizeof(float) * (2 * (N2 / 2 + 1) * 2 * TUB + 2 * TUB * N2), sm2 = sizeof(float) * TUB * N1;
  if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1) != cudaSuccess ||
      cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2) != cudaSuccess)
    return false;
  const int64_t pblocks = (P + TUB - 1) / TUB;
  int per1 = 1, per2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k1, 2 * TUB, sm1);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k2, 2 * TUB, sm2);
  const int64_t Qc = fourstep_chunk(P, Q, (int64_t)N1 * N2);
  for (int64_t q0 = 0; q0 < Q; q0 += Qc) {
    int64_t Qi = std::min(Qc, Q - q0);
    CUtensorMap mc, mw1, mw2, mx;
    if (!map_cbar_5d(&mc, Cre + q0 * ld, P, ld, Qi, N1, N2 / 2 + 1, TUB, Q) ||
        !map_f32_4d(&mw1, tw.scratch, P, Qi, N1, N2, TUB, 1, N2) ||
        !map_f32_4d(&mw2, tw.scratch, P, Qi, N1, N2, TUB, N1, 1) ||
        !map_f32_4d(&mx, X + P * q0, P, Qi, N2, N1, TUB, 1, N1, Q))
      return false;
    const int64_t it1 = pblocks * Qi * (N1 / 2 + 1), it2 = pblocks * Qi * N2;
    const int g1 = (int)std::min<int64_t>(it1, (int64_t)num_sms * std::max(per1, 1));
    const int g2 = (int)std::min<int64_t>(it2, (int64_t)num_sms * std::max(per2, 1));
    int n1i = N1, n2i = N2;
    const float2* st1 = tw.st_n1;
    const float2* st2 = tw.st_n2;
    const float2* twn = tw.tw;
    OutUnscale uc{u.row, u.col ? u.col + q0 : nullptr};
    void* a1[] = {(void*)&mc, (void*)&mw1, (void*)&P, (void*)&Qi, (void*)&n1i, (void*)&st2, (void*)&twn};
    if (cudaLaunchKernel(k1, dim3(g1), dim3(2 * TUB), a1, sm1, s) != cudaSuccess) return false;
    void* a2[] = {(void*)&mw2, (void*)&mx, (void*)&P, (void*)&Qi, (void*)&n2i, (void*)&st1, (void*)&uc};
    if (cudaLaunchKernel(k2, dim3(g2), dim3(2 * TUB), a2, sm2, s) != cudaSuccess) return false;
  }
  return true;
}
}  // namespace

bool tube_supported(int64_t n3) { return n3 == 32 || n3 == 64 || n3 == 128 || n3 == 256; }

void fourstep_factors(int64_t n3, int* n1, int* n2) {
  *n1 = *n2 = 0;
  if (n3 == 4096) { *n1 = 64; *n2 = 64; }
  else if (n3 == 8192) { *n1 = 128; *n2 = 64; }
  else if (n3 == 16384) { *n1 = 128; *n2 = 128; }
}

bool launch_inv_4step(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const Twiddles32& tw,
                      OutUnscale u, float* X, int num_sms, cudaStream_t s) {
  int N1, N2;
  fourstep_factors(n3, &N1, &N2);
  if (!N1 || !tw.st_n1 || !tw.st_n2 || !tw.scratch || tw.scratch_bytes < (size_t)(4 * P * Q * n3) || P % 4 != 0 ||
      ((uintptr_t)X & 15) != 0 || ld % 4 != 0)
    return false;
  const bool wide = P >= 128;
  if (N1 == 64 && N2 == 64)
    return wide ? launch_inv4_t<64, 64, 128>(Cre, ld, P, Q, tw, u, X, num_sms, s)
                : launch_inv4_t<64, 64, 64>(Cre, ld, P, Q, tw, u, X, num_sms, s);
  if (N1 == 128 && N2 == 64)
    return wide ? launch_inv4_t<128, 64, 128>(Cre, ld, P, Q, tw, u, X, num_sms, s)
                : launch_inv4_t<128, 64, 64>(Cre, ld, P, Q, tw, u, X, num_sms, s);
  return wide ? launch_inv4_t<128, 128, 128>(Cre, ld, P, Q, tw, u, X, num_sms, s)
              : launch_inv4_t<128, 128, 64>(Cre, ld, P, Q, tw, u, X, num_sms, s);
}

bool launch_fwd_4step(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                      const Twiddles32& tw, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  int N1, N2;
  fourstep_factors(n3, &N1, &N2);
  if (!N1 || !tw.st_n1 || !tw.st_n2 || !tw.scratch || tw.scratch_bytes < (size_t)(4 * P * Q * n3) || P % 4 != 0 ||
      ((uintptr_t)X & 15) != 0 || ld % 2 != 0)
    return false;
  const bool wide = P >= 128;
  if (N1 == 64 && N2 == 64)
    return wide ? launch_fwd4_t<64, 64, 128>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s)
                : launch_fwd4_t<64, 64, 64>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s);
  if (N1 == 128 && N2 == 64)
    return wide ? launch_fwd4_t<128, 64, 128>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s)
                : launch_fwd4_t<128, 64, 64>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s);
  return wide ? launch_fwd4_t<128, 128, 128>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s)
              : launch_fwd4_t<128, 128, 64>(X, P, Q, role, maxbits, tw, out, ld, unscale, num_sms, s);
}

// Measured (B200, K1/K3 stage times): the tube kernels win the forward transform for n3 = 64
// (config 5: 10.1 -> 7.0 ms with the TMA-store epilogue), 128 and 256 (1.6-2.4x over the
// buffer-major FFT kernels), and with the TMA-store epilogue the inverse for 64 (config 5 K3
// 4.2 -> 3.7 ms) and 128 (0.27 -> 0.09 ms on 1024x512x128); the register kernels of
// transforms_dense.cu stay faster for n3 = 32.  (n3 = 256's C-bar tile has 2h = 258 > 256 rows, more
// than one TMA box; that inverse stays on the FFT kernel.)
static bool tube_fwd_pick(int64_t n3) { return n3 == 64 || n3 == 128 || n3 == 256; }
static bool tube_inv_pick(int64_t n3) { return n3 == 64 || n3 == 128; }

bool launch_fwd_tube(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                     const float2* st, __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  if (!st || !tube_fwd_pick(n3) || P % 4 != 0 || ((uintptr_t)X & 15) != 0 || ld % 2 != 0) return false;
  switch (n3) {
    case 32: return launch_fwd_tube_n<32>(X, P, Q, role, maxbits, st, out, ld, unscale, num_sms, s);
    case 64: return launch_fwd_tube_n<64>(X, P, Q, role, maxbits, st, out, ld, unscale, num_sms, s);
    case 128: return launch_fwd_tube_n<128>(X, P, Q, role, maxbits, st, out, ld, unscale, num_sms, s);
    default: return launch_fwd_tube_n<256>(X, P, Q, role, maxbits, st, out, ld, unscale, num_sms, s);
  }
}

bool inv_tube_stream_ok(int64_t P, int64_t n3, int64_t ld, const float* X) {
  return n3 == 64 && tube_inv_pick(n3) && P % 4 == 0 && ((uintptr_t)X & 15) == 0 && (ld * 4) % 16 == 0;
}

bool launch_inv_tube(const float* Cre, int64_t ld, int64_t P, int64_t Q, int64_t n3, const float2* st,
                     OutUnscale u, float* X, int num_sms, cudaStream_t s, OverlapK3* ov) {
  if (!st || !tube_inv_pick(n3) || P % 4 != 0 || ((uintptr_t)X & 15) != 0 || (ld * 4) % 16 != 0) return false;
  switch (n3) {
    case 32: return launch_inv_tube_n<32>(Cre, ld, P, Q, st, u, X, num_sms, s, ov);
    case 64: return launch_inv_tube_n<64>(Cre, ld, P, Q, st, u, X, num_sms, s, ov);
    case 128: return launch_inv_tube_n<128>(Cre, ld, P, Q, st, u, X, num_sms, s, ov);
    default: return launch_inv_tube_n<256>(Cre, ld, P, Q, st, u, X, num_sms, s, ov);
  }
}

bool launch_fwd_tma(const float* X, int64_t P, int64_t Q, int64_t n3, int role, const unsigned* maxbits,
                    __half* out, int64_t ld, float* unscale, int num_sms, cudaStream_t s) {
  // power-of-two n3 takes the register real-FFT kernels (transforms_dense.cu) instead
  if (n3 < TMIN || n3 > TMAX || (n3 & (n3 - 1)) == 0 || ld % 2 != 0 || !ensure_tw()) return false;
  CUtensorMap m;
  if (!map_f32(&m, X, (uint64_t)P, (uint64_t)P, (uint64_t)Q, (uint64_t)n3, (uint32_t)n3)) return false;
  FwdFn fn = role == 0 ? fns().f0[n3] : fns().f1[n3];
  const size_t smem = 2 * sizeof(float) * TP * (size_t)n3;
  if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return false;
  const int64_t items = (P + TP - 1) / TP * Q;
  const int thr = threads_of(n3);
  const int grid = grid_for(items, smem, thr, num_sms);
  void* args[] = {(void*)&m, (void*)&P, (void*)&Q, (void*)&maxbits, (void*)&out, (void*)&ld, (void*)&unscale};
  return cudaLaunchKernel((const void*)fn, dim3(grid), dim3(thr), args, smem, s) == cudaSuccess;
}

}  // namespace tprod
