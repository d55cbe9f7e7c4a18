// K2: per-frequency complex GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C-bar_f = A-bar_f . B-bar_f,  f = 0..h-1       (Algorithm 1 step 2, first branch, PAPER.md:L177;
//                                                   Eq. (10))
// Operands are the split fp16 planes written by K1 (internal.h):
//   A-bar_f ~ 2^-e_i (Arh + Arl + i(Aih + Ail)),  B-bar_f ~ 2^-e_j (Brh + Brl + i(Bih + Bil))
// and each real product X.Y is evaluated as Xh.Yh + Xh.Yl + Xl.Yh (the lo.lo term is below fp32
// rounding), with the complex product in the 4M form
//   Cr = Ar.Br - Ai.Bi,   Ci = Ar.Bi + Ai.Br        (-Ai via the instruction descriptor's negate-A bit)
// i.e. 12 tcgen05.mma.kind::f16 per K step, all accumulating in fp32 in TMEM (Cr in columns
// [0, BN), Ci in [BN, 2 BN)).  The epilogue stores the accumulators as they are -- C-bar at the
// operands' exact scales 2^(e_i + e_j), unscaled per output tube after the inverse transform
// (R18) -- as fp32 planes [f][re|im][j][i] coalesced along i.
//
// Kernel structure (one 128 x BN output tile of one frequency per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer -- per K block of BK=32: 8 boxes of A (4 planes x 2 M-halves,
//                     MN-major, 128B swizzle) + 4 boxes of B (4 planes, K-major, 64B swizzle)
//                     into a STAGES-deep ring guarded by full/empty mbarriers
//   warp 1 / lane 0 : MMA issuer -- waits full[s], issues 24 MMAs (M=128, N=BN, K=16), commits
//                     empty[s]; after the last K block commits tmem_full
//   all 4 warps     : epilogue -- tcgen05.ld 32x32b.x16 from TMEM lanes 32w..32w+31, scale, store
// Deterministic: fixed K order, no split-K, no atomics (C column j independent of n4).
#include "internal.h"
#include "common.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <cstdio>
#include <cstdlib>

namespace tprod {

namespace tc {

using namespace ptx;

constexpr int BM = 128;
constexpr int BK = 32;            // K elements per stage (two MMA K-steps; 64 B rows of B)
constexpr int B_ROW = BK * 2;     // bytes per K-major B row in smem
constexpr uint32_t B_SWZ = (BK == 32) ? 4u : 6u;   // smem-descriptor swizzle code: 64B / 32B
constexpr CUtensorMapSwizzle B_TMA_SWZ = (BK == 32) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;

// ---------------------------------------------------------------------------------- kernel
// Persistent warp-specialised kernel, 1 CTA per SM, (2 + 8) warps:
//   warp 0          TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1          MMA issuer (one lane) + TMEM allocator; accumulates K segment g of the
//                   current tile into TMEM buffer g&1 (Cr | Ci, 2*BN columns each buffer)
//   warps 2..9      epilogue: per segment, tcgen05.ld the buffer and add it into fp32 REGISTER
//                   accumulators (round-to-nearest), then release the buffer; after the last
//                   segment of a tile, scale by 2^-(e_i+e_j) and store.
// Promotion: tensor-core accumulation rounds the fp32 accumulator toward zero at every MMA, so
// the error of one TMEM accumulator grows linearly with the number of MMAs it absorbs (measured:
// 7e-6 at K=1024, 3e-5 at K=4096 without promotion).  Restarting the TMEM accumulator every
// SEG_KB K-blocks and summing the segments in fp32 registers keeps the error flat in K.
constexpr int SEG_KB = 128 / BK;           // K-blocks per promoted segment (K = 128)
constexpr int EPI_WARPS = 8;
constexpr int NTHREADS2 = 32 * (2 + EPI_WARPS);

template <int BN>
struct Cfg {
  static constexpr int A_PLANE = BK * BM * 2;                  // bytes: BK rows x 128 i x fp16
  static constexpr int B_PLANE = BN * BK * 2;                  // bytes: BN rows x BK l x fp16
  static constexpr int STAGE = NPLANES * (A_PLANE + B_PLANE);
  static constexpr int STAGES_FIT = (227 * 1024 - 2048) / STAGE;          // deepest ring that fits
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int BUF_COLS = 2 * BN;                      // Cr | Ci of one segment buffer
  static constexpr int TMEM_COLS = 2 * BUF_COLS;               // double-buffered
  static constexpr int COLS_PER_THREAD = BN / 2;               // each epilogue warp: half of N
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

struct TileInfo {
  int f, m0, n0;   // n0: index of this CTA's N tile (in tiles)
};

// Cluster tile ct -> (f, m, n-group); CTA `rank` of a CN-wide cluster takes N tile n-group*CN+rank.
// n fastest, then m, then f: concurrently running clusters share the A_f / B_f panels in L2.
__device__ __forceinline__ TileInfo tile_of(int64_t ct, int mt, int ntg, int CN, int rank) {
  TileInfo ti;
  ti.n0 = (int)(ct % ntg) * CN + rank;
  int64_t r = ct / ntg;
  ti.m0 = (int)(r % mt) * BM;
  ti.f = (int)(r / mt);
  return ti;
}

// CN = 1: independent CTAs.  CN = 2: a cluster of two CTAs along N computes two adjacent N
// tiles of the same (f, m); both need the same A tile, so each CTA TMA-loads one 64-row half of A
// and multicasts it to both (per-SM L2->smem traffic 64 KB -> 48 KB per K block), and each MMA
// commit arrives on the `empty` barriers of both CTAs (a slot is refilled only after both
// consumers are done with it).
template <int BN, int CN>
__global__ void __launch_bounds__(NTHREADS2, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   float* __restrict__ Cb, int64_t ldc, int n1, int n2, int n4, int h,
                   long long* __restrict__ dbg, int nyq) {
  using G = Cfg<BN>;
  const long long t_start = clock64();
  long long w0 = 0, w1 = 0;   // per-role wait cycles (diagnostics, dbg != nullptr)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + G::STAGES * G::STAGE);
  uint64_t* empty = full + G::STAGES;
  uint64_t* seg_full = empty + G::STAGES;     // [2]
  uint64_t* seg_empty = seg_full + 2;         // [2]
  uint32_t* tmem_slot = (uint32_t*)(seg_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (n2 + BK - 1) / BK;
  const int nseg = (nk + SEG_KB - 1) / SEG_KB;
  const int mt = (n1 + BM - 1) / BM, nt = (n4 + BN - 1) / BN;
  const int ntg = (nt + CN - 1) / CN;
  const int64_t nctiles = (int64_t)mt * ntg * h;
  const int rank = CN > 1 ? (int)cluster_ctarank() : 0;
  const int64_t cid = blockIdx.x / CN, ncl = gridDim.x / CN;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < G::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CN);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (CN > 1) cluster_sync();      // peers' barriers are initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {  // whole warp; single-thread instructions are elect.sync-predicated
      // ---------------------------------------------------------- TMA producer
      uint32_t it = 0;
      for (int64_t t = cid; t < nctiles; t += ncl) {
        const TileInfo ti = tile_of(t, mt, ntg, CN, rank);
        const int n0 = ti.n0 * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % G::STAGES;
          const uint32_t ph = (it / G::STAGES) & 1;
          { long long t0 = dbg ? clock64() : 0; mbar_wait(empty + s, ph ^ 1); if (dbg) w0 += clock64() - t0; }
          uint8_t* st = smem + s * G::STAGE;
          mbar_expect_tx(full + s, G::STAGE);
          const int k0 = kb * BK;
#pragma unroll
          for (int p = 0; p < NPLANES; ++p) {
            uint8_t* a = st + p * G::A_PLANE;
            if (CN == 1) {
              tma_load_3d(a, &tmA, full + s, ti.m0, k0, 4 * ti.f + p);
              tma_load_3d(a + BK * 128, &tmA, full + s, ti.m0 + 64, k0, 4 * ti.f + p);
            } else {
              tma_load_3d_mc(a + rank * BK * 128, &tmA, full + s, ti.m0 + 64 * rank, k0, 4 * ti.f + p,
                             (uint16_t)((1u << CN) - 1));
            }
            uint8_t* b = st + NPLANES * G::A_PLANE + p * G::B_PLANE;
            tma_load_3d(b, &tmB, full + s, k0, n0, 4 * ti.f + p);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp; single-thread instructions are elect.sync-predicated
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t ID_POS = idesc_f16(BM, BN, 0);
      constexpr uint32_t ID_NEG = idesc_f16(BM, BN, 1);
      uint32_t it = 0, g = 0;
      for (int64_t t = cid; t < nctiles; t += ncl) {
        // (the real DC / Nyquist shortcut of gemm_tc2_kernel is not taken here: measured 7% slower on
        // config 4, where this kernel runs)
        const bool real_f = false;
        for (int sg = 0; sg < nseg; ++sg, ++g) {
          const uint32_t b = g & 1, use = g >> 1;
          { long long t0 = dbg ? clock64() : 0; mbar_wait(seg_empty + b, (use & 1) ^ 1); if (dbg) w0 += clock64() - t0; }  // epilogue drained this buffer
          tc_fence_after();
          const uint32_t tCr = tmem + b * G::BUF_COLS, tCi = tCr + BN;
          const int kb_end = min(nk, (sg + 1) * SEG_KB);
          for (int kb = sg * SEG_KB; kb < kb_end; ++kb, ++it) {
            const int s = it % G::STAGES;
            const uint32_t ph = (it / G::STAGES) & 1;
            { long long t0 = dbg ? clock64() : 0; mbar_wait(full + s, ph); if (dbg) w1 += clock64() - t0; }
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * G::STAGE);
            const uint32_t bbase = base + NPLANES * G::A_PLANE;
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks) {
              uint64_t a[NPLANES], bd[NPLANES];
#pragma unroll
              for (int p = 0; p < NPLANES; ++p) {
                // A: MN-major, 128B swizzle; LBO = second 64-row half, SBO = 8 K-rows
                a[p] = sdesc(base + p * G::A_PLANE + ks * 2048, BK * 128, 1024, 2);
                // B: K-major, BK*2-byte rows swizzled; SBO = 8 rows
                bd[p] = sdesc(bbase + p * G::B_PLANE + ks * 32, 16, 8 * B_ROW, B_SWZ);
              }
              const uint32_t acc0 = (kb > sg * SEG_KB || ks > 0) ? 1u : 0u;
              // Cr = Ar.Br - Ai.Bi   (hi.hi + hi.lo + lo.hi each)
              mma_f16(tCr, a[PL_RE_HI], bd[PL_RE_HI], ID_POS, acc0);
              mma_f16(tCr, a[PL_RE_HI], bd[PL_RE_LO], ID_POS, 1);
              mma_f16(tCr, a[PL_RE_LO], bd[PL_RE_HI], ID_POS, 1);
              if (!real_f) {
                mma_f16(tCr, a[PL_IM_HI], bd[PL_IM_HI], ID_NEG, 1);
                mma_f16(tCr, a[PL_IM_HI], bd[PL_IM_LO], ID_NEG, 1);
                mma_f16(tCr, a[PL_IM_LO], bd[PL_IM_HI], ID_NEG, 1);
                // Ci = Ar.Bi + Ai.Br
                mma_f16(tCi, a[PL_RE_HI], bd[PL_IM_HI], ID_POS, acc0);
                mma_f16(tCi, a[PL_RE_HI], bd[PL_IM_LO], ID_POS, 1);
                mma_f16(tCi, a[PL_RE_LO], bd[PL_IM_HI], ID_POS, 1);
                mma_f16(tCi, a[PL_IM_HI], bd[PL_RE_HI], ID_POS, 1);
                mma_f16(tCi, a[PL_IM_HI], bd[PL_RE_LO], ID_POS, 1);
                mma_f16(tCi, a[PL_IM_LO], bd[PL_RE_HI], ID_POS, 1);
              }
            }
            // smem slot free once these MMAs have read it (in every CTA that wrote into it)
            if (CN == 1) mma_commit(empty + s);
            else mma_commit_mc(empty + s, (uint16_t)((1u << CN) - 1));
          }
          mma_commit(seg_full + b);      // segment accumulators complete
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    const int q = warp & 3;                      // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;            // which half of the N columns
    constexpr int CPT = G::COLS_PER_THREAD;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int64_t plane = (int64_t)n4 * ldc;
    uint32_t g = 0;
    for (int64_t t = cid; t < nctiles; t += ncl) {
      const TileInfo ti = tile_of(t, mt, ntg, CN, rank);
      const int n0 = ti.n0 * BN + half * CPT;
      const bool real_f = false;
      float accr[CPT], acci[CPT];
#pragma unroll
      for (int x = 0; x < CPT; ++x) accr[x] = acci[x] = 0.f;
      for (int sg = 0; sg < nseg; ++sg, ++g) {
        const uint32_t b = g & 1, use = g >> 1;
        { long long t0 = dbg ? clock64() : 0; mbar_wait(seg_full + b, use & 1); if (dbg) w0 += clock64() - t0; }
        tc_fence_after();
        const uint32_t base = tmem + lane_addr + b * G::BUF_COLS + half * CPT;
#pragma unroll
        for (int c = 0; c < CPT; c += 16) {
          uint32_t vr[16], vi[16];
          tmem_ld16_nowait(base + c, vr);
          tmem_ld16_nowait(base + BN + c, vi);     // (stale for real slices: selected away below)
          tmem_wait();
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            accr[c + x] += __uint_as_float(vr[x]);
            acci[c + x] += real_f ? 0.f : __uint_as_float(vi[x]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(seg_empty + b)) : "memory");
      }
      const long long ts0 = dbg ? clock64() : 0;
      const int i = ti.m0 + q * 32 + lane;
      if (i < n1) {
        float* Cr = Cb + (int64_t)(2 * ti.f) * plane + (int64_t)n0 * ldc + i;
        float* Ci = Cr + plane;
#pragma unroll
        for (int x = 0; x < CPT; ++x) {
          if (n0 + x < n4) {
            Cr[(int64_t)x * ldc] = accr[x];
            Ci[(int64_t)x * ldc] = acci[x];
          }
        }
      }
      if (dbg) w1 += clock64() - ts0;
    }
  }

  if (dbg && lane == 0 && warp <= 2) {
    // [0] total cycles  [1] producer: wait empty  [2] MMA: wait seg_empty  [3] MMA: wait full
    // [4] epilogue(warp 2): wait seg_full  [5] epilogue(warp 2): store phase  [6] CTAs
    if (warp == 0) { atomicAdd((unsigned long long*)dbg + 0, (unsigned long long)(clock64() - t_start));
                     atomicAdd((unsigned long long*)dbg + 1, (unsigned long long)w0);
                     atomicAdd((unsigned long long*)dbg + 6, 1ull); }
    if (warp == 1) { atomicAdd((unsigned long long*)dbg + 2, (unsigned long long)w0);
                     atomicAdd((unsigned long long*)dbg + 3, (unsigned long long)w1); }
    if (warp == 2) { atomicAdd((unsigned long long*)dbg + 4, (unsigned long long)w0);
                     atomicAdd((unsigned long long*)dbg + 5, (unsigned long long)w1); }
  }
  tc_fence_before();
  __syncthreads();
  if (CN > 1) cluster_sync();      // no CTA leaves while its peer may still signal its barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------- 2-SM kernel
// CTA pair (cta_group::2): one 256 x 128 output tile of one frequency per cluster of two CTAs on
// the two SMs of a TPC.  CTA r holds rows m0 + 128 r .. +127 of A (its own 128 TMEM lanes of the
// accumulators) and N rows n0 + 64 r .. +63 of B; the leader (r = 0) issues
// tcgen05.mma.cta_group::2 (M = 256, N = 128), which reads A and B from both CTAs' shared memory
// at the same offsets.  Per SM and per MMA that is 4 KB of A + 2 KB of B (96 B/clk at the MMA
// rate, against 128 B/clk for the single-CTA 128 x 128 tile), and 48 KB of TMA traffic per
// K block.  Barriers:
//   full[s]      leader's; armed by the leader with both CTAs' bytes, completed by both CTAs'
//                TMA loads (cta_group::2 TMA signals the leader's barrier)
//   empty[s]     both CTAs'; the leader's MMA commit arrives on both (multicast)
//   seg_full[b]  both CTAs'; multicast commit after the last MMA of a promoted segment
//   seg_empty[b] leader's; all 2 x 8 epilogue warps of the pair arrive (the peer's remotely)
// Same arithmetic, K order and epilogue as gemm_tc_kernel<128, *>: results are bitwise identical.
//
// CM = 2: clusters of 2 CM = 4 CTAs, two pairs stacked along M (cluster tile 512 x 128).  Both pairs
// need the same B tile, so CTA r of pair j loads only rows (64 / CM) j .. of its 64-row B half and
// multicasts them to CTA r of every pair: each B-bar panel is read from L2 / DRAM once per 512 A
// rows instead of once per 256 (the panels of a frequency do not fit the L2, so this halves the
// GEMM's DRAM traffic on config 5).  empty[s] then counts the commits of all CM pair leaders (a
// slot is refilled only after every pair's MMAs have read the multicast data in it).
template <int SEGKB, int CM>
__global__ void __launch_bounds__(NTHREADS2, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    float* __restrict__ Cb, int64_t ldc, int n1, int n2, int n4, int h, int nyq,
                    int* __restrict__ done, int ovord) {
  constexpr int BN = 128;
  constexpr int A_PLANE = BK * BM * 2;              // 128 rows of this CTA
  constexpr int B_PLANE = (BN / 2) * BK * 2;        // 64 N rows of this CTA
  constexpr int STAGE = NPLANES * (A_PLANE + B_PLANE);
  constexpr int STAGES = (227 * 1024 - 2048) / STAGE;
  constexpr int BUF_COLS = 2 * BN;
  constexpr int TMEM_COLS = 2 * BUF_COLS;
  constexpr int CPT = BN / 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* seg_full = empty + STAGES;     // [2]
  uint64_t* seg_empty = seg_full + 2;      // [2]
  uint32_t* tmem_slot = (uint32_t*)(seg_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1, pr = crank >> 1, lead = crank & ~1u;   // role in the pair, pair, its leader
  constexpr int BSUB = (BN / 2) / CM;               // B rows each CTA loads (and multicasts) per plane
  constexpr uint16_t ALL = (uint16_t)((1u << (2 * CM)) - 1);
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pr));
  uint16_t same_role = 0;                           // CTA `rank` of every pair
#pragma unroll
  for (int j = 0; j < CM; ++j) same_role |= (uint16_t)(1u << (2 * j + rank));
  const int nk = (n2 + BK - 1) / BK;
  const int nseg = (nk + SEGKB - 1) / SEGKB;
  const int mt = (n1 + 2 * CM * BM - 1) / (2 * CM * BM), nt = (n4 + BN - 1) / BN;
  const int64_t ntiles = (int64_t)mt * nt * h;
  const int64_t cid = blockIdx.x / (2 * CM), ncl = gridDim.x / (2 * CM);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CM);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 2 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                 // both CTAs' barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // K2 -> K3 overlap (internal.h OverlapK3): every CTA is resident now, so the dependent inverse may
  // launch; its blocks take the SMs this grid leaves idle and wait on `done` per output tile.
  if (done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Tile order: n fastest, then m, then f; concurrently running pairs share the A_f panel.
  // (Measured on config 5, DRAM read per launch: n fastest 149-165 GB, m fastest 185 GB, groups of
  // 6 m-tiles per n sweep 180 GB -- the pairs drift apart in K by up to a tile, longer than an L2
  // residency, so no raster order recovers the reuse; the plain order stays.)
  // With `done` (few tile rounds, K3 overlapped): the (m, n) output tiles must complete one after
  // another so that the inverse of the first ones runs during the last round -- f fastest
  // (ovord & 1 == 0) or, the default, m slowest, then f, n fastest.
  const int64_t tpf = (int64_t)mt * nt;
  // (ovord = 1: m slowest, then f, n fastest -- concurrent pairs still share the A_f panel and
  // the (m, n) tiles of an m row complete together.)
  int r = 0;                                       // (m, n) index of the last tile_of2 call
  auto tile_of2 = [&](int64_t t, int& f, int& m0, int& n0) {   // m0: this pair's first row
    if (done && (ovord & 1) == 0) {
      r = (int)(t / h);
      f = (int)(t - (int64_t)r * h);
    } else if (done) {
      const int64_t hn = (int64_t)h * nt;
      const int mm = (int)(t / hn), rem = (int)(t - mm * hn);
      f = rem / nt;
      r = mm * nt + (rem - f * nt);
    } else {
      f = (int)(t / tpf);
      r = (int)(t - (int64_t)f * tpf);
    }
    n0 = (r % nt) * BN;
    m0 = (r / nt) * (2 * CM * BM) + 2 * BM * (int)pr;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (both CTAs)
    const uint32_t full_cl = mapa_u32(smem_u32(full), lead);   // the pair leader's full[0]
    const uint32_t full_mc = smem_u32(full) & 0xFEFFFFFFu;       // multicast: each destination's pair leader
    uint32_t it = 0;
    for (int64_t t = cid; t < ntiles; t += ncl) {
      int f, m0, n0;
      tile_of2(t, f, m0, n0);
      // real DC / Nyquist slice: only the Re planes are loaded (the MMAs read nothing else)
      const bool real_f = f == 0 || (nyq && f == h - 1);
      const int np = real_f ? 2 : NPLANES;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(empty + s, ph ^ 1);
        uint8_t* st = smem + s * STAGE;
        if (rank == 0) mbar_expect_tx(full + s, 2 * (STAGE / NPLANES) * np);
        const uint32_t bar = full_cl + s * 8;
        const int k0 = kb * BK;
        const int mr = m0 + BM * (int)rank, nr = n0 + (BN / 2) * (int)rank + BSUB * (int)pr;
#pragma unroll
        for (int p = 0; p < NPLANES; ++p) {
          if (p >= np) break;
          uint8_t* a = st + p * A_PLANE;
          tma_load_3d_pair(a, &tmA, bar, mr, k0, 4 * f + p);
          tma_load_3d_pair(a + BK * 128, &tmA, bar, mr + 64, k0, 4 * f + p);
          uint8_t* bdst = st + NPLANES * A_PLANE + p * B_PLANE;
          if (CM == 1)
            tma_load_3d_pair(bdst, &tmB, bar, k0, nr, 4 * f + p);
          else
            tma_load_3d_pair_mc(bdst + BSUB * pr * B_ROW, &tmB, full_mc + s * 8, k0, nr, 4 * f + p, same_role);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // -------------------------------------------------------------- MMA issuer (pair leaders only)
      constexpr uint32_t ID_POS = idesc_f16(2 * BM, BN, 0);
      constexpr uint32_t ID_NEG = idesc_f16(2 * BM, BN, 1);
      uint32_t it = 0, g = 0;
      for (int64_t t = cid; t < ntiles; t += ncl) {
        int tf, tm, tn;
        tile_of2(t, tf, tm, tn);
        const bool real_f = tf == 0 || (nyq && tf == h - 1);     // DC / Nyquist: Ar.Br only
        for (int sg = 0; sg < nseg; ++sg, ++g) {
          const uint32_t b = g & 1, use = g >> 1;
          mbar_wait_cluster(seg_empty + b, (use & 1) ^ 1);    // both CTAs drained this buffer
          tc_fence_after();
          const uint32_t tCr = tmem + b * BUF_COLS, tCi = tCr + BN;
          const int kb_end = min(nk, (sg + 1) * SEGKB);
          for (int kb = sg * SEGKB; kb < kb_end; ++kb, ++it) {
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            mbar_wait_cluster(full + s, ph);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * STAGE);
            const uint32_t bbase = base + NPLANES * A_PLANE;
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks) {
              uint64_t a[NPLANES], bd[NPLANES];
#pragma unroll
              for (int p = 0; p < NPLANES; ++p) {
                a[p] = sdesc(base + p * A_PLANE + ks * 2048, BK * 128, 1024, 2);
                bd[p] = sdesc(bbase + p * B_PLANE + ks * 32, 16, 8 * B_ROW, B_SWZ);
              }
              const uint32_t acc0 = (kb > sg * SEGKB || ks > 0) ? 1u : 0u;
              mma2_f16(tCr, a[PL_RE_HI], bd[PL_RE_HI], ID_POS, acc0);
              mma2_f16(tCr, a[PL_RE_HI], bd[PL_RE_LO], ID_POS, 1);
              mma2_f16(tCr, a[PL_RE_LO], bd[PL_RE_HI], ID_POS, 1);
              if (!real_f) {
                mma2_f16(tCr, a[PL_IM_HI], bd[PL_IM_HI], ID_NEG, 1);
                mma2_f16(tCr, a[PL_IM_HI], bd[PL_IM_LO], ID_NEG, 1);
                mma2_f16(tCr, a[PL_IM_LO], bd[PL_IM_HI], ID_NEG, 1);
                // Ci = Ar.Bi + Ai.Br
                mma2_f16(tCi, a[PL_RE_HI], bd[PL_IM_HI], ID_POS, acc0);
                mma2_f16(tCi, a[PL_RE_HI], bd[PL_IM_LO], ID_POS, 1);
                mma2_f16(tCi, a[PL_RE_LO], bd[PL_IM_HI], ID_POS, 1);
                mma2_f16(tCi, a[PL_IM_HI], bd[PL_RE_HI], ID_POS, 1);
                mma2_f16(tCi, a[PL_IM_HI], bd[PL_RE_LO], ID_POS, 1);
                mma2_f16(tCi, a[PL_IM_LO], bd[PL_RE_HI], ID_POS, 1);
              }
            }
            mma2_commit_mc(empty + s, ALL);              // slot s read by this pair (every CTA counts CM)
          }
          mma2_commit_mc(seg_full + b, pair_mask);      // segment accumulators complete (both of the pair)
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int64_t plane = (int64_t)n4 * ldc;
    const uint32_t segE_cl = mapa_u32(smem_u32(seg_empty), lead);   // the pair leader's seg_empty[0]
    uint32_t g = 0;
    for (int64_t t = cid; t < ntiles; t += ncl) {
      int f, m0, n0t;
      tile_of2(t, f, m0, n0t);
      const int n0 = n0t + half * CPT;
      const bool real_f = f == 0 || (nyq && f == h - 1);
      float accr[CPT], acci[CPT];
#pragma unroll
      for (int x = 0; x < CPT; ++x) accr[x] = acci[x] = 0.f;
      for (int sg = 0; sg < nseg; ++sg, ++g) {
        const uint32_t b = g & 1, use = g >> 1;
        mbar_wait(seg_full + b, use & 1);
        tc_fence_after();
        const uint32_t base = tmem + lane_addr + b * BUF_COLS + half * CPT;
#pragma unroll
        for (int c = 0; c < CPT; c += 16) {
          uint32_t vr[16], vi[16];
          tmem_ld16_nowait(base + c, vr);
          tmem_ld16_nowait(base + BN + c, vi);     // (stale for real slices: selected away below)
          tmem_wait();
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            accr[c + x] += __uint_as_float(vr[x]);
            acci[c + x] += real_f ? 0.f : __uint_as_float(vi[x]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(segE_cl + b * 8)
                       : "memory");
      }
      const int i = m0 + BM * (int)rank + q * 32 + lane;
      if (i < n1) {
        float* Cr = Cb + (int64_t)(2 * f) * plane + (int64_t)n0 * ldc + i;
        float* Ci = Cr + plane;
#pragma unroll
        for (int x = 0; x < CPT; ++x) {
          if (n0 + x < n4) {
            Cr[(int64_t)x * ldc] = accr[x];
            Ci[(int64_t)x * ldc] = acci[x];
          }
        }
      }
      if (done && (ovord & 2)) {                   // the CTA's part of tile (m, n) at f is stored:
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");   // the 8 epilogue warps
        if (warp == 2 && lane == 0) {
          if (ovord & 4) {
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(done + r) : "memory");
          } else {
            __threadfence();
            atomicAdd(done + r, 1);
          }
        }
      } else if (done) {                           // this warp's part of tile (m, n) at f is stored
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(done + r, 1);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 3-D fp16 tensor map: dims {d0, d1, d2}, row pitch ld0 elements (d0 contiguous), plane pitch
// d1*ld0 elements; box {b0, b1, 1}.
bool make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld0,
              uint32_t b0, uint32_t b1, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld0 * 2, d1 * ld0 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int CN>
int launch_bn(const CUtensorMap& ma, const __half* Bb, int64_t ldb, float* Cb, int64_t ldc, int64_t n1,
              int64_t n2, int64_t n4, int64_t h, int nyq, int num_sms,
              cudaStream_t s) {
  using G = Cfg<BN>;
  CUtensorMap mb;
  if (!make_map(&mb, Bb, (uint64_t)n2, (uint64_t)n4, (uint64_t)(NPLANES * h), (uint64_t)ldb, BK, BN,
                B_TMA_SWZ))
    return 4;
  auto kern = gemm_tc_kernel<BN, CN>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) != cudaSuccess)
    return 4;
  const int64_t ntg = ((n4 + BN - 1) / BN + CN - 1) / CN;
  const int64_t nct = ((n1 + BM - 1) / BM) * ntg * h;       // cluster tiles
  const int64_t max_cl = num_sms / CN;
  const int grid = (int)((nct < max_cl ? nct : max_cl) * CN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS2);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CN;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int in1 = (int)n1, in2 = (int)n2, in4 = (int)n4, ih = (int)h;
  // Diagnostics (env TPROD_GEMM_DEBUG=1): per-role barrier-wait cycles, printed after a sync.
  static long long* dbg_buf = nullptr;
  static const bool want_dbg = getenv("TPROD_GEMM_DEBUG") != nullptr;
  long long* dbg = nullptr;
  if (want_dbg) {
    if (!dbg_buf) cudaMalloc(&dbg_buf, 8 * sizeof(long long));
    cudaMemsetAsync(dbg_buf, 0, 8 * sizeof(long long), s);
    dbg = dbg_buf;
  }
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, Cb, ldc, in1, in2, in4, ih, dbg, nyq) != cudaSuccess)
    return 4;
  if (dbg) {
    long long hv[8];
    cudaMemcpyAsync(hv, dbg, sizeof(hv), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double c = hv[6] ? (double)hv[6] : 1.0;
    fprintf(stderr, "[tprod gemm BN=%d CN=%d] per CTA (cycles): total %.0f | producer wait empty %.0f | "
            "mma wait seg_empty %.0f, wait full %.0f | epi wait seg_full %.0f, store %.0f\n", BN, CN,
            hv[0] / c, hv[1] / c, hv[2] / c, hv[3] / c, hv[4] / c, hv[5] / c);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

template <int SEGKB, int CM>
int launch_pair(const CUtensorMap& ma, const __half* Bb, int64_t ldb, float* Cb, int64_t ldc, int64_t n1,
                int64_t n2, int64_t n4, int64_t h, int nyq, int num_sms,
                cudaStream_t s, int* done, OverlapK3* ov) {
  constexpr int BN = 128;
  constexpr int STAGE = NPLANES * (BK * BM * 2 + (BN / 2) * BK * 2);
  constexpr int STAGES = (227 * 1024 - 2048) / STAGE;
  constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  CUtensorMap mb;
  if (!make_map(&mb, Bb, (uint64_t)n2, (uint64_t)n4, (uint64_t)(NPLANES * h), (uint64_t)ldb, BK, BN / 2 / CM,
                B_TMA_SWZ))
    return 4;
  auto kern = gemm_tc2_kernel<SEGKB, CM>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) return 4;
  if (CM > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  const int64_t nct = ((n1 + 2 * CM * BM - 1) / (2 * CM * BM)) * ((n4 + BN - 1) / BN) * h;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NTHREADS2);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * CM;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be co-resident (GPC sizes need not be multiples of 2 CM)
  int max_cl = num_sms / (2 * CM);
  {
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3((unsigned)(2 * CM * max_cl));
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, kern, &q) == cudaSuccess && nclu > 0) max_cl = std::min(max_cl, nclu);
    else cudaGetLastError();
  }
  const int grid = (int)((nct < max_cl ? nct : max_cl) * 2 * CM);
  cfg.gridDim = dim3((unsigned)grid);
  attr[0].val.clusterDim.x = 2 * CM;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int in1 = (int)n1, in2 = (int)n2, in4 = (int)n4, ih = (int)h;
  // K3 overlap only pays when the grid runs few tile rounds (the last one partial): the counters need
  // the row-by-row order, which on long runs re-reads panels the f-slowest order shares in L2
  const int64_t mtl = (n1 + 2 * CM * BM - 1) / (2 * CM * BM), ntl = (n4 + BN - 1) / BN;
  const int64_t rounds = (nct + max_cl - 1) / max_cl;
  // (a streaming K3 consumer -- OverlapK3::stream -- follows the row-by-row order over any number of
  // rounds: with m slowest, then f, n fastest, the concurrent clusters still share the A_f rows and
  // B_f is read once per m-row, as in the f-slowest order)
  if (!(done && ov && rounds >= 2 && (rounds <= 8 || ov->stream) && mtl * ntl <= OVERLAP_COUNTERS)) done = nullptr;
  if (done) {
    if (cudaMemsetAsync(done, 0, sizeof(int) * (mtl * ntl + 1), s) != cudaSuccess) return 4;
    ov->done = done;
    ov->work = done + mtl * ntl;                     // K3's item counter (streaming consumer)
    ov->target = (int)(h * 2 * CM * EPI_WARPS);
    ov->pb_per_m = CM;                               // 2 CM * 128 rows = CM blocks of 256 rows
    ov->cols_per_n = BN;
    ov->nt = (int)ntl;
  }
  // TPROD_OV_ORDER (measurement only) bits: 1 = (m, f, n) tile order instead of f fastest, 2 = one
  // counter arrive per CTA after a named barrier of the epilogue warps instead of one per warp, 4 =
  // red.release instead of fence + atomic.  Measured on config 3 (K2 + K3 stage, same box): 0: 164.9,
  // 2: 163.5, 6: 163.4, 3: 162.5 us (default); the GEMM alone (ncu) ~151.5 us with counters in every
  // variant vs 147.5 us without.
  static const int ovord = getenv("TPROD_OV_ORDER") ? atoi(getenv("TPROD_OV_ORDER")) : 3;
  if (done && (ovord & 2)) ov->target = (int)(h * 2 * CM);     // one arrival per CTA and frequency
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, Cb, ldc, in1, in2, in4, ih, nyq, done, ovord) != cudaSuccess) return 4;
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tc

bool gemm_tc_supported() { return tc::encode_fn() != nullptr; }

int launch_gemm_tc_split(const __half* Ab, int64_t lda, const __half* Bb, int64_t ldb, float* Cb,
                         int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h, int nyq, int force_bn, int force_cn,
                         int num_sms, cudaStream_t s, int* done, OverlapK3* ov) {
  CUtensorMap ma;
  if (!tc::make_map(&ma, Ab, (uint64_t)n1, (uint64_t)n2, (uint64_t)(NPLANES * h), (uint64_t)lda, 64,
                    tc::BK, CU_TENSOR_MAP_SWIZZLE_128B))
    return 4;
  int bn = force_bn;
  const int64_t mt = (n1 + tc::BM - 1) / tc::BM;
  if (bn == 0) {
    // N = 128 unless that leaves SMs idle (small problems) or n4 <= 64 fits one 64-wide tile
    // (a 128-wide tile would be half padding: config 4's 64 x 64 x 64 slices, 84 -> see DESIGN)
    bn = (n4 > 64 && mt * ((n4 + 127) / 128) * h >= num_sms) ? 128 : 64;
  }
  const int64_t nt = (n4 + bn - 1) / bn;
  int cn = force_cn;
  // cta_group::2 pairs: 256 x 128 tiles (enough of them to fill the SM pairs)
  const bool pair_ok = bn == 128 || force_bn == 0;
  // 4-CTA clusters (two pairs sharing B by multicast) when A has at least 1024 rows and the 512 x 128
  // cluster tiles still fill the GPU several times over (fewer, larger tiles would lengthen the tail)
  if (cn == 4 || (cn == 0 && force_bn == 0 && n1 >= 1024 &&
                  ((n1 + 511) / 512) * ((n4 + 127) / 128) * h >= 4 * (num_sms / 4))) {
    if (pair_ok) return tc::launch_pair<tc::SEG_KB, 2>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s, done, ov);
  }
  if (cn == 3 || (cn == 0 && force_bn == 0 && n1 > 128 &&
                  ((n1 + 255) / 256) * ((n4 + 127) / 128) * h >= num_sms / 2)) {
    if (pair_ok) return tc::launch_pair<tc::SEG_KB, 1>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s, done, ov);
  }
  if (cn == 0) cn = (nt >= 2 && mt * ((nt + 1) / 2) * h >= num_sms / 2) ? 2 : 1;   // share A tiles
  if (bn == 128)
    return cn == 2 ? tc::launch_bn<128, 2>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s)
                   : tc::launch_bn<128, 1>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s);
  return cn == 2 ? tc::launch_bn<64, 2>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s)
                 : tc::launch_bn<64, 1>(ma, Bb, ldb, Cb, ldc, n1, n2, n4, h, nyq, num_sms, s);
}

}  // namespace tprod
