// SIMT per-frequency complex GEMMs (Algorithm 1 step 2, first branch, PAPER.md:L177;
// Eq. (10)):  C-bar_f = A-bar_f . B-bar_f  for f = 0..h-1.
//
//  * gemm_simt_split : fp32 path REFERENCE engine.  Reads the same split fp16 operand planes the
//                      tcgen05 engine reads, decodes hi+lo to fp32 and accumulates in fp32.  It
//                      exists to cross-check the tensor-core kernel on identical inputs
//                      (TPROD_OPT_ENGINE = 1); the production fp32 path uses gemm_tc.cu.
//  * gemm_simt_f64   : the fp64 path's GEMM (tcgen05 has no f64 kind; DFMA on CUDA cores).
//
// Operand layouts (internal.h): A-bar planes [f][s][l][lda] (i fastest), B-bar planes
// [f][s][j][ldb] (l fastest), C-bar planes [f][re|im][j][ldc] (i fastest).
#include "internal.h"
#include "common.cuh"

namespace tprod {

constexpr int TS = 16;

__global__ void gemm_simt_split_kernel(const __half* __restrict__ Ab, int64_t lda,
                                       const __half* __restrict__ Bb, int64_t ldb,
                                       float* __restrict__ Cb, int64_t ldc, int n1, int n2, int n4) {
  __shared__ float sAr[TS][TS + 1], sAi[TS][TS + 1], sBr[TS][TS + 1], sBi[TS][TS + 1];
  const int f = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.x * TS + tx, j = blockIdx.y * TS + ty;
  const int64_t pa = (int64_t)n2 * lda, pb = (int64_t)n4 * ldb;
  const __half* A0 = Ab + (int64_t)(4 * f) * pa;
  const __half* B0 = Bb + (int64_t)(4 * f) * pb;
  float cr = 0.f, ci = 0.f;
  for (int l0 = 0; l0 < n2; l0 += TS) {
    {  // A tile: rows l = l0 + ty, cols i = blockIdx.x*TS + tx
      int l = l0 + ty, ii = blockIdx.x * TS + tx;
      float r = 0.f, im = 0.f;
      if (l < n2 && ii < n1) {
        int64_t o = (int64_t)l * lda + ii;
        r = __half2float(A0[PL_RE_HI * pa + o]) + __half2float(A0[PL_RE_LO * pa + o]);
        im = __half2float(A0[PL_IM_HI * pa + o]) + __half2float(A0[PL_IM_LO * pa + o]);
      }
      sAr[ty][tx] = r;
      sAi[ty][tx] = im;
    }
    {  // B tile: rows j = blockIdx.y*TS + ty, cols l = l0 + tx
      int l = l0 + tx, jj = blockIdx.y * TS + ty;
      float r = 0.f, im = 0.f;
      if (l < n2 && jj < n4) {
        int64_t o = (int64_t)jj * ldb + l;
        r = __half2float(B0[PL_RE_HI * pb + o]) + __half2float(B0[PL_RE_LO * pb + o]);
        im = __half2float(B0[PL_IM_HI * pb + o]) + __half2float(B0[PL_IM_LO * pb + o]);
      }
      sBr[ty][tx] = r;
      sBi[ty][tx] = im;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TS; ++kk) {
      float ar = sAr[kk][tx], ai = sAi[kk][tx], br = sBr[ty][kk], bi = sBi[ty][kk];
      cr = fmaf(ar, br, cr);
      cr = fmaf(-ai, bi, cr);
      ci = fmaf(ar, bi, ci);
      ci = fmaf(ai, br, ci);
    }
    __syncthreads();
  }
  if (i < n1 && j < n4) {
    int64_t o = (int64_t)j * ldc + i;
    int64_t pc = (int64_t)n4 * ldc;
    Cb[(int64_t)(2 * f) * pc + o] = cr;          // at the operands' scales (unscaled in K3, R18)
    Cb[(int64_t)(2 * f + 1) * pc + o] = ci;
  }
}

void launch_gemm_simt_split(const __half* Ab, int64_t lda, const __half* Bb, int64_t ldb, float* Cb,
                            int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h, cudaStream_t s) {
  dim3 grid((unsigned)((n1 + TS - 1) / TS), (unsigned)((n4 + TS - 1) / TS), (unsigned)h);
  gemm_simt_split_kernel<<<grid, dim3(TS, TS), 0, s>>>(Ab, lda, Bb, ldb, Cb, ldc, (int)n1, (int)n2,
                                                      (int)n4);
}

__global__ void gemm_simt_f64_kernel(const double* __restrict__ Ab, int64_t lda,
                                     const double* __restrict__ Bb, int64_t ldb,
                                     double* __restrict__ Cb, int64_t ldc, int n1, int n2, int n4) {
  __shared__ double sAr[TS][TS + 1], sAi[TS][TS + 1], sBr[TS][TS + 1], sBi[TS][TS + 1];
  const int f = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.x * TS + tx, j = blockIdx.y * TS + ty;
  const int64_t pa = (int64_t)n2 * lda, pb = (int64_t)n4 * ldb;
  const double* A0 = Ab + (int64_t)(2 * f) * pa;
  const double* B0 = Bb + (int64_t)(2 * f) * pb;
  double cr = 0.0, ci = 0.0;
  for (int l0 = 0; l0 < n2; l0 += TS) {
    {
      int l = l0 + ty, ii = blockIdx.x * TS + tx;
      bool ok = l < n2 && ii < n1;
      int64_t o = (int64_t)l * lda + ii;
      sAr[ty][tx] = ok ? A0[o] : 0.0;
      sAi[ty][tx] = ok ? A0[pa + o] : 0.0;
    }
    {
      int l = l0 + tx, jj = blockIdx.y * TS + ty;
      bool ok = l < n2 && jj < n4;
      int64_t o = (int64_t)jj * ldb + l;
      sBr[ty][tx] = ok ? B0[o] : 0.0;
      sBi[ty][tx] = ok ? B0[pb + o] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TS; ++kk) {
      double ar = sAr[kk][tx], ai = sAi[kk][tx], br = sBr[ty][kk], bi = sBi[ty][kk];
      cr = fma(ar, br, cr);
      cr = fma(-ai, bi, cr);
      ci = fma(ar, bi, ci);
      ci = fma(ai, br, ci);
    }
    __syncthreads();
  }
  if (i < n1 && j < n4) {
    int64_t o = (int64_t)j * ldc + i;
    int64_t pc = (int64_t)n4 * ldc;
    Cb[(int64_t)(2 * f) * pc + o] = cr;
    Cb[(int64_t)(2 * f + 1) * pc + o] = ci;
  }
}

// Register-tiled fp64 complex GEMM (the fp64 path's K2): a 64 x 64 output tile per CTA of 16 x 16
// threads, each thread 4 x 4 outputs (rows tx + 16 a, columns ty + 16 b: conflict-free shared
// reads), K blocks of 16 staged in shared memory (A as [l][i], B transposed to [l][j]), complex 4M
// with fp64 FMAs: 64 DFMA per 16 shared loads.  Same K order for every output (deterministic).
constexpr int T64 = 64, KB64 = 16;
__global__ void __launch_bounds__(256) gemm_f64_tiled_kernel(const double* __restrict__ Ab, int64_t lda,
                                                             const double* __restrict__ Bb, int64_t ldb,
                                                             double* __restrict__ Cb, int64_t ldc, int n1, int n2,
                                                             int n4) {
  __shared__ double sA[2][KB64][T64];
  __shared__ double sB[2][KB64][T64 + 1];
  const int f = blockIdx.z;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.x * T64, j0 = blockIdx.y * T64;
  const int64_t pa = (int64_t)n2 * lda, pb = (int64_t)n4 * ldb;
  const double* A0 = Ab + (int64_t)(2 * f) * pa;
  const double* B0 = Bb + (int64_t)(2 * f) * pb;
  double cr[4][4], ci[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) cr[a][b] = ci[a][b] = 0.0;
  for (int l0 = 0; l0 < n2; l0 += KB64) {
    // A tile: KB64 rows l x 64 columns i (coalesced along i); B tile: 64 rows j x KB64 l (coalesced
    // along l), stored transposed
#pragma unroll
    for (int r = 0; r < (KB64 * T64) / 256; ++r) {
      const int e = threadIdx.x + 256 * r;
      const int ii = e % T64, l = e / T64;
      const bool ok = l0 + l < n2 && i0 + ii < n1;
      const int64_t o = (int64_t)(l0 + l) * lda + i0 + ii;
      sA[0][l][ii] = ok ? A0[o] : 0.0;
      sA[1][l][ii] = ok ? A0[pa + o] : 0.0;
      const int ll = e % KB64, jj = e / KB64;
      const bool okb = l0 + ll < n2 && j0 + jj < n4;
      const int64_t ob = (int64_t)(j0 + jj) * ldb + l0 + ll;
      sB[0][ll][jj] = okb ? B0[ob] : 0.0;
      sB[1][ll][jj] = okb ? B0[pb + ob] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KB64; ++kk) {
      double ar[4], ai[4], br[4], bi[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ar[a] = sA[0][kk][tx + 16 * a];
        ai[a] = sA[1][kk][tx + 16 * a];
        br[a] = sB[0][kk][ty + 16 * a];
        bi[a] = sB[1][kk][ty + 16 * a];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          cr[a][b] = fma(ar[a], br[b], cr[a][b]);
          cr[a][b] = fma(-ai[a], bi[b], cr[a][b]);
          ci[a][b] = fma(ar[a], bi[b], ci[a][b]);
          ci[a][b] = fma(ai[a], br[b], ci[a][b]);
        }
    }
    __syncthreads();
  }
  const int64_t pc = (int64_t)n4 * ldc;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = j0 + ty + 16 * b;
    if (j >= n4) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = i0 + tx + 16 * a;
      if (i < n1) {
        const int64_t o = (int64_t)j * ldc + i;
        Cb[(int64_t)(2 * f) * pc + o] = cr[a][b];
        Cb[(int64_t)(2 * f + 1) * pc + o] = ci[a][b];
      }
    }
  }
}

void launch_gemm_simt_f64(const double* Ab, int64_t lda, const double* Bb, int64_t ldb, double* Cb,
                          int64_t ldc, int64_t n1, int64_t n2, int64_t n4, int64_t h, cudaStream_t s) {
  if (n1 * n4 >= 64 * 64) {                          // register-tiled kernel once a tile is mostly full
    dim3 g((unsigned)((n1 + T64 - 1) / T64), (unsigned)((n4 + T64 - 1) / T64), (unsigned)h);
    gemm_f64_tiled_kernel<<<g, 256, 0, s>>>(Ab, lda, Bb, ldb, Cb, ldc, (int)n1, (int)n2, (int)n4);
    return;
  }
  dim3 grid((unsigned)((n1 + TS - 1) / TS), (unsigned)((n4 + TS - 1) / TS), (unsigned)h);
  gemm_simt_f64_kernel<<<grid, dim3(TS, TS), 0, s>>>(Ab, lda, Bb, ldb, Cb, ldc, (int)n1, (int)n2,
                                                    (int)n4);
}

}  // namespace tprod
