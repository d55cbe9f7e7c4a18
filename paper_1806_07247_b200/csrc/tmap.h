// Host-side TMA tensor-map encoding shared by the TMA kernels of libtprod.so.  The driver entry
// point cuTensorMapEncodeTiled is fetched once through the runtime (no -lcuda link).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace tprod {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
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

// 3-D map {d0 (contiguous, row pitch ld0 elements), d1, d2 (pitch ld0 * d1)} with box {b0, b1, b2},
// optional swizzle (default none), element size `es` bytes (4: fp32, 2: fp16).  false if TMA cannot describe it.
inline bool tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int es, const void* base, uint64_t d0, uint64_t ld0,
                    uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1, uint32_t b2,
                    CUtensorMapL2promotion l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  auto fn = tmap_encode_fn();
  if (!fn || (ld0 * es) % 16 != 0 || ((uintptr_t)base & 15) != 0 || b0 > 256 || b1 > 256 || b2 > 256) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld0 * es, ld0 * d1 * es};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t el[3] = {1, 1, 1};
  return fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, l2,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tprod
