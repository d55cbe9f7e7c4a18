// tcgen05 per-frequency complex GEMM -- placeholder until the tensor-core kernel lands.
#include "internal.h"

namespace tprod {
bool gemm_tc_supported() { return false; }
int launch_gemm_tc_split(const __half*, int64_t, const __half*, int64_t, float*, int64_t, int64_t,
                         int64_t, int64_t, int64_t, int64_t, const unsigned*, const unsigned*, int,
                         int, cudaStream_t) {
  return 6;
}
}  // namespace tprod
