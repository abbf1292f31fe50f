// Routing hooks for the tcgen05 kernels.  Until a tensor-core kernel covers a
// shape these return false and the caller uses its SIMT / cuBLAS path.
#include "common.cuh"

namespace evo {
struct AttnGeom;

bool gemm_tc_try(int64_t, int64_t, int64_t, const void*, int64_t, int, int64_t, const void*,
                 int64_t, int, int64_t, void*, int64_t, int64_t, int, float, float, int, int,
                 cudaStream_t) {
  return false;
}
bool attn_fwd_tc_try(const void*, const float*, const float*, const float*, void*, void*, void*,
                     float*, const AttnGeom&, int, cudaStream_t) {
  return false;
}
bool attn_bwd_tc_try(const void*, const float*, const float*, const void*, const void*,
                     const void*, const float*, void*, float*, float*, int, void*, size_t,
                     const AttnGeom&, int, cudaStream_t) {
  return false;
}
int64_t attn_bwd_tc_workspace(const AttnGeom&, int) { return 0; }
}  // namespace evo
