// Dynamic Axial Parallelism re-layouts (src/harness.py:262-293, src/model.py:331-398).
//
// Every DAP collective moves whole residue/sequence rows of a token-major
// activation.  torch.distributed's all_to_all_single / all_gather_into_tensor /
// reduce_scatter_tensor exchange contiguous dim-0 chunks, so each exchange is
// bracketed by one outer-axis swap:
//   dst[b, a, :] = src[a, b, :]      (src [A, B, E bytes], dst [B, A, E bytes])
// e.g. the MSA shard [s, R, C] = [s, d, r*C] -> [d, s, r*C] before the
// column-attention all-to-all, or the gathered bias [d, H, r*R] -> [H, d, r*R].
// HBM-bound: 16-B vector copies, consecutive threads write consecutive
// chunks of one destination row (and read consecutive chunks of one source row).
#include "common.cuh"
#include "reduce.cuh"

namespace evo {

template <typename V>
__global__ void __launch_bounds__(256) swap01_kernel(const V* __restrict__ src, V* __restrict__ dst,
                                                     int64_t A, int64_t B, int64_t EV) {
  const int64_t n = A * B * EV;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % EV, ba = e / EV;
    const int64_t a = ba % A, b = ba / A;  // destination row (b, a)
    dst[e] = src[(a * B + b) * EV + c];
  }
}

}  // namespace evo

using namespace evo;

extern "C" {

int evo_swap01(const void* src, void* dst, int64_t A, int64_t B, int64_t elem_bytes, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(A >= 0 && B >= 0 && elem_bytes >= 0, EVO_ERR_ARG, "swap01: negative extent");
  EVO_REQUIRE(src != dst || A * B * elem_bytes == 0, EVO_ERR_ARG, "swap01: src and dst must not alias");
  const int64_t bytes = A * B * elem_bytes;
  if (bytes == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)elem_bytes;
  auto grid = [&](int64_t n) { return (unsigned)imin64((n + 255) / 256, (int64_t)num_sms() * 8); };
  if ((al & 15) == 0) {
    const int64_t ev = elem_bytes / 16;
    swap01_kernel<uint4><<<grid(A * B * ev), 256, 0, s>>>((const uint4*)src, (uint4*)dst, A, B, ev);
  } else if ((al & 3) == 0) {
    const int64_t ev = elem_bytes / 4;
    swap01_kernel<uint32_t><<<grid(A * B * ev), 256, 0, s>>>((const uint32_t*)src, (uint32_t*)dst, A, B, ev);
  } else {
    swap01_kernel<uint8_t><<<grid(bytes), 256, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, A, B, elem_bytes);
  }
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

}  // extern "C"
