// Shared helpers for the Evoformer sm_100a library (libevoformer_sm100.so).
//
// Conventions of the C ABI (include/evoformer_sm100.h):
//  * every entry point returns int (EVO_OK = 0) and records a thread-local
//    message retrievable with evo_last_error();
//  * the caller owns every buffer (PyTorch's caching allocator on the host
//    side); the library never allocates device memory on the hot path;
//  * all work is enqueued on the cudaStream_t passed in; no host sync.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/evoformer_sm100.h"

namespace evo {

constexpr int EVO_STREAM_SLOTS = 8;
int stream_slot(cudaStream_t s);  // api.cu

void set_error(const std::string& msg);

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define EVO_REQUIRE(cond, code, msg)                                   \
  do {                                                                 \
    if (!(cond)) throw ::evo::Error((code), std::string(msg));         \
  } while (0)

#define EVO_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw ::evo::Error(EVO_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define EVO_LAUNCH_CHECK() EVO_CUDA(cudaGetLastError())

// Wrap an entry point body: converts exceptions into status codes.
#define EVO_API_BEGIN try {
#define EVO_API_END                                   \
  return EVO_OK;                                      \
  }                                                   \
  catch (const ::evo::Error& e) {                     \
    ::evo::set_error(e.what());                       \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception& e) {                   \
    ::evo::set_error(e.what());                       \
    return EVO_ERR_INTERNAL;                          \
  }

// ---------------------------------------------------------------------------
// storage types: activations are fp32 (parity mode) or bf16 (perf mode);
// math is always fp32.

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int num_sms() {
  static thread_local int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// dispatch on the storage dtype code (EVO_F32 / EVO_BF16)
#define EVO_DISPATCH_T(dtype, T, ...)                                  \
  do {                                                                 \
    if ((dtype) == EVO_F32) {                                          \
      using T = float;                                                 \
      __VA_ARGS__;                                                     \
    } else if ((dtype) == EVO_BF16) {                                  \
      using T = __nv_bfloat16;                                         \
      __VA_ARGS__;                                                     \
    } else {                                                           \
      throw ::evo::Error(EVO_ERR_ARG, "unsupported dtype code");       \
    }                                                                  \
  } while (0)

}  // namespace evo
