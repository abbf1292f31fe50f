// 8-element vector access helpers for bandwidth-bound kernels: one 16-byte
// load/store for bf16, two for fp32.  Every "chunk" in the glue kernels is 8
// consecutive channels of one token row.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace evo {

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float (&f)[8]);
template <>
__device__ __forceinline__ void ld8<float>(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <>
__device__ __forceinline__ void ld8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

template <typename T>
__device__ __forceinline__ void st8(T* p, const float (&f)[8]);
template <>
__device__ __forceinline__ void st8<float>(float* p, const float (&f)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}
template <>
__device__ __forceinline__ void st8<__nv_bfloat16>(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// raw 8-element vectors: load now, convert later (keeps the registers of
// several in-flight loads at their storage width)
template <typename T>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  uint4 u;
};
template <>
struct Vec8<float> {
  float4 a, b;
};
__device__ __forceinline__ void ldv8(const __nv_bfloat16* p, Vec8<__nv_bfloat16>& v) {
  v.u = *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void ldv8(const float* p, Vec8<float>& v) {
  v.a = reinterpret_cast<const float4*>(p)[0];
  v.b = reinterpret_cast<const float4*>(p)[1];
}
__device__ __forceinline__ void cvt8(const Vec8<__nv_bfloat16>& v, float (&f)[8]) {
  const uint32_t w[4] = {v.u.x, v.u.y, v.u.z, v.u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __uint_as_float(w[k] << 16);
    f[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void cvt8(const Vec8<float>& v, float (&f)[8]) {
  f[0] = v.a.x; f[1] = v.a.y; f[2] = v.a.z; f[3] = v.a.w;
  f[4] = v.b.x; f[5] = v.b.y; f[6] = v.b.z; f[7] = v.b.w;
}

// 4-element variants (8-byte bf16 / 16-byte fp32 accesses)
template <typename T>
__device__ __forceinline__ void ld4(const T* p, float (&f)[4]);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&f)[4]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
}
template <>
__device__ __forceinline__ void ld4<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[4]) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xFFFF0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xFFFF0000u);
}
template <typename T>
__device__ __forceinline__ void st4(T* p, const float (&f)[4]);
template <>
__device__ __forceinline__ void st4<float>(float* p, const float (&f)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
}

// sum over the LANES consecutive lanes of a row group (LANES power of 2 <= 32)
template <int LANES>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace evo
