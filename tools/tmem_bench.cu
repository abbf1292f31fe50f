// Microbenchmark: TMEM read / write throughput per SM (tcgen05.ld / st
// 32x32b, x16 / x32) with 4, 8 and 16 warps issuing, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2207_05477_b200/csrc \
//        tools/tmem_bench.cu -o ab/tmb && ab/tmb
#include <cstdio>
#include <cstdint>
#include "tc_common.cuh"

using namespace evo;

template <int X, bool STORE>
__global__ void bench(float* out, int iters, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tl = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * X) % 512;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (STORE) {
      float v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = acc + e;
      tc::tmem_st16u(tl, reinterpret_cast<const uint32_t(&)[16]>(v));
      if constexpr (X == 32) tc::tmem_st16u(tl + 16, reinterpret_cast<const uint32_t(&)[16]>(v));
      tc::wait_st();
      acc += 1.f;
    } else {
      if constexpr (X == 32) {
        float v[32];
        tc::tmem_ld32(tl, v);
        tc::wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += v[e];
      } else {
        float v[16];
        tc::tmem_ld16(tl, v);
        tc::wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) acc += v[e];
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(slot);
}

template <int X, bool STORE>
void run(int nw, float* out, long long* cyc) {
  const int iters = 2048;
  bench<X, STORE><<<148, nw * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double bytes = (double)nw * 32 * X * 4 * iters;
  printf("%s x%-2d warps %2d: %.1f B/clk per SM (%.1f cycles per warp-op)\n", STORE ? "st" : "ld", X, nw,
         bytes / avg, avg / iters);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  for (int nw : {1, 4, 8, 16}) {
    run<16, false>(nw, out, cyc);
    run<32, false>(nw, out, cyc);
    run<16, true>(nw, out, cyc);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
