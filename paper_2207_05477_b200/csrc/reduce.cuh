// Deterministic two-stage column reductions: kernels write per-block partial
// rows [G, ld] into a workspace; finalize_partials sums C of those columns in
// a fixed order (no atomics, bitwise reproducible run to run).
#pragma once
#include "common.cuh"

namespace evo {

void count_launch(int n);
unsigned partial_grid(int64_t rows);

// block per 32 columns; warp w sums partial rows g = w, w+8, ...; the 8 warp
// sums are then added in warp order.
static __global__ void __launch_bounds__(256) finalize_partials_kernel(
    const float* __restrict__ partials, int G, int64_t C, int64_t ld, float* __restrict__ out,
    int accumulate) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < C) {
#pragma unroll 4
    for (int g = w; g < G; g += 8) s += partials[(int64_t)g * ld + c];
  }
  sm[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < C) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    out[c] = accumulate ? out[c] + t : t;
  }
}

inline void finalize_partials(const float* partials, int G, int64_t C, float* out, int accumulate,
                              cudaStream_t s, int64_t ld = -1) {
  if (!out) return;
  if (ld < 0) ld = C;
  finalize_partials_kernel<<<cdiv(C, 32), 256, 0, s>>>(partials, G, C, ld, out, accumulate);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

}  // namespace evo
