// Deterministic two-stage column reductions: kernels write per-block partial
// rows [G, ld] into a workspace; finalize_partials sums C of those columns in
// block order (no atomics, bitwise reproducible).
#pragma once
#include "common.cuh"

namespace evo {

void count_launch(int n);
unsigned partial_grid(int64_t rows);

static __global__ void finalize_partials_kernel(const float* __restrict__ partials, int G,
                                                int64_t C, int64_t ld, float* __restrict__ out,
                                                int accumulate) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= C) return;
  float acc = 0.f;
  for (int g = 0; g < G; ++g) acc += partials[(int64_t)g * ld + c];
  out[c] = accumulate ? out[c] + acc : acc;
}

inline void finalize_partials(const float* partials, int G, int64_t C, float* out, int accumulate,
                              cudaStream_t s, int64_t ld = -1) {
  if (!out) return;
  if (ld < 0) ld = C;
  finalize_partials_kernel<<<cdiv(C, 256), 256, 0, s>>>(partials, G, C, ld, out, accumulate);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

}  // namespace evo
