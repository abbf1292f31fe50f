// Deterministic two-stage column reductions: kernels write per-block partial
// rows [G, ld] into a workspace; finalize_partials sums C of those columns in
// a fixed order (no atomics, bitwise reproducible run to run).
//
// Deferred mode (evo_defer_begin / evo_defer_end): the partial rows of every
// reduction issued in between are placed in a caller-provided arena and their
// finalisation is batched into ONE launch at evo_defer_end -- one module's or
// one block's ~40 small bias/LN-affine reductions cost one kernel instead of
// forty.  Partials that are not in the arena are finalised immediately.
#pragma once
#include <vector>

#include "common.cuh"

namespace evo {

void count_launch(int n);
unsigned partial_grid(int64_t rows);

struct FinDesc {
  const float* part;
  float* out;
  int64_t ld;
  int G;
  int C;
  int accumulate;
  int pad;
};

constexpr int FIN_BATCH = 96;
struct FinBatch {
  int n;
  int pad;
  FinDesc d[FIN_BATCH];
};

struct DeferState {
  bool on = false;
  char* arena = nullptr;
  size_t cap = 0, used = 0;
  std::vector<FinDesc> list;
};
DeferState& defer_state();

// workspace for `bytes` of partial rows: the arena in deferred mode, else ws
inline float* partial_buffer(void* ws, size_t bytes) {
  DeferState& d = defer_state();
  if (!d.on) return (float*)ws;
  const size_t a = (d.used + 255) / 256 * 256;
  EVO_REQUIRE(a + bytes <= d.cap, EVO_ERR_ARG, "deferred-reduction arena exhausted");
  d.used = a + bytes;
  return (float*)(d.arena + a);
}

// block per 32 columns; warp w sums partial rows g = w, w+8, ...; the 8 warp
// sums are then added in warp order.
static __device__ __forceinline__ void finalize_cols(const float* __restrict__ partials, int G,
                                                     int64_t C, int64_t ld, float* __restrict__ out,
                                                     int accumulate, int64_t cblk, float (*sm)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = cblk * 32 + lane;
  // eight independent accumulators (eight loads in flight per lane; the
  // partial blocks reach thousands of rows), combined in a fixed order
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < C) {
    int g = w;
    for (; g + 56 < G; g += 64) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += partials[(int64_t)(g + 8 * j) * ld + c];
    }
    for (int j = 0; g < G; g += 8, ++j) a[j] += partials[(int64_t)g * ld + c];
  }
  const float s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  sm[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < C) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    out[c] = accumulate ? out[c] + t : t;
  }
}

static __global__ void __launch_bounds__(256) finalize_partials_kernel(
    const float* __restrict__ partials, int G, int64_t C, int64_t ld, float* __restrict__ out,
    int accumulate) {
  __shared__ float sm[8][33];
  finalize_cols(partials, G, C, ld, out, accumulate, blockIdx.x, sm);
}

inline void finalize_partials(const float* partials, int G, int64_t C, float* out, int accumulate,
                              cudaStream_t s, int64_t ld = -1) {
  if (!out) return;
  if (ld < 0) ld = C;
  DeferState& d = defer_state();
  if (d.on && (const char*)partials >= d.arena && (const char*)partials < d.arena + d.cap) {
    d.list.push_back(FinDesc{partials, out, ld, G, (int)C, accumulate, 0});
    return;
  }
  finalize_partials_kernel<<<cdiv(C, 32), 256, 0, s>>>(partials, G, C, ld, out, accumulate);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

}  // namespace evo
