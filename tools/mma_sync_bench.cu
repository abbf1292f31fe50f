// Microbenchmark: throughput of the warp-level mma.sync shapes on sm_100a
// (bf16 m16n8k16, tf32 m16n8k8), NW warps per block, 4 independent
// accumulator chains per warp, one block per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mma_sync_bench.cu -o /tmp/msb && /tmp/msb
#include <cstdio>
#include <cstdint>

template <int KIND>
__global__ void bench(float* out, int iters) {
  float d[4][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (KIND == 0)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0.f;
  for (int c = 0; c < 4; ++c)
    for (int e = 0; e < 4; ++e) s += d[c][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int nw : {4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) bench<0><<<148, nw * 32>>>(out, iters);
        else bench<1><<<148, nw * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 1) {
          const double mmas = 148.0 * nw * iters * 4;
          const double flop = mmas * (kind == 0 ? 2.0 * 16 * 8 * 16 : 2.0 * 16 * 8 * 8);
          printf("%s warps/SM %2d: %.3f ms, %.1f warp-MMA per SM-us, %.1f TFLOP/s\n",
                 kind == 0 ? "bf16 m16n8k16" : "tf32 m16n8k8 ", nw, ms, mmas / 148 / (ms * 1e3),
                 flop / (ms * 1e-3) / 1e12);
        }
      }
    }
  return 0;
}
