// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, cta_group::1) as
// a function of N, operand major-ness and A source (smem / TMEM), for an
// accumulation chain of NMMA instructions issued back to back by one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2207_05477_b200/csrc \
//        tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include "tc_common.cuh"

using namespace evo;

template <int N, bool A_MN, bool TS, int CHAINS>
__global__ void bench(long long* out, int nmma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  // zero smem operands (values irrelevant)
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) tc::mbar_init(&bar, 1);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = slot;
  const uint32_t idesc = tc::idesc_bf16(128, N, A_MN, false);
  uint32_t phase = 0;
  long long best = 1LL << 60;
  for (int rep = 0; rep < 5; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (warp == 0) {
      const uint32_t a0 = tc::smem_u32(smem), b0 = tc::smem_u32(smem + 32768);
      for (int k = 0; k < nmma; ++k) {
        const int c = k % CHAINS;
        const uint64_t bd = tc::sdesc(b0 + (k % 8) * 256, 128, 2 * 128);
        if (TS) {
          tc::mma_bf16_ts_w(tbase + 256 + c * 64, tbase + (k % 8) * 8, bd, idesc, k >= CHAINS ? 1u : 0u);
        } else {
          const uint64_t ad = A_MN ? tc::sdesc(a0 + (k % 8) * 2 * 16 * 128, 16 * 128, 128)
                                   : tc::sdesc(a0 + (k % 8) * 256, 128, 16 * 128);
          tc::mma_bf16_ss_w(tbase + 256 + c * 64, ad, bd, idesc, k >= CHAINS ? 1u : 0u);
        }
      }
      tc::mma_commit_w(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  if (threadIdx.x == 0) out[0] = best;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

template <int N, bool A_MN, bool TS, int CHAINS>
void run(const char* name, long long* d, int nmma) {
  auto k = bench<N, A_MN, TS, CHAINS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(d, nmma);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%-34s nmma=%3d  total %6lld cyc  %6.1f cyc/mma  %s\n", name, nmma, h, (double)h / nmma,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int n : {1, 8, 24, 64}) {
    run<16, false, false, 1>("SS N=16 K-major 1 chain", d, n);
    run<16, false, false, 3>("SS N=16 K-major 3 chains", d, n);
    run<16, true, false, 3>("SS N=16 A MN-major 3 chains", d, n);
    run<16, false, true, 1>("TS N=16 (A in TMEM) 1 chain", d, n);
    run<32, false, false, 1>("SS N=32 K-major 1 chain", d, n);
    run<64, false, false, 1>("SS N=64 K-major 1 chain", d, n);
    run<256, false, false, 1>("SS N=256 K-major 1 chain", d, n);
  }
  return 0;
}
