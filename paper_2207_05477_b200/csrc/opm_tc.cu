// Outer-product-mean backward, d(pair) -> d(num), as one tcgen05 GEMM with the
// re-layout and normalisation in its epilogue (src/model.py:372-378
// differentiated):
//
//   dnum[i*k + p, j*k + q] = rec[i, j] * sum_c d_act[(i, j), c] * w_out[p*k + q, c]
//
// The unfused sequence writes doutn = d_act . w_out^T ([R^2, k^2], 134 MB at
// the bench shape), reads it back to scale and permute it into dnum, and
// writes dnum: this kernel writes dnum once, straight from TMEM.
//
// Tile: 128 rows (i, j0 .. j0+127) x 256 columns (8 values of p x 32 q) with the
// whole K = c_z = 128 staged in shared memory (no-swizzle K-major core
// matrices), 8 MMAs of K = 16 issued by one warp, fp32 accumulator in TMEM.
// Epilogue: thread = row j, one 32-column TMEM load per p = the 32 q values of
// dnum row (i, p) at columns j*k .. j*k+31 -- 64 contiguous bytes per thread,
// 8 KB contiguous per warp-quarter, so the permuted store stays coalesced.
#include "common.cuh"
#include "reduce.cuh"
#include "tc_common.cuh"

namespace evo {
namespace {

using bf16 = __nv_bfloat16;
constexpr int OT_K = 128;             // c_z (the contraction)
constexpr int OT_M = 128, OT_N = 256;  // tile
constexpr int OT_DC = OT_K / 8;        // 16-byte k chunks per row
constexpr int OT_A = OT_M * OT_K * 2, OT_B = OT_N * OT_K * 2;
constexpr int OT_SMEM = OT_A + OT_B + 64;

__global__ void __launch_bounds__(256) opm_dnum_tc_kernel(const bf16* __restrict__ dact,
                                                          const bf16* __restrict__ wout,
                                                          const float* __restrict__ rec,
                                                          bf16* __restrict__ dnum, int64_t R, int k) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OT_A + OT_B);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * OT_M;  // d_act rows (i, j0 ..)
  const int n0 = blockIdx.y * OT_N;               // dnum columns (p, q) ..
  // stage A = d_act[m0 .. m0+127, 0 .. 127] and B = w_out[n0 .. n0+255, 0 .. 127]
  for (int e = tid; e < OT_M * OT_DC; e += 256) {
    const int r = e / OT_DC, c = e % OT_DC;
    tc::cp_async16(smem + ((r >> 3) * OT_DC + c) * 128 + (r & 7) * 16, dact + (m0 + r) * OT_K + c * 8);
  }
  for (int e = tid; e < OT_N * OT_DC; e += 256) {
    const int r = e / OT_DC, c = e % OT_DC;
    tc::cp_async16(smem + OT_A + ((r >> 3) * OT_DC + c) * 128 + (r & 7) * 16, wout + (int64_t)(n0 + r) * OT_K + c * 8);
  }
  tc::cp_async_commit();
  if (warp == 0) tc::tmem_alloc<256>(slot);
  if (tid == 0) tc::mbar_init(bar, 1);
  tc::cp_async_wait0();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;
  if (warp == 0) {
    const uint32_t idesc = tc::idesc_bf16(OT_M, OT_N, false, false);
    const uint32_t sa = tc::smem_u32(smem), sb = tc::smem_u32(smem + OT_A);
#pragma unroll
    for (int ks = 0; ks < OT_K / 16; ++ks)
      tc::mma_bf16_ss_w(tbase, tc::sdesc(sa + ks * 256, 128, OT_DC * 128), tc::sdesc(sb + ks * 256, 128, OT_DC * 128),
                        idesc, ks > 0 ? 1u : 0u);
    tc::mma_commit_w(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after();
  // epilogue: warp w reads TMEM lanes 32*(w&3) .. +31 (rows), columns half (w>>2)
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const int64_t t = m0 + row;                // d_act row = (i, j)
  const int64_t i = t / R, j = t % R;
  const float sc = rec[t];
  const int64_t Rk = R * k;
#pragma unroll 1
  for (int pc = 0; pc < OT_N / 2 / 32; ++pc) {  // 4 groups of 32 columns per thread
    const int col = half * (OT_N / 2) + pc * 32;
    float v[32];
    tc::tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + col, v);
    tc::wait_ld();
    const int p = (n0 + col) / k;  // k == 32: one p per 32 columns
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e] * sc, v[2 * e + 1] * sc);
    uint4* dst = reinterpret_cast<uint4*>(dnum + (i * k + p) * Rk + j * k);
#pragma unroll
    for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

}  // namespace

// d_act [NI*R, 128] bf16 (rows (i, j) of this shard), w_out [k*k, 128] bf16,
// rec [NI*R] -> dnum [NI*k, R*k] bf16.  false: shape not covered.
bool opm_dnum_tc(const void* dact, const void* wout, const float* rec, void* dnum, int64_t R, int64_t k,
                 int64_t NI, int64_t C, cudaStream_t s) {
  if (C != OT_K || k != 32 || (R % OT_M) != 0 || NI <= 0) return false;
  if (((uintptr_t)dact | (uintptr_t)wout | (uintptr_t)dnum) & 15) return false;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(opm_dnum_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OT_SMEM));
    attr = true;
  }
  dim3 grid((unsigned)(NI * R / OT_M), (unsigned)(k * k / OT_N));
  opm_dnum_tc_kernel<<<grid, 256, OT_SMEM, s>>>((const bf16*)dact, (const bf16*)wout, rec, (bf16*)dnum, R, (int)k);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

}  // namespace evo

extern "C" int evo_opm_dnum(const void* d_act, const void* w_out, const float* rec, void* dnum, int64_t R,
                            int64_t k, int64_t NI, int64_t C, int dtype, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(dtype == EVO_BF16, EVO_ERR_UNSUPPORTED, "opm_dnum: bf16 only");
  EVO_REQUIRE(evo::opm_dnum_tc(d_act, w_out, rec, dnum, R, k, NI, C, (cudaStream_t)stream), EVO_ERR_UNSUPPORTED,
              "opm_dnum: needs c_z = 128, k = 32, n_res a multiple of 128, 16-B aligned operands");
  EVO_API_END
}
