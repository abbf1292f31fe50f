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

// Persistent form: CTA (n, g) keeps the w_out rows of N-tile n resident and
// walks M-tiles g, g + G, ...; A tiles are double-buffered (cp.async two tiles
// ahead) and the accumulator is double-buffered in TMEM, so the MMAs of tile
// t+1 and the loads of t+2 run under the (store-bound) epilogue of tile t.
constexpr int OT_T = 512;  // 16 warps: 4 TMEM lane quarters x 4 column quarters in the epilogue
constexpr int OT_X = (OT_T / 32) * 32 * 64;  // per-warp 2 KB transpose buffers of the epilogue
constexpr int OT_SMEM_P = OT_B + 2 * OT_A + OT_X + 64;

__global__ void __launch_bounds__(OT_T, 1) opm_dnum_tc_kernel(const bf16* __restrict__ dact,
                                                             const bf16* __restrict__ wout,
                                                             const float* __restrict__ rec,
                                                             bf16* __restrict__ dnum, int64_t R, int k,
                                                             int64_t n_mt, int G) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sB = smem;
  uint8_t* sA = smem + OT_B;  // two buffers of OT_A
  uint8_t* sX = smem + OT_B + 2 * OT_A;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OT_B + 2 * OT_A + OT_X);  // [2]
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.y * OT_N;
  const int g = blockIdx.x;
  const int nt = (int)((n_mt - g + G - 1) / G);  // M-tiles of this CTA
  auto load_a = [&](int t, int buf) {
    const int64_t m0 = (int64_t)(g + (int64_t)t * G) * OT_M;
    uint8_t* d = sA + buf * OT_A;
    for (int e = tid; e < OT_M * OT_DC; e += OT_T) {
      const int r = e / OT_DC, c = e % OT_DC;
      tc::cp_async16(d + ((r >> 3) * OT_DC + c) * 128 + (r & 7) * 16, dact + (m0 + r) * OT_K + c * 8);
    }
  };
  for (int e = tid; e < OT_N * OT_DC; e += OT_T) {
    const int r = e / OT_DC, c = e % OT_DC;
    tc::cp_async16(sB + ((r >> 3) * OT_DC + c) * 128 + (r & 7) * 16, wout + (int64_t)(n0 + r) * OT_K + c * 8);
  }
  if (nt > 0) load_a(0, 0);
  if (nt > 1) load_a(1, 1);
  tc::cp_async_commit();
  if (warp == 0) tc::tmem_alloc<512>(slot);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
  }
  tc::cp_async_wait0();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;
  const uint32_t idesc = tc::idesc_bf16(OT_M, OT_N, false, false);
  const uint32_t sb = tc::smem_u32(sB);
  auto issue = [&](int t) {  // warp 0: MMAs of tile t into accumulator t & 1
    const uint32_t sa = tc::smem_u32(sA + (t & 1) * OT_A);
    const uint32_t acc = tbase + (uint32_t)((t & 1) * OT_N);
#pragma unroll
    for (int ks = 0; ks < OT_K / 16; ++ks)
      tc::mma_bf16_ss_w(acc, tc::sdesc(sa + ks * 256, 128, OT_DC * 128), tc::sdesc(sb + ks * 256, 128, OT_DC * 128),
                        idesc, ks > 0 ? 1u : 0u);
    tc::mma_commit_w(&bar[t & 1]);
  };
  if (warp == 0 && nt > 0) issue(0);
  const int quarter = warp & 3, cq = warp >> 2;  // TMEM lane quarter, column quarter
  const int row = quarter * 32 + lane;
  const int64_t Rk = R * k;
  for (int t = 0; t < nt; ++t) {
    if (warp == 0 && t + 1 < nt) issue(t + 1);  // A(t+1) resident, accumulator (t+1)&1 drained
    const int64_t tr = (int64_t)(g + (int64_t)t * G) * OT_M + row;  // d_act row = (i, j)
    const int64_t i = tr / R, j = tr % R;
    const float sc = __ldg(rec + tr);  // fetched while the MMAs run
    tc::mbar_wait(&bar[t & 1], (uint32_t)((t >> 1) & 1));
    tc::fence_after();
    if (t + 2 < nt) {  // MMA(t) is done with A buffer t & 1
      load_a(t + 2, t & 1);
      tc::cp_async_commit();
    }
#pragma unroll 1
    for (int pc = 0; pc < OT_N / 4 / 32; ++pc) {
      const int col = cq * (OT_N / 4) + pc * 32;
      float v[32];
      tc::tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((t & 1) * OT_N + col), v);
      tc::wait_ld();
      const int p = (n0 + col) / k;
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e] * sc, v[2 * e + 1] * sc);
      // the warp's 32 rows are 32 x 64 B = 2 KB contiguous in dnum row (i, p): go
      // through a per-warp shared buffer so each store instruction writes 512
      // contiguous bytes (chunk c = e*32 + lane <- row c/4, part c%4)
      uint4* xb = reinterpret_cast<uint4*>(sX + warp * 2048);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        xb[lane * 4 + (e ^ (lane & 3))] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(dnum + (i * k + p) * Rk + (j - lane) * k);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = e * 32 + lane, r = c >> 2, q = c & 3;
        dst[c] = xb[r * 4 + (q ^ (r & 3))];
      }
      __syncwarp();
    }
    tc::cp_async_wait0();  // A(t+2) landed: MMA(t+2) is issued at the top of the next iteration
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();  // A(t+2) visible to the tensor core; accumulator t & 1 drained
    tc::fence_after();
  }
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
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
    EVO_CUDA(cudaFuncSetAttribute(opm_dnum_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OT_SMEM_P));
    attr = true;
  }
  const int64_t n_mt = NI * R / OT_M;
  const int n_nt = (int)(k * k / OT_N);
  int G = num_sms() / n_nt;
  if (G < 1) G = 1;
  if (G > n_mt) G = (int)n_mt;
  dim3 grid((unsigned)G, (unsigned)n_nt);
  opm_dnum_tc_kernel<<<grid, OT_T, OT_SMEM_P, s>>>((const bf16*)dact, (const bf16*)wout, rec, (bf16*)dnum, R,
                                                  (int)k, n_mt, G);
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

// ---------------------------------------------------------------------------
// Forward: num = a^T c over this worker's sequences, written straight in the
// normalised [(i, j), p*k + q] layout the w_out projection reads
// (src/model.py:366-377):
//
//   outn[i*R + j, p*k + q] = rec[i*R + j] * sum_s a[s, i*k + p] * c[s, j*k + q]
//
// A = a^T and B = c are both MN-major in memory ([S, R*k] rows); K = S = 128 is
// staged whole.  Tile 128 rows (4 values of i x 32 p) x 256 columns (8 j x
// 32 q): TMEM lane quarter = one i, lane = p, and a 32-column slice = one j,
// so a warp's 32 lanes hold the 2 KB outn row (i, j); it goes out through the
// same per-warp shared-memory transpose as above (512 B per store).
namespace evo {
namespace {

constexpr int OF_K = 128;                        // sequences (contraction)
constexpr int OF_M = 128, OF_N = 256;
constexpr int OF_A = OF_M * OF_K * 2, OF_B = OF_N * OF_K * 2;
constexpr int OF_T = 512;
constexpr int OF_X = (OF_T / 32) * 2048;
constexpr int OF_SMEM = OF_B + 2 * OF_A + OF_X + 64;

// MN-major staging: element (kk, m) of a [K x E] tile (E contiguous in memory)
// -> core (kk/8, m/8) at ((kk/8)*(E/8) + m/8)*128 + (kk%8)*16 + (m%8)*2
template <int E>
__device__ __forceinline__ void stage_mn(uint8_t* dst, const bf16* src, int64_t ld, int tid) {
  constexpr int EC = E / 8;
  for (int e = tid; e < OF_K * EC; e += OF_T) {
    const int kk = e / EC, c = e % EC;
    tc::cp_async16(dst + ((kk >> 3) * EC + c) * 128 + (kk & 7) * 16, src + (int64_t)kk * ld + c * 8);
  }
}

__global__ void __launch_bounds__(OF_T, 1) opm_outn_tc_kernel(const bf16* __restrict__ a, const bf16* __restrict__ c,
                                                              const float* __restrict__ rec,
                                                              bf16* __restrict__ outn, int64_t R, int k,
                                                              int64_t n_mt, int G) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sB = smem;
  uint8_t* sA = smem + OF_B;
  uint8_t* sX = smem + OF_B + 2 * OF_A;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OF_B + 2 * OF_A + OF_X);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t Rk = R * k;
  const int64_t n0 = (int64_t)blockIdx.y * OF_N;  // c columns (j, q)
  const int g = blockIdx.x;
  const int nt = (int)((n_mt - g + G - 1) / G);
  auto load_a = [&](int t, int buf) {
    stage_mn<OF_M>(sA + buf * OF_A, a + (int64_t)(g + (int64_t)t * G) * OF_M, Rk, tid);
  };
  stage_mn<OF_N>(sB, c + n0, Rk, tid);
  if (nt > 0) load_a(0, 0);
  if (nt > 1) load_a(1, 1);
  tc::cp_async_commit();
  if (warp == 0) tc::tmem_alloc<512>(slot);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
  }
  tc::cp_async_wait0();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;
  const uint32_t idesc = tc::idesc_bf16(OF_M, OF_N, true, true);
  const uint32_t sb = tc::smem_u32(sB);
  auto issue = [&](int t) {
    const uint32_t sa = tc::smem_u32(sA + (t & 1) * OF_A);
    const uint32_t acc = tbase + (uint32_t)((t & 1) * OF_N);
#pragma unroll
    for (int ks = 0; ks < OF_K / 16; ++ks)
      tc::mma_bf16_ss_w(acc, tc::sdesc(sa + ks * 2 * (OF_M / 8) * 128, (OF_M / 8) * 128, 128),
                        tc::sdesc(sb + ks * 2 * (OF_N / 8) * 128, (OF_N / 8) * 128, 128), idesc, ks > 0 ? 1u : 0u);
    tc::mma_commit_w(&bar[t & 1]);
  };
  if (warp == 0 && nt > 0) issue(0);
  const int quarter = warp & 3, cq = warp >> 2;  // TMEM lane quarter (= one i), column quarter (2 j)
  for (int t = 0; t < nt; ++t) {
    if (warp == 0 && t + 1 < nt) issue(t + 1);
    const int64_t m0 = (int64_t)(g + (int64_t)t * G) * OF_M;  // rows (i, p) of num
    const int64_t i = m0 / k + quarter;
    const int p = lane;
    float scv[OF_N / 4 / 32];  // rec of this warp's (i, j) rows, fetched while the MMAs run
#pragma unroll
    for (int jc = 0; jc < OF_N / 4 / 32; ++jc) scv[jc] = __ldg(rec + i * R + (n0 + cq * (OF_N / 4) + jc * 32) / k);
    tc::mbar_wait(&bar[t & 1], (uint32_t)((t >> 1) & 1));
    tc::fence_after();
    if (t + 2 < nt) {
      load_a(t + 2, t & 1);
      tc::cp_async_commit();
    }
#pragma unroll
    for (int jc = 0; jc < OF_N / 4 / 32; ++jc) {
      const int col = cq * (OF_N / 4) + jc * 32;
      const int64_t j = (n0 + col) / k;
      float v[32];
      tc::tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((t & 1) * OF_N + col), v);
      tc::wait_ld();
      const float sc = scv[jc];
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e] * sc, v[2 * e + 1] * sc);
      // lane p's 64 B are at p*64 in the 2 KB outn row (i, j)
      uint4* xb = reinterpret_cast<uint4*>(sX + warp * 2048);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        xb[p * 4 + (e ^ (p & 3))] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(outn + (i * R + j) * (int64_t)(k * k));
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int cc = e * 32 + lane, r = cc >> 2, q = cc & 3;
        dst[cc] = xb[r * 4 + (q ^ (r & 3))];
      }
      __syncwarp();
    }
    tc::cp_async_wait0();  // A(t+2) landed: MMA(t+2) is issued at the top of the next iteration
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

}  // namespace

// a, c [S = 128, NI*k] / [S, R*k] bf16 (this shard's rows of a; all of c),
// rec [NI*R] -> outn [NI*R, k*k] bf16.  false: shape not covered.
bool opm_outn_tc(const void* a, const void* c, const float* rec, void* outn, int64_t S, int64_t R, int64_t k,
                 int64_t NI, cudaStream_t s) {
  if (S != OF_K || k != 32 || ((R * k) % OF_N) != 0 || NI <= 0 || ((NI * k) % OF_M) != 0) return false;
  if (((uintptr_t)a | (uintptr_t)c | (uintptr_t)outn) & 15) return false;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(opm_outn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OF_SMEM));
    attr = true;
  }
  const int64_t n_mt = NI * k / OF_M;
  const int n_nt = (int)(R * k / OF_N);
  int G = num_sms() / n_nt;
  if (G < 1) G = 1;
  if (G > n_mt) G = (int)n_mt;
  dim3 grid((unsigned)G, (unsigned)n_nt);
  opm_outn_tc_kernel<<<grid, OF_T, OF_SMEM, s>>>((const bf16*)a, (const bf16*)c, rec, (bf16*)outn, R, (int)k,
                                                 n_mt, G);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

}  // namespace evo

extern "C" int evo_opm_outn(const void* a, const void* c, const float* rec, void* outn, int64_t S, int64_t R,
                            int64_t k, int64_t NI, int dtype, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(dtype == EVO_BF16, EVO_ERR_UNSUPPORTED, "opm_outn: bf16 only");
  EVO_REQUIRE(evo::opm_outn_tc(a, c, rec, outn, S, R, k, NI, (cudaStream_t)stream), EVO_ERR_UNSUPPORTED,
              "opm_outn: needs S = 128 sequences per worker, k = 32, n_res*k a multiple of 256");
  EVO_API_END
}
