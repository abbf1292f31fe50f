// Pair-bias forward on the warp-level tensor cores: nb[h, i] = LN(z_i) . w[:, h]
// (src/model.py:312-317) for bf16 pair activations with c_z = 128, H <= 8.
//
// With gw = g (x) w and the per-head constants G = sum_c gw[c, :],
// BW = sum_c b[c] w[c, :], the LayerNorm folds into the projection:
//   nb[h] = rstd * (sum_c z_c gw[c, h] - mean * G[h]) + BW[h].
// The contraction z . gw is an [64 tokens x 128] x [128 x 8] product per
// stage: mma.sync m16n8k16 (bf16 in, fp32 accumulate) with z read straight
// from a TMA-loaded, 128-B-swizzled tile by ldmatrix, and gw split into two
// bf16 halves (gw = hi + lo, |lo| <= 2^-9 |gw|) so the product keeps ~16
// significant bits of gw on top of the exact bf16 z -- the fp32-FMA kernel's
// accuracy well inside the bf16 output rounding.  The row statistics come
// from the same A fragments (each lane sums its 32 channels of two tokens,
// then a quad shuffle).
//
// Persistent blocks of 4 warps (16 tokens each per 64-token stage), two
// stages in flight; the triangle-end layout (swap) is a different TMA box over
// the same [NI][NJ][C] view, so both layouts write their nb planes in output
// order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "reduce.cuh"
#include "tc_common.cuh"

namespace evo {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();  // gemm_tc.cu

namespace {

constexpr int PBM_C = 128, PBM_TOK = 64, PBM_WARPS = 4;
constexpr int PBM_HALF = PBM_TOK * 64 * 2;  // one 64-channel box: 8 KB
constexpr int PBM_TILE = 2 * PBM_HALF;      // 16 KB per stage
// tiles, then barriers / G, BW / per-warp partials / LN affine (1408 B), plus
// the 1024-B alignment slack
constexpr int PBM_SMEM = 2 * PBM_TILE + 1024 + 1536;
// with the LayerNorm output: two more tiles stage xl for its TMA stores
constexpr int PBM_SMEM_LN = 4 * PBM_TILE + 1024 + 1536;

__device__ __forceinline__ void pbm_tma_load3(const CUtensorMap* m, uint32_t dst, uint32_t bar, int c0, int c1,
                                              int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float2 bf2f(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}

// bf16 hi / lo halves of the pair (x, y), packed (first element in the low half)
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 hx = __float2bfloat16_rn(x), hy = __float2bfloat16_rn(y);
  const __nv_bfloat16 lx = __float2bfloat16_rn(x - __bfloat162float(hx));
  const __nv_bfloat16 ly = __float2bfloat16_rn(y - __bfloat162float(hy));
  hi = (uint32_t)__bfloat16_as_ushort(hx) | ((uint32_t)__bfloat16_as_ushort(hy) << 16);
  lo = (uint32_t)__bfloat16_as_ushort(lx) | ((uint32_t)__bfloat16_as_ushort(ly) << 16);
}

__device__ __forceinline__ void pbm_tma_store3(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(src)
               : "memory");
}

// LN = true: also the LayerNorm of the same rows with its own affine
// (lg, lb) -> xl (bf16, TMA-stored through two swizzled staging tiles): the
// triangle attentions' input LayerNorm and their pair-bias LayerNorm read the
// same pair activations, so one pass serves both (src/model.py:381-398).
template <bool LN>
__global__ void __launch_bounds__(PBM_WARPS * 32) pair_bias_fwd_mma_kernel(
    const __grid_constant__ CUtensorMap tmz, const __grid_constant__ CUtensorMap tmx, const float* __restrict__ g,
    const float* __restrict__ b, const float* __restrict__ w, const float* __restrict__ lg,
    const float* __restrict__ lb, __nv_bfloat16* __restrict__ nb, float* __restrict__ mean, float* __restrict__ rstd,
    int64_t NI, int64_t NJ, int H, int swap, int64_t nstage, int64_t per_line) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NT = LN ? 4 : 2;  // z double buffer (+ xl double buffer)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NT * PBM_TILE);
  float* sG = reinterpret_cast<float*>(smem + NT * PBM_TILE + 64);  // [8] G, [8] BW
  float* spart = sG + 16;                                             // [4 warps][16]
  float* sLG = spart + 64;                                            // [128] lg, [128] lb (LN)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const uint32_t s_base = tc::smem_u32(smem);
  const uint32_t s_full = tc::smem_u32(full);

  auto coords = [&](int64_t st, int& c1, int& c2) {
    const int64_t line = st / per_line, off = (st % per_line) * PBM_TOK;
    if (swap) { c1 = (int)line; c2 = (int)off; }   // (y, x0..x0+63)
    else { c1 = (int)off; c2 = (int)line; }        // (y0..y0+63, x)
  };
  auto issue = [&](int64_t st, int buf) {
    int c1, c2;
    coords(st, c1, c2);
    const uint32_t bar = s_full + 8 * buf;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(PBM_TILE) : "memory");
    pbm_tma_load3(&tmz, s_base + buf * PBM_TILE, bar, 0, c1, c2);
    pbm_tma_load3(&tmz, s_base + buf * PBM_TILE + PBM_HALF, bar, 64, c1, c2);
  };

  if (LN) {
    sLG[tid] = lg[tid];
    sLG[PBM_C + tid] = lb[tid];
  }
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmz)) : "memory");
    if (LN) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((int64_t)blockIdx.x < nstage) issue(blockIdx.x, 0);
    if ((int64_t)blockIdx.x + gridDim.x < nstage) issue(blockIdx.x + gridDim.x, 1);
  }

  // B fragments of gw (hi / lo) for this lane: chunk kc covers channels
  // 16kc .. 16kc+15; b0 = rows 2tq, 2tq+1, b1 = rows 2tq+8, 2tq+9, column
  // (head) gq
  uint32_t bh0[8], bh1[8], bl0[8], bl1[8];
#pragma unroll
  for (int kc = 0; kc < 8; ++kc) {
    const int c = 16 * kc + 2 * tq;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (gq < H) {
      v[0] = g[c] * w[c * H + gq];
      v[1] = g[c + 1] * w[(c + 1) * H + gq];
      v[2] = g[c + 8] * w[(c + 8) * H + gq];
      v[3] = g[c + 9] * w[(c + 9) * H + gq];
    }
    split2(v[0], v[1], bh0[kc], bl0[kc]);
    split2(v[2], v[3], bh1[kc], bl1[kc]);
  }
  // G[h], BW[h]: thread = channel
  {
    float gs[8], bs[8];
    const float ge = g[tid], be = b[tid];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
      const float we = hh < H ? w[tid * H + hh] : 0.f;
      gs[hh] = ge * we;
      bs[hh] = be * we;
    }
#pragma unroll
    for (int hh = 0; hh < 8; ++hh)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gs[hh] += __shfl_xor_sync(0xffffffffu, gs[hh], o);
        bs[hh] += __shfl_xor_sync(0xffffffffu, bs[hh], o);
      }
    if (lane == 0)
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        spart[warp * 16 + hh] = gs[hh];
        spart[warp * 16 + 8 + hh] = bs[hh];
      }
  }
  __syncthreads();
  if (tid < 16) sG[tid] = spart[tid] + spart[16 + tid] + spart[32 + tid] + spart[48 + tid];
  __syncthreads();
  const float G0 = sG[2 * tq], G1 = sG[2 * tq + 1], B0 = sG[8 + 2 * tq], B1 = sG[8 + 2 * tq + 1];

  const int64_t RR = NI * NJ;
  // ldmatrix row address pieces (lane -> row of one of the four 8x8 matrices)
  const int lrow = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int lhi = lane >> 4;
  const uint32_t row_off = (uint32_t)lrow * 128;
  const int rsw = lrow & 7;
  int k = 0;
#pragma unroll 1
  for (int64_t st = blockIdx.x; st < nstage; st += gridDim.x, ++k) {
    const int buf = k & 1;
    tc::mbar_wait(&full[buf], (uint32_t)((k >> 1) & 1));
    const uint32_t tile = s_base + buf * PBM_TILE;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    float2 s0 = make_float2(0.f, 0.f), s1 = s0;
    uint32_t af[8][4];  // this lane's z values of the stage (kept for the second pass)
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
      const int cb = (2 * kc + lhi) & 7;
      const uint32_t addr = tile + (kc >> 2) * PBM_HALF + row_off + (uint32_t)((cb ^ rsw) << 4);
      ldsm_x4(addr, af[kc]);
      mma16816(acc, af[kc], bh0[kc], bh1[kc]);
      mma16816(acc, af[kc], bl0[kc], bl1[kc]);
      const float2 f0 = bf2f(af[kc][0]), f1 = bf2f(af[kc][1]), f2 = bf2f(af[kc][2]), f3 = bf2f(af[kc][3]);
      s0 = __fadd2_rn(s0, __fadd2_rn(f0, f2));
      s1 = __fadd2_rn(s1, __fadd2_rn(f1, f3));
    }
    // every warp has read this buffer: refill it with the stage two ahead
    __syncthreads();
    if (tid == 0 && st + 2 * (int64_t)gridDim.x < nstage) issue(st + 2 * (int64_t)gridDim.x, buf);
    float sa = s0.x + s0.y, sb = s1.x + s1.y;
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const float mua = sa / (float)PBM_C, mub = sb / (float)PBM_C;
    // second pass: sum of squared deviations (the LayerNorm's own two-pass form)
    float2 q0 = make_float2(0.f, 0.f), q1 = q0;
    {
      const float2 ma = make_float2(-mua, -mua), mb = make_float2(-mub, -mub);
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {
        const float2 d0 = __fadd2_rn(bf2f(af[kc][0]), ma), d2 = __fadd2_rn(bf2f(af[kc][2]), ma);
        const float2 d1 = __fadd2_rn(bf2f(af[kc][1]), mb), d3 = __fadd2_rn(bf2f(af[kc][3]), mb);
        q0 = __ffma2_rn(d0, d0, __ffma2_rn(d2, d2, q0));
        q1 = __ffma2_rn(d1, d1, __ffma2_rn(d3, d3, q1));
      }
    }
    float qa = q0.x + q0.y, qb = q1.x + q1.y;
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      qa += __shfl_xor_sync(0xffffffffu, qa, o);
      qb += __shfl_xor_sync(0xffffffffu, qb, o);
    }
    const float inva = rsqrtf(qa / (float)PBM_C + 1e-5f);
    const float invb = rsqrtf(qb / (float)PBM_C + 1e-5f);
    const int64_t line = st / per_line, off = (st % per_line) * PBM_TOK;
    if constexpr (LN) {
      // xl = (z - mean) * rstd * lg + lb for this lane's (token, channel pair)
      // fragments, into the swizzled staging tile of this stage's parity
      const uint32_t xt = s_base + (2 + buf) * PBM_TILE;
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // tile xt's last store read
      __syncthreads();
      const int r0 = warp * 16 + gq;
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + (q & 1) * 8, hi = q >> 1;       // a0: (g, lo) a1: (g+8, lo) a2: (g, hi) a3: (g+8, hi)
          const int c = 16 * kc + 8 * hi + 2 * tq;
          const float mu = (q & 1) ? mub : mua, iv = (q & 1) ? invb : inva;
          const float2 zf = bf2f(af[kc][q]);
          const float y0 = fmaf((zf.x - mu) * iv, sLG[c], sLG[PBM_C + c]);
          const float y1 = fmaf((zf.y - mu) * iv, sLG[c + 1], sLG[PBM_C + c + 1]);
          const int cb = (2 * kc + hi) & 7;
          const uint32_t a = xt + (kc >> 2) * PBM_HALF + r * 128 + ((cb ^ (r & 7)) << 4) + 4 * tq;
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(tc::pack_bf16(y0, y1)) : "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        int c1, c2;
        coords(st, c1, c2);
        pbm_tma_store3(&tmx, xt, 0, c1, c2);
        pbm_tma_store3(&tmx, xt + PBM_HALF, 64, c1, c2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    const int64_t lim = swap ? NI : NJ;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t r = off + warp * 16 + gq + half * 8;  // position along the stage's line
      if (r >= lim) continue;
      const int64_t i = swap ? line * NI + r : line * NJ + r;    // output position
      const int64_t tok = swap ? r * NJ + line : i;              // token row of z
      const float mu = half ? mub : mua, inv = half ? invb : inva;
      const float p0 = half ? acc[2] : acc[0], p1 = half ? acc[3] : acc[1];
      if (2 * tq < H) nb[(int64_t)(2 * tq) * RR + i] = __float2bfloat16_rn(fmaf(inv, p0 - mu * G0, B0));
      if (2 * tq + 1 < H) nb[(int64_t)(2 * tq + 1) * RR + i] = __float2bfloat16_rn(fmaf(inv, p1 - mu * G1, B1));
      if (tq == 0) {
        mean[tok] = mu;
        rstd[tok] = inv;
      }
    }
  }
  if (LN && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

bool pbm_disabled() {
  static const bool off = [] {
    const char* e = getenv("EVO_PB_MMA");
    return e && e[0] == '0';
  }();
  return off;
}

}  // namespace

static bool pbm_map(CUtensorMap* m, const void* base, int64_t NI, int64_t NJ, int swap) {
  auto enc = tmap_encoder();
  if (!enc || (((uintptr_t)base) & 15)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)PBM_C, (cuuint64_t)NJ, (cuuint64_t)NI};
  cuuint64_t strides[2] = {(cuuint64_t)(PBM_C * 2), (cuuint64_t)(NJ * PBM_C * 2)};
  cuuint32_t box[3] = {64, swap ? 1u : (cuuint32_t)PBM_TOK, swap ? (cuuint32_t)PBM_TOK : 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool pbm_launch(const void* z, const float* g, const float* b, const float* w, const float* lg,
                       const float* lb, void* xl, void* nb, float* mean, float* rstd, int64_t NI, int64_t NJ,
                       int64_t H, int swap, cudaStream_t s) {
  CUtensorMap mz, mx;
  if (!pbm_map(&mz, z, NI, NJ, swap)) return false;
  if (xl) {
    if (!pbm_map(&mx, xl, NI, NJ, swap)) return false;
  } else {
    mx = mz;
  }
  const int64_t lines = swap ? NJ : NI, along = swap ? NI : NJ;
  const int64_t per_line = (along + PBM_TOK - 1) / PBM_TOK;
  const int64_t nstage = lines * per_line;
  static bool attr[2] = {false, false};
  if (!attr[xl ? 1 : 0]) {
    if (xl)
      EVO_CUDA(cudaFuncSetAttribute(pair_bias_fwd_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    PBM_SMEM_LN));
    else
      EVO_CUDA(cudaFuncSetAttribute(pair_bias_fwd_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    PBM_SMEM));
    attr[xl ? 1 : 0] = true;
  }
  static const int bps = [] {
    const char* e = getenv("EVO_PB_MMA_BPS");  // resident blocks per SM (sweeps)
    const int v = e ? atoi(e) : 0;
    return v > 0 && v <= 8 ? v : 0;
  }();
  const int64_t want = (int64_t)num_sms() * (bps ? bps : (xl ? 3 : 4));
  const unsigned grid = (unsigned)(nstage < want ? nstage : want);
  if (xl)
    pair_bias_fwd_mma_kernel<true><<<grid, PBM_WARPS * 32, PBM_SMEM_LN, s>>>(
        mz, mx, g, b, w, lg, lb, (__nv_bfloat16*)nb, mean, rstd, NI, NJ, (int)H, swap, nstage, per_line);
  else
    pair_bias_fwd_mma_kernel<false><<<grid, PBM_WARPS * 32, PBM_SMEM, s>>>(
        mz, mx, g, b, w, nullptr, nullptr, (__nv_bfloat16*)nb, mean, rstd, NI, NJ, (int)H, swap, nstage, per_line);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool pair_bias_fwd_mma(const void* z, int dt, const float* g, const float* b, const float* w, void* nb, float* mean,
                       float* rstd, int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap, cudaStream_t s) {
  if (pbm_disabled() || dt != EVO_BF16 || C != PBM_C || H > 8 || H < 1) return false;
  if (NI * NJ < 4096 || NI > (1 << 30) || NJ > (1 << 30)) return false;
  return pbm_launch(z, g, b, w, nullptr, nullptr, nullptr, nb, mean, rstd, NI, NJ, H, swap, s);
}

// LayerNorm (lg, lb) of the same rows in the same pass (xl: bf16, z's layout)
bool ln_pair_bias_fwd_mma(const void* z, int dt, const float* lg, const float* lb, const float* g, const float* b,
                          const float* w, void* xl, void* nb, float* mean, float* rstd, int64_t NI, int64_t NJ,
                          int64_t C, int64_t H, int swap, cudaStream_t s) {
  if (pbm_disabled() || dt != EVO_BF16 || C != PBM_C || H > 8 || H < 1 || !xl) return false;
  if (NI * NJ < 4096 || NI > (1 << 30) || NJ > (1 << 30)) return false;
  return pbm_launch(z, g, b, w, lg, lb, xl, nb, mean, rstd, NI, NJ, H, swap, s);
}

}  // namespace evo
