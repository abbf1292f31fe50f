// Gated attention core on the 5th-generation tensor cores (tcgen05 + TMEM),
// bf16 storage / fp32 accumulation (src/attention.py:118-174, fused op).
//
// One CTA per (query tile of 128 rows, head h, batch b); 8 warps.
//   1. Q [128 x D], K, V [Lp x D] staged into shared memory as UMMA core
//      matrices with 16-byte cp.async (token-major qkvg rows, any
//      (batch, position) strides -> the four Evoformer variants);
//   2. S = Q K^T on the tensor core into TMEM (one elected thread issues
//      D/16 tcgen05.mma of 128 x Lp x 16, completion via tcgen05.commit ->
//      mbarrier);
//   3. softmax from TMEM: the two warps sharing a TMEM lane quarter split the
//      columns; pass 1 forms logits = S*c^-1/2 + (mask-1)*1e9 + nb in the
//      reference's order and writes them back to TMEM, pass 2 exponentiates,
//      sums and writes P (bf16) into shared memory as the A operand;
//   4. O = P V on the tensor core, accumulated into TMEM columns aliasing S;
//   5. epilogue: ctx = O / rowsum, gate = sigmoid(g + bg), gated = ctx*gate,
//      and (row max, 1/rowsum) for the backward.
// The whole key range (Lp <= 256) is resident, so the softmax is exact
// two-pass rather than online.
#include "common.cuh"
#include "reduce.cuh"
#include "attn_geom.cuh"
#include "tc_common.cuh"

namespace evo {


namespace {

using bf16 = __nv_bfloat16;
constexpr float LOG2E = 1.4426950408889634f;

template <int LP>
struct TmemCols {
  static constexpr int value = LP <= 32 ? 32 : (LP <= 64 ? 64 : (LP <= 128 ? 128 : 256));
};

template <int D, int LP>
struct FwdSmem {
  static constexpr int q = 0;
  static constexpr int k = q + 128 * D * 2;
  static constexpr int v = k + LP * D * 2;
  static constexpr int p = v + LP * D * 2;
  static constexpr int mb = p + 128 * LP * 2;
  static constexpr int ex = mb + LP * 4;
  static constexpr int bar = ex + 512 * 4;
  static constexpr int slot = bar + 8;
  static constexpr int total = slot + 8;
};

__device__ __forceinline__ void st_zero16(void* p) {
  *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
}

template <int D, int LP>
__global__ void __launch_bounds__(256) attn_fwd_tc_kernel(
    const bf16* __restrict__ qkvg, const float* __restrict__ mask, const float* __restrict__ bias_t,
    const float* __restrict__ bg, bf16* __restrict__ ctx, bf16* __restrict__ gate,
    bf16* __restrict__ gated, float* __restrict__ lse, AttnGeom g, float scale) {
  using SM = FwdSmem<D, LP>;
  constexpr int TCOLS = TmemCols<(LP > D ? LP : D)>::value;
  constexpr int DC = D / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem + SM::q);
  bf16* sK = reinterpret_cast<bf16*>(smem + SM::k);
  bf16* sV = reinterpret_cast<bf16*>(smem + SM::v);
  bf16* sP = reinterpret_cast<bf16*>(smem + SM::p);
  float* sMb = reinterpret_cast<float*>(smem + SM::mb);
  float* sEx = reinterpret_cast<float*>(smem + SM::ex);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::bar);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + SM::slot);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t b = blockIdx.z, h = blockIdx.y;
  const int q0 = blockIdx.x * 128;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;

  if (warp == 0) tc::tmem_alloc<TCOLS>(slot);
  if (tid == 32) tc::mbar_init(bar, 1);

  // ---- stage Q, K, V (core-matrix layout) and the key mask bias ----
  for (int e = tid; e < 128 * DC; e += 256) {
    const int r = e / DC, c = e % DC;
    bf16* dst = sQ + ((r >> 3) * DC + c) * 64 + (r & 7) * 8;
    if (q0 + r < L)
      tc::cp_async16(dst, qkvg + g.tok(b, q0 + r) * g.ld + h * D + c * 8);
    else
      st_zero16(dst);
  }
  for (int e = tid; e < LP * DC; e += 256) {
    const int j = e / DC, c = e % DC;
    const int off = ((j >> 3) * DC + c) * 64 + (j & 7) * 8;
    if (j < L) {
      const bf16* src = qkvg + g.tok(b, j) * g.ld + HD + h * D + c * 8;
      tc::cp_async16(sK + off, src);
      tc::cp_async16(sV + off, src + HD);
    } else {
      st_zero16(sK + off);
      st_zero16(sV + off);
    }
  }
  for (int j = tid; j < LP; j += 256)
    sMb[j] = j < L ? (mask[b * g.msb + (int64_t)j * g.msl] - 1.0f) * 1e9f : -INFINITY;
  tc::cp_async_wait_all();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;

  // ---- S = Q K^T  (M=128, N=LP, K=D) ----
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16(128, LP, false, false);
#pragma unroll
    for (int k = 0; k < D / 16; ++k) {
      const uint64_t ad = tc::sdesc(tc::smem_u32(sQ) + k * 256, 128, DC * 128);
      const uint64_t bd = tc::sdesc(tc::smem_u32(sK) + k * 256, 128, DC * 128);
      tc::mma_bf16_ss(tbase, ad, bd, idesc, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after();

  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const int i = q0 + row;
  const bool valid = i < L;
  const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16);
  constexpr int HALF = LP / 2;
  constexpr int NCH = HALF / 32;
  const float* brow = (bias_t != nullptr && valid) ? bias_t + (size_t)h * L * L + i : nullptr;

  // ---- pass 1: logits (reference order) + row max, logits back to TMEM ----
  float mx = -INFINITY;
#pragma unroll 1
  for (int ch = 0; ch < NCH; ++ch) {
    const int c0 = half * HALF + ch * 32;
    float v[32];
    tc::tmem_ld32(tl + c0, v);
    tc::wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int j = c0 + e;
      float x = v[e] * scale;
      x = x + sMb[j];
      if (brow != nullptr && j < L) x = x + brow[(size_t)j * L];
      v[e] = x;
      mx = fmaxf(mx, x);
    }
    tc::tmem_st32(tl + c0, v);
  }
  tc::wait_st();
  sEx[half * 128 + row] = mx;
  __syncthreads();
  const float m = fmaxf(sEx[row], sEx[128 + row]);

  // ---- pass 2: P = exp(logits - m) -> bf16 A operand; row sums ----
  float sum = 0.f;
#pragma unroll 1
  for (int ch = 0; ch < NCH; ++ch) {
    const int c0 = half * HALF + ch * 32;
    float v[32];
    tc::tmem_ld32(tl + c0, v);
    tc::wait_ld();
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float p0 = tc::ex2((v[e] - m) * LOG2E);
      const float p1 = tc::ex2((v[e + 1] - m) * LOG2E);
      sum += p0 + p1;
      pk[e / 2] = tc::pack_bf16(p0, p1);
    }
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
      bf16* dst = sP + ((row >> 3) * (LP / 8) + (c0 >> 3) + qd) * 64 + (row & 7) * 8;
      *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * qd], pk[4 * qd + 1], pk[4 * qd + 2], pk[4 * qd + 3]);
    }
  }
  sEx[256 + half * 128 + row] = sum;
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();

  // ---- O = P V  (M=128, N=D, K=LP), accumulated over S's first D columns ----
  if (tid == 0) {
    tc::fence_after();
    const uint32_t idesc = tc::idesc_bf16(128, D, false, true);
#pragma unroll 4
    for (int k = 0; k < LP / 16; ++k) {
      const uint64_t ad = tc::sdesc(tc::smem_u32(sP) + k * 256, 128, (LP / 8) * 128);
      const uint64_t bd = tc::sdesc(tc::smem_u32(sV) + k * 2 * DC * 128, DC * 128, 128);
      tc::mma_bf16_ss(tbase, ad, bd, idesc, k > 0 ? 1u : 0u);
    }
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 1);
  tc::fence_after();

  // ---- epilogue: normalise, gate, store ----
  const float l = sEx[256 + row] + sEx[384 + row];
  const float invl = 1.0f / l;
  constexpr int DH = D / 2;
  float o[DH];
  if constexpr (DH == 16) {
    tc::tmem_ld16(tl + half * DH, o);
  } else {
    tc::tmem_ld8(tl + half * DH, o);
  }
  tc::wait_ld();
  if (valid) {
    const int64_t t = g.tok(b, i);
    const int64_t c0 = h * D + half * DH;
    const bf16* gp = qkvg + t * g.ld + 3 * HD + c0;
    uint32_t pc[DH / 2], pg[DH / 2], pgd[DH / 2];
#pragma unroll
    for (int k = 0; k < DH; k += 2) {
      const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(gp + k);
      const float c0f = o[k] * invl, c1f = o[k + 1] * invl;
      const float g0 = 1.0f / (1.0f + __expf(-(__bfloat162float(g2.x) + bg[c0 + k])));
      const float g1 = 1.0f / (1.0f + __expf(-(__bfloat162float(g2.y) + bg[c0 + k + 1])));
      pc[k / 2] = tc::pack_bf16(c0f, c1f);
      pg[k / 2] = tc::pack_bf16(g0, g1);
      pgd[k / 2] = tc::pack_bf16(c0f * g0, c1f * g1);
    }
#pragma unroll
    for (int k = 0; k < DH / 8; ++k) {
      reinterpret_cast<uint4*>(ctx + t * HD + c0)[k] = make_uint4(pc[4 * k], pc[4 * k + 1], pc[4 * k + 2], pc[4 * k + 3]);
      reinterpret_cast<uint4*>(gate + t * HD + c0)[k] = make_uint4(pg[4 * k], pg[4 * k + 1], pg[4 * k + 2], pg[4 * k + 3]);
      reinterpret_cast<uint4*>(gated + t * HD + c0)[k] = make_uint4(pgd[4 * k], pgd[4 * k + 1], pgd[4 * k + 2], pgd[4 * k + 3]);
    }
    if (half == 0) {
      lse[2 * ((b * g.H + h) * L + i)] = m;
      lse[2 * ((b * g.H + h) * L + i) + 1] = invl;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<TCOLS>(tbase);
}

bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_DISABLE_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int D, int LP>
void launch_fwd(const void* qkvg, const float* mask, const float* bias_t, const float* bg, void* ctx,
                void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  using SM = FwdSmem<D, LP>;
  auto k = attn_fwd_tc_kernel<D, LP>;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::total));
    attr = true;
  }
  dim3 grid(cdiv(g.L, 128), (unsigned)g.H, (unsigned)g.B);
  const float scale = (float)(1.0 / sqrt((double)D));
  k<<<grid, 256, SM::total, s>>>((const bf16*)qkvg, mask, bias_t, bg, (bf16*)ctx, (bf16*)gate,
                                 (bf16*)gated, lse, g, scale);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

template <int D>
void launch_fwd_lp(const void* qkvg, const float* mask, const float* bias_t, const float* bg,
                   void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  const int64_t L = g.L;
  if (L <= 64) launch_fwd<D, 64>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
  else if (L <= 128) launch_fwd<D, 128>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
  else if (L <= 192) launch_fwd<D, 192>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd<D, 256>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
}

}  // namespace

bool attn_fwd_tc_try(const void* qkvg, const float* mask, const float* bias_t, const float* bg,
                     void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, int dtype,
                     cudaStream_t s) {
  if (tc_disabled() || dtype != EVO_BF16) return false;
  if (!(g.D == 16 || g.D == 32) || g.L > 256 || g.L < 1) return false;
  if ((g.ld % 8) != 0 || (((uintptr_t)qkvg) & 15) != 0) return false;
  if (((uintptr_t)ctx | (uintptr_t)gate | (uintptr_t)gated) & 15) return false;
  if (g.D == 16)
    launch_fwd_lp<16>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
  else
    launch_fwd_lp<32>(qkvg, mask, bias_t, bg, ctx, gate, gated, lse, g, s);
  return true;
}

bool attn_bwd_tc_try(const void*, const float*, const float*, const void*, const void*, const void*,
                     const float*, void*, float*, float*, int, void*, size_t, const AttnGeom&, int,
                     cudaStream_t) {
  return false;
}
int64_t attn_bwd_tc_workspace(const AttnGeom&, int) { return 0; }

}  // namespace evo
