// Gated attention core forward on the 5th-generation tensor cores (tcgen05 +
// TMEM), bf16 storage / fp32 accumulation -- the fused op of
// src/attention.py:118-174.  Backward: attention_tc_bwd.cu.
//
// One CTA per (batch group, head h, query tile of 128 rows), 8 warps, looping
// over the batches of its group:
//   * the pair-bias tile nb[h, q0:q0+128, :] is the same for every batch and
//     is staged into shared memory once per CTA (cp.async, padded rows);
//   * Q [128 x D], K, V [Lp x D] of the next batch are prefetched with 16-byte
//     cp.async into UMMA core-matrix layout while the current batch runs
//     (token-major qkvg rows, any (batch, position) strides -> all four
//     Evoformer variants read the same buffers without transposes);
//   * S = Q K^T on the tensor core into TMEM (one thread issues D/16
//     tcgen05.mma 128 x Lp x 16; tcgen05.commit -> mbarrier);
//   * softmax from TMEM: the two warps sharing a TMEM lane quarter split the
//     keys; pass 1 forms logits = S*c^-1/2 + (mask-1)*1e9 + nb in the
//     reference's order (src/attention.py:151-156), times log2(e), back into
//     TMEM; pass 2 exponentiates (ex2), sums, and packs P as bf16 pairs back
//     into TMEM over the logits it has consumed;
//   * O = P V with the A operand read from TMEM (tcgen05.mma ... [a_tmem]),
//     V as an MN-major shared-memory operand;
//   * epilogue: ctx = O / rowsum, gate = sigmoid(g + bg), gated = ctx*gate,
//     and (row max, 1/rowsum) for the backward.
#include "common.cuh"
#include "reduce.cuh"
#include "attn_geom.cuh"
#include "tc_common.cuh"

namespace evo {

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void st_zero16(void* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u); }

__device__ __forceinline__ void bf16x8_to_f(const uint4& u, float* f) {
  const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(hh[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

constexpr int pow2_cols(int n) { return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 256 ? 256 : 512))); }

template <int D, int LP>
struct Fwd {
  static constexpr int DC = D / 8;
  static constexpr int HALF = LP / 2;
  static constexpr int OC = (D <= HALF / 2) ? HALF / 2 : LP;  // O columns (free after pass 2)
  static constexpr int TCOLS = pow2_cols(OC + D > LP ? OC + D : LP);
  static constexpr int BROW = LP + 8;
  static constexpr int NS = (D == 16) ? 2 : 1;  // Q/K/V staging buffers
  static constexpr int q = 0;
  static constexpr int k = 128 * D * 2;
  static constexpr int v = k + LP * D * 2;
  static constexpr int mb = v + LP * D * 2;
  static constexpr int STAGE = mb + LP * 4;
  static constexpr int bias = NS * STAGE;
  static constexpr int ex = bias + 128 * BROW * 2;
  static constexpr int bar = ex + 512 * 4;
  static constexpr int slot = bar + 8;
  static constexpr int total = slot + 8;
};

// Per-thread staging plan: the (row, 16-B column chunk) pairs of the Q, K, V
// tiles a thread copies are the same for every batch, so their global offsets
// (minus the batch term) and shared-memory offsets are computed once; a batch
// then costs one add and one cp.async per chunk.
template <int D, int LP>
struct FwdStager {
  using F = Fwd<D, LP>;
  static constexpr int DC = F::DC;
  static constexpr int NQ = (128 * DC + 255) / 256;
  static constexpr int NK = (LP * DC + 255) / 256;
  int qoff[NQ], koff[NK];      // element offsets from the batch's token-row base; -1 = zero-fill
  int qdst[NQ], kdst[NK];      // byte offsets inside a stage
  int moff;                    // mask element offset (-1: none / beyond L)
  int mdst;
  __device__ __forceinline__ void init(const AttnGeom& g, int64_t h, int q0, int tid) {
    const int L = (int)g.L;
    const int64_t HD = g.H * D;
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int e = tid + u * 256;
      const int r = e / DC, c = e % DC;
      qdst[u] = e < 128 * DC ? F::q + (((r >> 3) * DC + c) * 64 + (r & 7) * 8) * 2 : -1;
      qoff[u] = (e < 128 * DC && q0 + r < L) ? (int)((q0 + r) * g.sl * g.ld + h * D + c * 8) : -1;
    }
#pragma unroll
    for (int u = 0; u < NK; ++u) {
      const int e = tid + u * 256;
      const int j = e / DC, c = e % DC;
      kdst[u] = e < LP * DC ? (((j >> 3) * DC + c) * 64 + (j & 7) * 8) * 2 : -1;
      koff[u] = (e < LP * DC && j < L) ? (int)(j * g.sl * g.ld + HD + h * D + c * 8) : -1;
    }
    mdst = tid < LP ? F::mb + tid * 4 : -1;
    moff = tid < L ? (int)(tid * g.msl) : -1;
  }
  // Q, K and the key mask of batch b
  __device__ __forceinline__ void qkm(uint8_t* st, const bf16* qkvg, const float* mask, const AttnGeom& g,
                                      int64_t b) const {
    const bf16* base = qkvg + b * g.sb * g.ld;
#pragma unroll
    for (int u = 0; u < NQ; ++u)
      if (qdst[u] >= 0) {
        if (qoff[u] >= 0) tc::cp_async16(st + qdst[u], base + qoff[u]);
        else st_zero16(st + qdst[u]);
      }
#pragma unroll
    for (int u = 0; u < NK; ++u)
      if (kdst[u] >= 0) {
        if (koff[u] >= 0) tc::cp_async16(st + F::k + kdst[u], base + koff[u]);
        else st_zero16(st + F::k + kdst[u]);
      }
    if (mdst >= 0) {
      if (moff >= 0) tc::cp_async4(st + mdst, mask + b * g.msb + moff);  // converted by mask_to_bias
      else *reinterpret_cast<float*>(st + mdst) = -INFINITY;
    }
  }
  __device__ __forceinline__ void v(uint8_t* st, const bf16* qkvg, const AttnGeom& g, int64_t b) const {
    const bf16* base = qkvg + b * g.sb * g.ld + g.H * D;
#pragma unroll
    for (int u = 0; u < NK; ++u)
      if (kdst[u] >= 0) {
        if (koff[u] >= 0) tc::cp_async16(st + F::v + kdst[u], base + koff[u]);
        else st_zero16(st + F::v + kdst[u]);
      }
  }
};

template <int LP>
__device__ __forceinline__ void stage_bias_rows(bf16* sB, const bf16* nb, int64_t h, int q0, int L,
                                                int tid) {
  constexpr int BROW = LP + 8;
  constexpr int CPR = LP / 8;
  const bool vec_ok = (L % 8) == 0;
  for (int e = tid; e < 128 * CPR; e += 256) {
    const int r = e / CPR, c = e % CPR;
    bf16* dst = sB + r * BROW + c * 8;
    const int qq = q0 + r;
    if (qq < L && vec_ok && c * 8 + 8 <= L) {
      tc::cp_async16(dst, nb + ((size_t)h * L + qq) * L + c * 8);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        dst[u] = (qq < L && c * 8 + u < L) ? nb[((size_t)h * L + qq) * L + c * 8 + u]
                                           : __float2bfloat16(0.f);
    }
  }
}

template <int D, int LP, bool BIAS>
__global__ void __launch_bounds__(256, 2) attn_fwd_tc_kernel(
    const bf16* __restrict__ qkvg, const float* __restrict__ mask, const bf16* __restrict__ nb,
    const float* __restrict__ bg, bf16* __restrict__ ctx, bf16* __restrict__ gate,
    bf16* __restrict__ gated, float* __restrict__ lse, AttnGeom g, float scale, int NG) {
  using F = Fwd<D, LP>;
  constexpr int DC = F::DC, HALF = F::HALF, NCH = HALF / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  float* sEx = reinterpret_cast<float*>(smem + F::ex);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F::bar);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + F::slot);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x;
  const int64_t h = blockIdx.y;
  const int q0 = blockIdx.z * 128;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  const int64_t b_lo = (g.B * grp) / NG, b_hi = (g.B * (grp + 1)) / NG;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const int i = q0 + row;
  const bool valid = i < L;
  const bf16* sBrow = reinterpret_cast<const bf16*>(smem + F::bias) + row * F::BROW;

  if (warp == 0) tc::tmem_alloc<F::TCOLS>(slot);
  if (tid == 32) tc::mbar_init(bar, 1);
  if (BIAS) stage_bias_rows<LP>(reinterpret_cast<bf16*>(smem + F::bias), nb, h, q0, L, tid);
  FwdStager<D, LP> stg;
  stg.init(g, h, q0, tid);
  if (b_lo < b_hi) {
    stg.qkm(smem, qkvg, mask, g, b_lo);
    stg.v(smem, qkvg, g, b_lo);
  }
  tc::cp_async_commit();
  uint32_t phase = 0;
  constexpr int DH = D / 2;  // output channels of this thread (its half of the head)
  const int64_t cbase = h * D + half * DH;
  float bgv[DH];  // gate bias, loaded once
#pragma unroll
  for (int k = 0; k < DH; ++k) bgv[k] = bg[cbase + k];

  for (int64_t b = b_lo; b < b_hi; ++b) {
    const int buf = F::NS == 2 ? (int)((b - b_lo) & 1) : 0;
    uint8_t* st = smem + buf * F::STAGE;
    // this row's gate pre-activations: issued now, consumed after P.V
    uint4 graw[DH / 8];
    const int64_t tok = valid ? g.tok(b, i) : 0;
    if (valid) {
#pragma unroll
      for (int k = 0; k < DH / 8; ++k)
        graw[k] = __ldg(reinterpret_cast<const uint4*>(qkvg + tok * g.ld + 3 * HD + cbase) + k);
    }
    tc::cp_async_wait0();
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *slot;
    const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16);
    if (F::NS == 2 && b + 1 < b_hi) {
      stg.qkm(smem + (buf ^ 1) * F::STAGE, qkvg, mask, g, b + 1);
      stg.v(smem + (buf ^ 1) * F::STAGE, qkvg, g, b + 1);
    }
    tc::cp_async_commit();
    const bf16* sQ = reinterpret_cast<const bf16*>(st + F::q);
    const bf16* sK = reinterpret_cast<const bf16*>(st + F::k);
    const bf16* sV = reinterpret_cast<const bf16*>(st + F::v);
    const float* sMb = reinterpret_cast<const float*>(st + F::mb);

    // ---- S = Q K^T  (M=128, N=LP, K=D) ----
    if (warp == 0) {  // warp-collective issue (uniform descriptors)
      const uint32_t idesc = tc::idesc_bf16(128, LP, false, false);
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint64_t ad = tc::sdesc(tc::smem_u32(sQ) + k * 256, 128, DC * 128);
        const uint64_t bd = tc::sdesc(tc::smem_u32(sK) + k * 256, 128, DC * 128);
        tc::mma_bf16_ss_w(tbase, ad, bd, idesc, k > 0 ? 1u : 0u);
      }
      tc::mma_commit_w(bar);
    }
    tc::mask_to_bias(const_cast<float*>(sMb), LP, L, tid, 256);
    __syncthreads();
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::fence_after();

    // ---- pass 1: logits (reference order), log2 domain, row max ----
    float mx = -INFINITY;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      const int c0 = half * HALF + ch * 32;
      float v[32];
      uint32_t braw[16];
      tc::tmem_ld32(tl + c0, v);
      if (BIAS) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 u = *reinterpret_cast<const uint4*>(sBrow + c0 + 8 * k);
          braw[4 * k] = u.x, braw[4 * k + 1] = u.y, braw[4 * k + 2] = u.z, braw[4 * k + 3] = u.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) braw[k] = 0u;
      }
      tc::wait_ld();
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        const float4 mb4 = *reinterpret_cast<const float4*>(sMb + c0 + e);
        const float2 x0 = tc::logit2(make_float2(v[e], v[e + 1]), tc::bf16x2_f2(braw[e / 2]),
                                     make_float2(mb4.x, mb4.y), scale);
        const float2 x1 = tc::logit2(make_float2(v[e + 2], v[e + 3]), tc::bf16x2_f2(braw[e / 2 + 1]),
                                     make_float2(mb4.z, mb4.w), scale);
        v[e] = x0.x, v[e + 1] = x0.y, v[e + 2] = x1.x, v[e + 3] = x1.y;
        mx = fmaxf(mx, fmaxf(fmaxf(x0.x, x0.y), fmaxf(x1.x, x1.y)));
      }
      tc::tmem_st32(tl + c0, v);
    }
    tc::wait_st();
    sEx[half * 128 + row] = mx;
    __syncthreads();
    const float m = fmaxf(sEx[row], sEx[128 + row]);
    if (F::NS == 1 && b + 1 < b_hi) {  // Q, K (S is done) and the mask (pass 1 is done) are free
      stg.qkm(smem, qkvg, mask, g, b + 1);
      tc::cp_async_commit();
    }

    // ---- pass 2: P = exp2(logits - m), packed bf16 pairs back into TMEM ----
    float2 sum2 = make_float2(0.f, 0.f);
    const float2 nm2 = make_float2(-m, -m);
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      const int c0 = half * HALF + ch * 32;
      float v[32];
      tc::tmem_ld32(tl + c0, v);
      tc::wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float2 d = __fadd2_rn(make_float2(v[e], v[e + 1]), nm2);  // exact near the max
        const float2 p = make_float2(tc::ex2(d.x), tc::ex2(d.y));
        sum2 = __fadd2_rn(sum2, p);
        pk[e / 2] = tc::pack_bf16(p.x, p.y);
      }
      // keys [c0, c0+32) -> columns half*HALF + (c0 - half*HALF)/2 ... (+16)
      tc::tmem_st16u(tl + half * HALF + ch * 16, pk);
    }
    tc::wait_st();
    sEx[256 + half * 128 + row] = sum2.x + sum2.y;
    tc::fence_before();
    __syncthreads();

    // ---- O = P V  (M=128, N=D, K=LP), A from TMEM ----
    if (warp == 0) {  // warp-collective issue (uniform descriptors)
      tc::fence_after();
      const uint32_t idesc = tc::idesc_bf16(128, D, false, true);
#pragma unroll 4
      for (int k = 0; k < LP / 16; ++k) {
        const int key0 = 16 * k;
        const uint32_t pcol = (key0 / HALF) * HALF + (key0 % HALF) / 2;
        const uint64_t bd = tc::sdesc(tc::smem_u32(sV) + k * 2 * DC * 128, DC * 128, 128);
        tc::mma_bf16_ts_w(tbase + F::OC, tbase + pcol, bd, idesc, k > 0 ? 1u : 0u);
      }
      tc::mma_commit_w(bar);
    }
    // gate = sigmoid(g + bg) while the tensor core runs P.V
    float gt[DH];
    if (valid) {
#pragma unroll
      for (int k = 0; k < DH / 8; ++k) {
        const uint32_t w4[4] = {graw[k].x, graw[k].y, graw[k].z, graw[k].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 gp = tc::bf16x2_f2(w4[q]);
          gt[8 * k + 2 * q] = __fdividef(1.0f, 1.0f + __expf(-(gp.x + bgv[8 * k + 2 * q])));
          gt[8 * k + 2 * q + 1] = __fdividef(1.0f, 1.0f + __expf(-(gp.y + bgv[8 * k + 2 * q + 1])));
        }
      }
    }
    const float l = sEx[256 + row] + sEx[384 + row];
    const float invl = 1.0f / l;
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::fence_after();
    if (F::NS == 1 && b + 1 < b_hi) {  // P.V is done with V
      stg.v(smem, qkvg, g, b + 1);
      tc::cp_async_commit();
    }

    // ---- epilogue: normalise, gate, store ----
    float o[DH];
    if constexpr (DH == 16) {
      tc::tmem_ld16(tl + F::OC + half * DH, o);
    } else {
      tc::tmem_ld8(tl + F::OC + half * DH, o);
    }
    tc::wait_ld();
    if (valid) {
      const int64_t t = tok;
      const int64_t c0 = cbase;
      uint32_t pc[DH / 2], pg[DH / 2], pgd[DH / 2];
#pragma unroll
      for (int k = 0; k < DH; k += 2) {
        const float c0f = o[k] * invl, c1f = o[k + 1] * invl;
        pc[k / 2] = tc::pack_bf16(c0f, c1f);
        pg[k / 2] = tc::pack_bf16(gt[k], gt[k + 1]);
        pgd[k / 2] = tc::pack_bf16(c0f * gt[k], c1f * gt[k + 1]);
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
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<F::TCOLS>(*slot);
}

bool fwd_tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_DISABLE_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int D, int LP, bool BIAS>
void launch_fwd(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx,
                void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  using F = Fwd<D, LP>;
  auto k = attn_fwd_tc_kernel<D, LP, BIAS>;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, F::total));
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  const int nqt = (int)((g.L + 127) / 128);
  // resident CTAs per SM (smem-bound), one wave; each CTA loops over its batch group
  const int per_sm = (int)((228 * 1024) / (F::total + 1024)) >= 2 ? 2 : 1;
  int ng = (per_sm * num_sms()) / ((int)g.H * nqt);
  if (ng > g.B) ng = (int)g.B;
  if (ng < 1) ng = 1;
  dim3 grid((unsigned)ng, (unsigned)g.H, (unsigned)nqt);
  const float scale = (float)(1.0 / sqrt((double)D));
  k<<<grid, 256, F::total, s>>>((const bf16*)qkvg, mask, (const bf16*)nb, bg, (bf16*)ctx, (bf16*)gate,
                                (bf16*)gated, lse, g, scale, ng);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

template <int D, int LP>
void launch_fwd_b(bool bias, const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx,
                  void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  if (bias) launch_fwd<D, LP, true>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd<D, LP, false>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
}

template <int D>
void launch_fwd_lp(bool bias, const void* qkvg, const float* mask, const void* nb, const float* bg,
                   void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  const int64_t L = g.L;
  if (L <= 64) launch_fwd_b<D, 64>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else if (L <= 128) launch_fwd_b<D, 128>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else if (L <= 192) launch_fwd_b<D, 192>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd_b<D, 256>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
}

}  // namespace

bool attn_fwd_tc_try(const void* qkvg, const float* mask, const void* nb, const float* bg,
                     void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, int dtype,
                     cudaStream_t s) {
  if (fwd_tc_disabled() || dtype != EVO_BF16) return false;
  // same L range as the tcgen05 backward (attention_tc_bwd.cu): a problem's
  // forward and backward must form the logits with the same operation order,
  // or a fully-masked row's recomputed logits could round one ulp (128 at the
  // -1e9 mask) away from the saved row max
  if (!(g.D == 16 || g.D == 32) || g.L > 256 || g.L < 65) return false;
  if ((g.ld % 8) != 0 || (((uintptr_t)qkvg) & 15) != 0) return false;
  if (((uintptr_t)ctx | (uintptr_t)gate | (uintptr_t)gated) & 15) return false;
  const bool bias = nb != nullptr;
  if (g.D == 16)
    launch_fwd_lp<16>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else
    launch_fwd_lp<32>(bias, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  return true;
}

}  // namespace evo
