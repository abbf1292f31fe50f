// Gated attention core forward for rows longer than 256 keys (the fine-tune
// shape F, L = 384 / 512, and the triangle-attention stress shape X,
// L = 1024) on the tcgen05 tensor cores -- the fused op of
// src/attention.py:118-174.  The L <= 256 kernel (attention_tc_fwd.cu) keeps
// a query tile's whole score row in TMEM; here the keys are processed in
// 256-key blocks:
//   per (batch b, key block kb): S = Q K_kb^T into TMEM, the two-pass softmax
//   of that block (block max m_kb, P = exp2(x - m_kb) packed into TMEM, block
//   sum l_kb), O_kb = P V_kb on the tensor core; then every thread merges its
//   row's O_kb into register accumulators
//       m = max(m, m_kb);  O = O 2^(m_old - m) + O_kb 2^(m_kb - m);  l likewise
//   and after the last block writes ctx = O / l, the gate, and (m, 1/l) -- the
//   same saved statistics as the single-block kernel, so the backward is
//   unchanged.  Logits use the fused order of the other tcgen05 kernels.
// The pair-bias tile of a key block is restaged per step (it is L2-resident);
// Q, K, the mask and the bias of the next step are prefetched as soon as the
// current S and pass 1 are done, V after P.V.
#include "common.cuh"
#include "reduce.cuh"
#include "attn_geom.cuh"
#include "tc_common.cuh"

namespace evo {

namespace {

using bf16 = __nv_bfloat16;

constexpr int KB = 256;  // keys per block

template <int D>
struct FwdKb {
  static constexpr int DC = D / 8;
  static constexpr int HALF = KB / 2;
  static constexpr int OC = HALF / 2;  // O columns (free after pass 2)
  static constexpr int TCOLS = 256;
  static constexpr int BROW = KB + 8;
  static constexpr int q = 0;
  static constexpr int k = 128 * D * 2;
  static constexpr int v = k + KB * D * 2;
  static constexpr int mb = v + KB * D * 2;
  static constexpr int bias = mb + KB * 4;
  static constexpr int ex = bias + 128 * BROW * 2;
  static constexpr int bar = ex + 512 * 4;
  static constexpr int slot = bar + 8;
  static constexpr int total = slot + 8;
};

__device__ __forceinline__ void st_zero16(void* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u); }

// Q rows of batch b, K rows / key mask / bias columns of key block kb
template <int D, bool BIAS>
__device__ __forceinline__ void kb_stage_qkmb(uint8_t* smem, const bf16* qkvg, const float* mask, const bf16* nb,
                                              const AttnGeom& g, int64_t b, int kb, int64_t h, int q0, int tid) {
  using F = FwdKb<D>;
  constexpr int DC = F::DC;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  bf16* sQ = reinterpret_cast<bf16*>(smem + F::q);
  bf16* sK = reinterpret_cast<bf16*>(smem + F::k);
  float* sMb = reinterpret_cast<float*>(smem + F::mb);
  for (int e = tid; e < 128 * DC; e += 256) {
    const int r = e / DC, c = e % DC;
    bf16* dst = sQ + ((r >> 3) * DC + c) * 64 + (r & 7) * 8;
    if (q0 + r < L) tc::cp_async16(dst, qkvg + g.tok(b, q0 + r) * g.ld + h * D + c * 8);
    else st_zero16(dst);
  }
  const int k0 = kb * KB;
  for (int e = tid; e < KB * DC; e += 256) {
    const int j = e / DC, c = e % DC;
    bf16* dst = sK + ((j >> 3) * DC + c) * 64 + (j & 7) * 8;
    if (k0 + j < L) tc::cp_async16(dst, qkvg + g.tok(b, k0 + j) * g.ld + HD + h * D + c * 8);
    else st_zero16(dst);
  }
  for (int j = tid; j < KB; j += 256)
    if (k0 + j < L) tc::cp_async4(sMb + j, mask + b * g.msb + (int64_t)(k0 + j) * g.msl);  // mask_to_bias later
    else sMb[j] = -INFINITY;
  if (BIAS) {
    bf16* sB = reinterpret_cast<bf16*>(smem + F::bias);
    const bool vec_ok = (L % 8) == 0;
    for (int e = tid; e < 128 * (KB / 8); e += 256) {
      const int r = e / (KB / 8), c = e % (KB / 8);
      bf16* dst = sB + r * F::BROW + c * 8;
      const int qq = q0 + r, kk = k0 + c * 8;
      if (qq < L && vec_ok && kk + 8 <= L) {
        tc::cp_async16(dst, nb + ((size_t)h * L + qq) * L + kk);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          dst[u] = (qq < L && kk + u < L) ? nb[((size_t)h * L + qq) * L + kk + u] : __float2bfloat16(0.f);
      }
    }
  }
}

template <int D>
__device__ __forceinline__ void kb_stage_v(uint8_t* smem, const bf16* qkvg, const AttnGeom& g, int64_t b, int kb,
                                           int64_t h, int tid) {
  using F = FwdKb<D>;
  constexpr int DC = F::DC;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  bf16* sV = reinterpret_cast<bf16*>(smem + F::v);
  const int k0 = kb * KB;
  for (int e = tid; e < KB * DC; e += 256) {
    const int j = e / DC, c = e % DC;
    bf16* dst = sV + ((j >> 3) * DC + c) * 64 + (j & 7) * 8;
    if (k0 + j < L) tc::cp_async16(dst, qkvg + g.tok(b, k0 + j) * g.ld + 2 * HD + h * D + c * 8);
    else st_zero16(dst);
  }
}

template <int D, bool BIAS>
__global__ void __launch_bounds__(256, 2) attn_fwd_tc_kb_kernel(
    const bf16* __restrict__ qkvg, const float* __restrict__ mask, const bf16* __restrict__ nb,
    const float* __restrict__ bg, bf16* __restrict__ ctx, bf16* __restrict__ gate,
    bf16* __restrict__ gated, float* __restrict__ lse, AttnGeom g, float scale, int NG, int nkb) {
  using F = FwdKb<D>;
  constexpr int DC = F::DC, HALF = F::HALF, NCH = HALF / 32;
  constexpr int DH = D / 2;  // output channels of this thread (its half of the head)
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
  const bf16* sV = reinterpret_cast<const bf16*>(smem + F::v);
  float* sMb = reinterpret_cast<float*>(smem + F::mb);

  if (warp == 0) tc::tmem_alloc<F::TCOLS>(slot);
  if (tid == 32) tc::mbar_init(bar, 1);
  if (b_lo < b_hi) {
    kb_stage_qkmb<D, BIAS>(smem, qkvg, mask, nb, g, b_lo, 0, h, q0, tid);
    kb_stage_v<D>(smem, qkvg, g, b_lo, 0, h, tid);
  }
  tc::cp_async_commit();
  uint32_t phase = 0;
  const int64_t cbase = h * D + half * DH;
  float bgv[DH];
#pragma unroll
  for (int k = 0; k < DH; ++k) bgv[k] = bg[cbase + k];

  for (int64_t b = b_lo; b < b_hi; ++b) {
    const int64_t tok = valid ? g.tok(b, i) : 0;
    float m_run = -INFINITY, l_run = 0.f, oacc[DH], gt[DH];
#pragma unroll
    for (int k = 0; k < DH; ++k) oacc[k] = 0.f, gt[k] = 0.f;
    for (int kb = 0; kb < nkb; ++kb) {
      const bool last_kb = kb == nkb - 1;
      const bool has_next = !last_kb || b + 1 < b_hi;
      const int64_t nb_b = last_kb ? b + 1 : b;
      const int nb_kb = last_kb ? 0 : kb + 1;
      uint4 graw[DH / 8];
      if (kb == 0 && valid) {
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

      // ---- S = Q K_kb^T  (M=128, N=256, K=D) ----
      if (warp == 0) {
        const uint32_t idesc = tc::idesc_bf16(128, KB, false, false);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t ad = tc::sdesc(tc::smem_u32(smem + F::q) + k * 256, 128, DC * 128);
          const uint64_t bd = tc::sdesc(tc::smem_u32(smem + F::k) + k * 256, 128, DC * 128);
          tc::mma_bf16_ss_w(tbase, ad, bd, idesc, k > 0 ? 1u : 0u);
        }
        tc::mma_commit_w(bar);
      }
      const int nvalid = L - kb * KB < KB ? L - kb * KB : KB;
      tc::mask_to_bias(sMb, KB, nvalid, tid, 256);
      __syncthreads();
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after();

      // ---- pass 1: logits (fused order), log2 domain, block row max ----
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
      const float m_kb = fmaxf(sEx[row], sEx[128 + row]);
      // Q, K, mask and bias are free (S done, pass 1 done): next step's
      if (has_next) {
        kb_stage_qkmb<D, BIAS>(smem, qkvg, mask, nb, g, nb_b, nb_kb, h, q0, tid);
        tc::cp_async_commit();
      }

      // ---- pass 2: P = exp2(logits - m_kb), packed bf16 pairs back into TMEM ----
      float2 sum2 = make_float2(0.f, 0.f);
      const float2 nm2 = make_float2(-m_kb, -m_kb);
#pragma unroll 1
      for (int ch = 0; ch < NCH; ++ch) {
        const int c0 = half * HALF + ch * 32;
        float v[32];
        tc::tmem_ld32(tl + c0, v);
        tc::wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 d = __fadd2_rn(make_float2(v[e], v[e + 1]), nm2);
          const float2 p = make_float2(tc::ex2(d.x), tc::ex2(d.y));
          sum2 = __fadd2_rn(sum2, p);
          pk[e / 2] = tc::pack_bf16(p.x, p.y);
        }
        tc::tmem_st16u(tl + half * HALF + ch * 16, pk);
      }
      tc::wait_st();
      sEx[256 + half * 128 + row] = sum2.x + sum2.y;
      tc::fence_before();
      __syncthreads();

      // ---- O_kb = P V_kb  (M=128, N=D, K=256), A from TMEM ----
      if (warp == 0) {
        tc::fence_after();
        const uint32_t idesc = tc::idesc_bf16(128, D, false, true);
#pragma unroll 4
        for (int k = 0; k < KB / 16; ++k) {
          const int key0 = 16 * k;
          const uint32_t pcol = (key0 / HALF) * HALF + (key0 % HALF) / 2;
          const uint64_t bd = tc::sdesc(tc::smem_u32(sV) + k * 2 * DC * 128, DC * 128, 128);
          tc::mma_bf16_ts_w(tbase + F::OC, tbase + pcol, bd, idesc, k > 0 ? 1u : 0u);
        }
        tc::mma_commit_w(bar);
      }
      if (kb == 0 && valid) {  // gate = sigmoid(g + bg) while the tensor core runs P.V
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
      const float l_kb = sEx[256 + row] + sEx[384 + row];
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after();
      if (has_next) {  // P.V is done with V
        kb_stage_v<D>(smem, qkvg, g, nb_b, nb_kb, h, tid);
        tc::cp_async_commit();
      }

      // ---- merge O_kb into the row's running (m, l, O) ----
      float o[DH];
      if constexpr (DH == 16) tc::tmem_ld16(tl + F::OC + half * DH, o);
      else tc::tmem_ld8(tl + F::OC + half * DH, o);
      tc::wait_ld();
      const float mn = fmaxf(m_run, m_kb);
      const float a = tc::ex2(m_run - mn), c = tc::ex2(m_kb - mn);  // m_run = -inf on the first block -> a = 0
#pragma unroll
      for (int k = 0; k < DH; ++k) oacc[k] = oacc[k] * a + o[k] * c;
      l_run = l_run * a + l_kb * c;
      m_run = mn;

      if (last_kb && valid) {  // ---- epilogue: normalise, gate, store ----
        const float invl = 1.0f / l_run;
        uint32_t pc[DH / 2], pg[DH / 2], pgd[DH / 2];
#pragma unroll
        for (int k = 0; k < DH; k += 2) {
          const float c0f = oacc[k] * invl, c1f = oacc[k + 1] * invl;
          pc[k / 2] = tc::pack_bf16(c0f, c1f);
          pg[k / 2] = tc::pack_bf16(gt[k], gt[k + 1]);
          pgd[k / 2] = tc::pack_bf16(c0f * gt[k], c1f * gt[k + 1]);
        }
#pragma unroll
        for (int k = 0; k < DH / 8; ++k) {
          reinterpret_cast<uint4*>(ctx + tok * HD + cbase)[k] = make_uint4(pc[4 * k], pc[4 * k + 1], pc[4 * k + 2], pc[4 * k + 3]);
          reinterpret_cast<uint4*>(gate + tok * HD + cbase)[k] = make_uint4(pg[4 * k], pg[4 * k + 1], pg[4 * k + 2], pg[4 * k + 3]);
          reinterpret_cast<uint4*>(gated + tok * HD + cbase)[k] =
              make_uint4(pgd[4 * k], pgd[4 * k + 1], pgd[4 * k + 2], pgd[4 * k + 3]);
        }
        if (half == 0) {
          lse[2 * ((b * g.H + h) * L + i)] = m_run;
          lse[2 * ((b * g.H + h) * L + i) + 1] = invl;
        }
      }
      tc::fence_before();
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<F::TCOLS>(*slot);
}

template <int D, bool BIAS>
void launch_fwd_kb(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx, void* gate,
                   void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  using F = FwdKb<D>;
  auto k = attn_fwd_tc_kb_kernel<D, BIAS>;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, F::total));
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  const int nqt = (int)((g.L + 127) / 128);
  const int nkb = (int)((g.L + KB - 1) / KB);
  int ng = (2 * num_sms()) / ((int)g.H * nqt);
  if (ng > g.B) ng = (int)g.B;
  if (ng < 1) ng = 1;
  dim3 grid((unsigned)ng, (unsigned)g.H, (unsigned)nqt);
  const float scale = (float)(1.0 / sqrt((double)D));
  k<<<grid, 256, F::total, s>>>((const bf16*)qkvg, mask, (const bf16*)nb, bg, (bf16*)ctx, (bf16*)gate,
                                (bf16*)gated, lse, g, scale, ng, nkb);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

}  // namespace

static bool kb_tc_disabled() {  // EVO_DISABLE_TC=1, as in attention_tc_bwd.cu
  static const bool v = [] {
    const char* e = getenv("EVO_DISABLE_TC");
    return e && e[0] == '1';
  }();
  return v;
}

// 256 < L <= 1024 (and a tcgen05-capable problem otherwise): the key-blocked
// kernel.  The bounds and the EVO_DISABLE_TC switch are the backward's
// (bwd_supported), so every problem's forward and backward take the same
// path and form the logits in the same operation order.
bool attn_fwd_tc_kb_try(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx,
                        void* gate, void* gated, float* lse, const AttnGeom& g, int dtype, cudaStream_t s) {
  if (kb_tc_disabled() || dtype != EVO_BF16 || g.L <= 256 || g.L > 1024) return false;
  if (!(g.D == 16 || g.D == 32)) return false;
  if ((g.ld % 8) != 0 || (((uintptr_t)qkvg) & 15) != 0) return false;
  if (((uintptr_t)ctx | (uintptr_t)gate | (uintptr_t)gated) & 15) return false;
  const bool bias = nb != nullptr;
  if (g.D == 16) {
    if (bias) launch_fwd_kb<16, true>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
    else launch_fwd_kb<16, false>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  } else {
    if (bias) launch_fwd_kb<32, true>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
    else launch_fwd_kb<32, false>(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  }
  return true;
}

}  // namespace evo
