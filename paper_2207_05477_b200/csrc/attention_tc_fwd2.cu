// Gated attention core forward, second generation: warp-specialised, TMA-fed
// and double-buffered in TMEM.  The fused op of src/attention.py:118-174
// (logits = q.k * c^-1/2 + (mask - 1) * 1e9 + nb, softmax, P.V, sigmoid gate).
//
// One CTA per SM (10 warps) owns (head h, query tile of 128 rows, batch group)
// and walks its batches with two tiles in flight:
//   warp 0      loader: Q, K, V and the gate pre-activations G of a batch by
//               TMA (a 3-D tensor map over the token-major qkvg buffer, so the
//               four Evoformer geometries are just strides) into a ring of
//               stages; the key mask as the rank-1 operand of the mask MMA and
//               a per-batch "every key masked" flag;
//   warp 1      MMA issuer: per batch, into TMEM region n & 1 (256 columns),
//                 S  = Q K^T              (D/16 MMAs, N = LP)
//                 S += e_0 (x) mbias      (1 MMA: (mask - 1) * 2^32 per key)
//               then, once the softmax has written P, O = P V with A read
//               from TMEM;
//   warps 2-5   softmax for even batches, warps 6-9 for odd ones: one thread
//               per query row holds the whole row.  Pass 1 forms
//               t = S c^-1/2 + nb (bias from a swizzled shared-memory tile,
//               the backward's exact inner operation) and its row max and
//               writes t back; pass 2 is one FFMA, one EX2, one add and a pack
//               per logit (P overwrites the consumed columns as bf16 pairs);
//               then the gate epilogue: [32 x D] tiles of ctx, gate and gated
//               staged in shared memory and written by TMA, (row max, 1/sum).
// A batch whose keys are all masked is flagged by the loader and gets the
// reference's uniform row (logits all equal to the mask constant), with the
// same saved statistics the backward (attention_tc_bwd.cu) recomputes from.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "attn_geom.cuh"
#include "common.cuh"
#include "reduce.cuh"
#include "tc_common.cuh"

namespace evo {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();  // gemm_tc.cu

#ifdef EVO_F2_TRACE
__device__ long long g_f2_trace[8192];
#define F2T(slot) do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0) g_f2_trace[(slot)] = clock64(); } while (0)
#else
#define F2T(slot) do {} while (0)
#endif

namespace {

using bf16 = __nv_bfloat16;

constexpr int F2_THREADS = 320;
constexpr float MASK_BIG = 4294967296.0f;  // 2^32: (m - 1) * 2^32 swamps every logit (bf16-exact)
constexpr float PAD_BIG = -1.0e30f;         // keys beyond L

template <int D, int LP, bool BIAS>
struct F2 {
  static constexpr int NKG = D / 8;               // 8-channel groups of a head
  static constexpr int Q_B = NKG * 128 * 16;      // TMA writes one 16-byte row per token
  static constexpr int K_B = NKG * LP * 16;
  static constexpr int M_B = (LP / 8) * 128 * 2;  // mask operand: j-group 0 (row 0 live), j-group 1 zero
  static constexpr int OFF_K = Q_B, OFF_V = Q_B + K_B, OFF_M = Q_B + 2 * K_B, OFF_G = OFF_M + M_B;
  static constexpr int STAGE = OFF_G + Q_B;       // + G, laid out like Q
  static constexpr int NSTG = (D == 16) ? 3 : 2;
  // D = 16: the bias joins S on the tensor core, S += 4 I_128 . nb (c^-1/2 = 1/4,
  // so the identity coefficient is exact); D = 32 adds it in the softmax
  static constexpr bool MMAB = BIAS && D == 16;
  static constexpr int OFF_BIAS = NSTG * STAGE;
  static constexpr int BIAS_B = BIAS ? 128 * LP * 2 : 0;
  static constexpr int OFF_ID = OFF_BIAS + BIAS_B;  // identity operand (zero padded, 7.5 KB used)
  static constexpr int OFF_AM = OFF_ID + (MMAB ? 8192 : 0);
  static constexpr int OUT_B = 32 * D * 2;        // one warp's [32 rows x D] output tile
  static constexpr int OFF_OUT = OFF_AM + 4096;   // 8 softmax warps x 2 staging tiles
  static constexpr int OFF_FLAG = OFF_OUT + 8 * 2 * OUT_B;
  static constexpr int OFF_BAR = OFF_FLAG + 64;
  static constexpr int NBAR = 2 * NSTG + 8;
  static constexpr int TOTAL = OFF_BAR + NBAR * 8 + 16 + 1024;  // + runtime 1 KB alignment
  static_assert(TOTAL <= 232448, "shared memory budget");
  static_assert(LP % 64 == 0 && LP <= 256 && LP / 2 + D <= LP, "tile");
};

// byte offset of (row r, 16-byte chunk c) in the [128 x LP] bf16 bias tile:
// the chunk index is XORed with r & 7 so a warp's 32 rows at one column hit
// 8 different bank groups
template <int LP>
__device__ __forceinline__ int bias_off(int r, int c) {
  return r * LP * 2 + ((c ^ (r & 7)) << 4);
}

__device__ __forceinline__ void tma_load3(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_store3(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 2^x on the MUFU for all lanes of a packed pair
__device__ __forceinline__ float2 ex2x2(float2 x) { return make_float2(tc::ex2(x.x), tc::ex2(x.y)); }

template <int D, int LP, bool BIAS>
__global__ void __launch_bounds__(F2_THREADS, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmc,
                        const __grid_constant__ CUtensorMap tmg, const __grid_constant__ CUtensorMap tmgd,
                        const bf16* __restrict__ qkvg,
                        const float* __restrict__ mask, const bf16* __restrict__ nb, const float* __restrict__ bg,
                        bf16* __restrict__ ctx, bf16* __restrict__ gate, bf16* __restrict__ gated,
                        float* __restrict__ lse, AttnGeom g, float scale, int NG) {
  using F = F2<D, LP, BIAS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F::OFF_BAR);
  uint64_t* empty = full + F::NSTG;
  uint64_t* sfull = empty + F::NSTG;  // [2] MMA -> softmax: S of region r
  uint64_t* pready = sfull + 2;       // [2] softmax -> MMA: P of region r written
  uint64_t* ofull = pready + 2;       // [2] MMA -> softmax: O of region r
  uint64_t* tfree = ofull + 2;        // [2] softmax -> MMA: region r read out
  uint32_t* slot = reinterpret_cast<uint32_t*>(tfree + 2);
  int* flag = reinterpret_cast<int*>(smem + F::OFF_FLAG);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x;
  const int64_t h = blockIdx.y;
  const int q0 = blockIdx.z * 128;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  const int64_t b_lo = (g.B * grp) / NG, b_hi = (g.B * (grp + 1)) / NG;
  const int nbt = (int)(b_hi - b_lo);

  // ---- one-time setup: constant operands, bias tile, barriers, TMEM ----
  {
    // zero the mask operands of every stage, the identity regions and A_mask
    for (int s = 0; s < F::NSTG; ++s) {
      uint4* mz = reinterpret_cast<uint4*>(smem + s * F::STAGE + F::OFF_M);
      for (int e = tid; e < F::M_B / 16; e += F2_THREADS) mz[e] = make_uint4(0u, 0u, 0u, 0u);
    }
    uint4* z = reinterpret_cast<uint4*>(smem + F::OFF_ID);
    for (int e = tid; e < (F::OFF_AM + 4096 - F::OFF_ID) / 16; e += F2_THREADS) z[e] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (BIAS) {
    // nb[h, q0 + r, :] -> swizzled row-major tile (zero beyond L)
    constexpr int CPR = LP / 8;
    const bool vec_ok = (L % 8) == 0;
    for (int e = tid; e < 128 * CPR; e += F2_THREADS) {
      const int r = e / CPR, c = e % CPR;
      // MMA operand: MN-major core matrices, (key group c, query group r/8) at
      // (r/8) * LP/8 * 128 + c * 128, query r % 8 at +16 (r % 8); softmax: swizzled rows
      const int off = F::MMAB ? (r >> 3) * CPR * 128 + c * 128 + (r & 7) * 16 : bias_off<LP>(r, c);
      bf16* dst = reinterpret_cast<bf16*>(smem + F::OFF_BIAS + off);
      const int qq = q0 + r, k = c * 8;
      if (qq < L && vec_ok && k + 8 <= L) {
        tc::cp_async16(dst, nb + ((size_t)h * L + qq) * L + k);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          dst[u] = (qq < L && k + u < L) ? nb[((size_t)h * L + qq) * L + k + u] : __float2bfloat16(0.f);
      }
    }
  }
  tc::cp_async_commit();
  __syncthreads();  // zero fills before the constant entries below
  if (tid < 128) {
    // A_mask [128 x 16] K-major: column 0 ones (core (g, 0) at 256 g, row r at +16 r)
    const int r = tid;
    *reinterpret_cast<bf16*>(smem + F::OFF_AM + (r >> 3) * 256 + (r & 7) * 16) = __float2bfloat16(1.0f);
  }
  if (F::MMAB && tid < 16) {
    // identity operand for query chunk c: base OFF_ID + 3584 - 512 c (LBO 128,
    // SBO 256) puts its two diagonal cores at OFF_ID + 3584 and + 3968
    const int r = tid & 7, which = tid >> 3;
    *reinterpret_cast<bf16*>(smem + F::OFF_ID + 3584 + which * 384 + r * 16 + r * 2) = __float2bfloat16(4.0f);
  }
  if (tid == 0) {
    for (int s = 0; s < F::NSTG; ++s) {
      tc::mbar_init(&full[s], 2);  // TMA (expect_tx) + mask operand
      tc::mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < 2; ++r) {
      tc::mbar_init(&sfull[r], 1);
      tc::mbar_init(&pready[r], 4);
      tc::mbar_init(&ofull[r], 1);
      tc::mbar_init(&tfree[r], 4);
    }
  }
  if (warp == 1) tc::tmem_alloc<512>(slot);
  tc::cp_async_wait0();
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;

  if (warp == 0) {
    // ======================= loader =======================
    for (int n = 0; n < nbt; ++n) {
      const int s = n % F::NSTG;
      const int64_t b = b_lo + n;
      uint8_t* st = smem + s * F::STAGE;
      tc::mbar_wait(&empty[s], ((n / F::NSTG) & 1) ^ 1);
      if (lane == 0) {
        expect_tx(&full[s], 2 * F::Q_B + 2 * F::K_B);
        const int cq = (int)(h * D), ck = (int)(HD + h * D), cv = (int)(2 * HD + h * D), cg = (int)(3 * HD + h * D);
#pragma unroll
        for (int kq = 0; kq < F::NKG; ++kq) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            tma_load3(&tmq, st + kq * 2048 + i * 1024, &full[s], cq + 8 * kq, q0 + 64 * i, (int)b);
            tma_load3(&tmq, st + F::OFF_G + kq * 2048 + i * 1024, &full[s], cg + 8 * kq, q0 + 64 * i, (int)b);
          }
#pragma unroll
          for (int i = 0; i < LP / 64; ++i) {
            tma_load3(&tmq, st + F::OFF_K + kq * LP * 16 + i * 1024, &full[s], ck + 8 * kq, 64 * i, (int)b);
            tma_load3(&tmq, st + F::OFF_V + kq * LP * 16 + i * 1024, &full[s], cv + 8 * kq, 64 * i, (int)b);
          }
        }
      }
      // key mask -> row 0 of the mask operand's cores (8 keys per lane)
      bool live = false;
      if (lane * 8 < LP) {
        float mv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = lane * 8 + u;
          const float m = k < L ? __ldg(mask + b * g.msb + k * g.msl) : 0.f;
          live |= (k < L && m != 0.f);
          mv[u] = k < L ? (m - 1.0f) * MASK_BIG : PAD_BIG;
        }
        uint4 w = make_uint4(tc::pack_bf16(mv[0], mv[1]), tc::pack_bf16(mv[2], mv[3]), tc::pack_bf16(mv[4], mv[5]),
                             tc::pack_bf16(mv[6], mv[7]));
        *reinterpret_cast<uint4*>(st + F::OFF_M + lane * 128) = w;
      }
      const bool any_live = __any_sync(0xffffffffu, live);
      if (lane == 0) flag[s] = any_live ? 0 : 1;
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[s]);
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    const uint32_t s0 = tc::smem_u32(smem);
    const uint32_t id_s = tc::idesc_bf16(128, LP, false, false);
    const uint32_t id_m = tc::idesc_bf16(128, LP, false, true);
    const uint32_t id_o = tc::idesc_bf16(128, D, false, true);
    auto issue_s = [&](int n) {
      const int s = n % F::NSTG;
      const uint32_t st = s0 + s * F::STAGE;
      const uint32_t tm = tbase + (uint32_t)((n & 1) * 256);
      tc::mbar_wait(&full[s], (n / F::NSTG) & 1);
      tc::fence_after();
#pragma unroll
      for (int m = 0; m < D / 16; ++m)
        tc::mma_bf16_ss_w(tm, tc::sdesc(st + m * 2 * 2048, 2048, 128),
                          tc::sdesc(st + F::OFF_K + m * 2 * LP * 16, LP * 16, 128), id_s, m > 0 ? 1u : 0u);
      tc::mma_bf16_ss_w(tm, tc::sdesc(s0 + F::OFF_AM, 128, 256), tc::sdesc(st + F::OFF_M, (LP / 8) * 128, 128), id_m,
                        1u);
      if constexpr (F::MMAB) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          tc::mma_bf16_ss_w(tm, tc::sdesc(s0 + F::OFF_ID + 3584 - 512 * c, 128, 256),
                            tc::sdesc(s0 + F::OFF_BIAS + 2 * c * (LP / 8) * 128, (LP / 8) * 128, 128), id_m, 1u);
      }
      tc::mma_commit_w(&sfull[n & 1]);
    };
    if (nbt > 0) issue_s(0);
    if (nbt > 1) issue_s(1);
    for (int n = 0; n < nbt; ++n) {
      const int r = n & 1, s = n % F::NSTG;
      const uint32_t st = s0 + s * F::STAGE;
      const uint32_t tm = tbase + (uint32_t)(r * 256);
      F2T(2048 + 8 * n + 0);
      tc::mbar_wait(&pready[r], (n >> 1) & 1);
      F2T(2048 + 8 * n + 1);
      tc::fence_after();
#pragma unroll
      for (int m = 0; m < LP / 16; ++m)
        tc::mma_bf16_ts_w(tm + LP / 2, tm + 8 * m, tc::sdesc(st + F::OFF_V + m * 256, 128, LP * 16), id_o,
                          m > 0 ? 1u : 0u);
      tc::mma_commit_w(&ofull[r]);
      tc::mma_commit_w(&empty[s]);
      if (n + 2 < nbt) {
        tc::mbar_wait(&tfree[r], (n >> 1) & 1);
        F2T(2048 + 8 * n + 2);
        tc::fence_after();
        issue_s(n + 2);
        F2T(2048 + 8 * n + 3);
      }
    }
  } else {
    // ======================= softmax + epilogue =======================
    const int wg = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int i = q0 + row;
    const bool valid = i < L;
    const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(wg * 256);
    const int64_t cb = h * D;
    const float2 sc2 = make_float2(scale, scale), l2e = make_float2(tc::LOG2E_F, tc::LOG2E_F);
    const float cexp = scale * tc::LOG2E_F;  // the backward's constant (attention_tc_bwd.cu)
    const float2 ce2 = make_float2(cexp, cexp);
    const uint8_t* brow = smem + F::OFF_BIAS + row * LP * 2;
    float bmax = 0.f;  // max of this query row's bias (the tile is the same for every batch)
    if (BIAS && !F::MMAB) {
      bmax = -INFINITY;
      const int nk = L < LP ? L : LP;
      for (int k = 0; k < nk; ++k) {
        const bf16 v = *reinterpret_cast<const bf16*>(brow + (((k >> 3) ^ (row & 7)) << 4) + (k & 7) * 2);
        bmax = fmaxf(bmax, __bfloat162float(v));
      }
    }
    for (int n = wg; n < nbt; n += 2) {
      const int64_t b = b_lo + n;
      const int s = n % F::NSTG;
      if (quarter == 2) F2T(16 * n + 0);
      tc::mbar_wait(&sfull[wg], (n >> 1) & 1);
      if (quarter == 2) F2T(16 * n + 1);
      tc::fence_after();
      const bool uniform = flag[s] != 0;
      float mx2;  // row max of the log2-domain logits (the backward's m)
      float2 sum2 = make_float2(0.f, 0.f);
      if (!uniform) {
        // ---- pass 1: row max of S (raw q.k; the mask MMA only lowers masked keys) ----
        float va[32], vb[32];
        float2 mm = make_float2(-INFINITY, -INFINITY);
        auto smax = [&](const float (&x)[32]) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            mm = make_float2(fmaxf(mm.x, fmaxf(x[e], x[e + 1])), fmaxf(mm.y, fmaxf(x[e + 2], x[e + 3])));
        };
        tc::tmem_ld32(tl, va);
#pragma unroll 1
        for (int c = 0; c < LP; c += 64) {
          tc::wait_ld();
          tc::tmem_ld32(tl + c + 32, vb);
          smax(va);
          tc::wait_ld();
          if (c + 64 < LP) tc::tmem_ld32(tl + c + 64, va);
          smax(vb);
        }
        // m = (max_k s_k c^-1/2 + max_k nb_k) log2 e bounds every logit from
        // above (a stabiliser only: P and the sum share it, and the backward
        // recomputes P from the saved (m, 1/sum))
        mx2 = F::MMAB ? fmaxf(mm.x, mm.y) * cexp : fmaf(fmaxf(mm.x, mm.y), scale, bmax) * tc::LOG2E_F;
        if (quarter == 2) F2T(16 * n + 2);
        // ---- pass 2: t = s c^-1/2 + nb (the backward's inner FFMA), P = 2^(t log2e - m),
        // packed bf16 pairs over the consumed columns ----
        const float2 nm = make_float2(-mx2, -mx2);
        auto expo = [&](const float (&x)[32], int c) {
          constexpr bool SB = BIAS && !F::MMAB;  // bias added here
          uint32_t braw[16];
          if (SB) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 u = *reinterpret_cast<const uint4*>(brow + (((c >> 3) + k) ^ (row & 7)) * 16);
              braw[4 * k] = u.x, braw[4 * k + 1] = u.y, braw[4 * k + 2] = u.z, braw[4 * k + 3] = u.w;
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 nbv = SB ? tc::bf16x2_f2(braw[e / 2]) : make_float2(0.f, 0.f);
            float2 p;
            if constexpr (F::MMAB) {  // S = s + 4 nb + mask: x = S c^-1/2 log2e - m in one FFMA
              p = ex2x2(__ffma2_rn(make_float2(x[e], x[e + 1]), ce2, nm));
            } else {
              const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, nbv);
              p = ex2x2(__ffma2_rn(t, l2e, nm));
            }
            sum2 = __fadd2_rn(sum2, p);
            pk[e / 2] = tc::pack_bf16(p.x, p.y);
          }
          tc::tmem_st16u(tl + c / 2, pk);
        };
        tc::tmem_ld32(tl, va);
#pragma unroll 1
        for (int c = 0; c < LP; c += 64) {
          tc::wait_ld();
          tc::tmem_ld32(tl + c + 32, vb);
          expo(va, c);
          tc::wait_ld();
          if (c + 64 < LP) tc::tmem_ld32(tl + c + 64, va);
          expo(vb, c + 32);
        }
      } else {
        // every key masked: the reference's logits all round onto the mask
        // constant, so the row is uniform over the L keys
        mx2 = (0.0f - 1.0f) * tc::MASK_BIAS_L2;
        const int nkeys = L;
#pragma unroll 1
        for (int c = 0; c < LP; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float p0 = (c + e < nkeys) ? 1.f : 0.f, p1 = (c + e + 1 < nkeys) ? 1.f : 0.f;
            sum2.x += p0;
            sum2.y += p1;
            pk[e / 2] = tc::pack_bf16(p0, p1);
          }
          tc::tmem_st16u(tl + c / 2, pk);
        }
      }
      // the gate pre-activations are read out of the stage before P is handed
      // over: the stage is recycled once P.V has completed
      uint4 graw[D / 8];
#pragma unroll
      for (int k = 0; k < D / 8; ++k)
        graw[k] = *reinterpret_cast<const uint4*>(smem + s * F::STAGE + F::OFF_G + row * 16 + k * 2048);
      tc::wait_st();
      if (quarter == 2) F2T(16 * n + 3);
      tc::fence_before();
      tc::mbar_arrive_warp(&pready[wg]);

      // gate = sigmoid(g + bg) while the tensor core runs P.V
      float gt[D];
      {
        float bgv[D];  // gate bias (the same addresses for every thread: broadcast loads)
#pragma unroll
        for (int k = 0; k < D / 4; ++k) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(bg + cb) + k);
          bgv[4 * k] = t.x, bgv[4 * k + 1] = t.y, bgv[4 * k + 2] = t.z, bgv[4 * k + 3] = t.w;
        }
#pragma unroll
        for (int k = 0; k < D / 8; ++k) {
          const uint32_t w4[4] = {graw[k].x, graw[k].y, graw[k].z, graw[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 gp = tc::bf16x2_f2(w4[q]);
            gt[8 * k + 2 * q] = __fdividef(1.0f, 1.0f + __expf(-(gp.x + bgv[8 * k + 2 * q])));
            gt[8 * k + 2 * q + 1] = __fdividef(1.0f, 1.0f + __expf(-(gp.y + bgv[8 * k + 2 * q + 1])));
          }
        }
      }
      const float invl = 1.0f / (sum2.x + sum2.y);
      tc::mbar_wait(&ofull[wg], (n >> 1) & 1);
      tc::fence_after();
      float o[D];
      if constexpr (D == 32) {
        tc::tmem_ld32(tl + LP / 2, o);
      } else {
        tc::tmem_ld16(tl + LP / 2, o);
      }
      tc::wait_ld();
      tc::fence_before();
      tc::mbar_arrive_warp(&tfree[wg]);
      // ---- epilogue: [32 rows x D] tiles of ctx, gate, gated through two
      // staging buffers per warp, written by TMA (rows beyond L are clipped) ----
      uint8_t* ob = smem + F::OFF_OUT + (warp - 2) * 2 * F::OUT_B;
      uint8_t* myrow0 = ob + lane * D * 2;
      uint8_t* myrow1 = ob + F::OUT_B + lane * D * 2;
      if (lane == 0) bulk_wait_read<0>();  // the previous tile's stores have read both buffers
      __syncwarp();
      uint32_t pc[D / 2], pg[D / 2];
#pragma unroll
      for (int k = 0; k < D; k += 2) {
        o[k] *= invl;
        o[k + 1] *= invl;
        pc[k / 2] = tc::pack_bf16(o[k], o[k + 1]);
        pg[k / 2] = tc::pack_bf16(gt[k], gt[k + 1]);
      }
#pragma unroll
      for (int k = 0; k < D / 8; ++k) {
        reinterpret_cast<uint4*>(myrow0)[k] = make_uint4(pc[4 * k], pc[4 * k + 1], pc[4 * k + 2], pc[4 * k + 3]);
        reinterpret_cast<uint4*>(myrow1)[k] = make_uint4(pg[4 * k], pg[4 * k + 1], pg[4 * k + 2], pg[4 * k + 3]);
      }
      tc::fence_proxy_async();
      __syncwarp();
      const int r0 = q0 + quarter * 32;
      if (lane == 0) {
        tma_store3(&tmc, ob, (int)cb, r0, (int)b);
        bulk_commit();
        tma_store3(&tmg, ob + F::OUT_B, (int)cb, r0, (int)b);
        bulk_commit();
        bulk_wait_read<1>();  // ctx has been read out of buffer 0
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < D; k += 2) pc[k / 2] = tc::pack_bf16(o[k] * gt[k], o[k + 1] * gt[k + 1]);
#pragma unroll
      for (int k = 0; k < D / 8; ++k)
        reinterpret_cast<uint4*>(myrow0)[k] = make_uint4(pc[4 * k], pc[4 * k + 1], pc[4 * k + 2], pc[4 * k + 3]);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store3(&tmgd, ob, (int)cb, r0, (int)b);
        bulk_commit();
      }
      if (valid) *reinterpret_cast<float2*>(lse + 2 * ((b * g.H + h) * L + i)) = make_float2(mx2, invl);
      if (quarter == 2) F2T(16 * n + 6);
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_all();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(tbase);
}

// 3-D map over qkvg viewed as [batch][position][channel]: channel stride 1,
// position stride sl * ld, batch stride sb * ld (elements); box 8 x 64 x 1
bool qkvg_map(CUtensorMap* m, const void* qkvg, const AttnGeom& g) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const int64_t es = 2;
  const int64_t ps = g.sl * g.ld * es, bs = g.sb * g.ld * es;
  if (((uintptr_t)qkvg & 15) || ps % 16 || bs % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)g.ld, (cuuint64_t)g.L, (cuuint64_t)g.B};
  cuuint64_t strides[2] = {(cuuint64_t)ps, (cuuint64_t)bs};
  cuuint32_t box[3] = {8, 64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(qkvg), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [batch][position][H*D] view of a token-major output (ctx / gate / gated):
// box D x 32 x 1 (one warp's rows)
bool out_map(CUtensorMap* m, const void* base, const AttnGeom& g) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const int64_t HD = g.H * g.D, es = 2;
  const int64_t ps = g.sl * HD * es, bs = g.sb * HD * es;
  if (((uintptr_t)base & 15) || ps % 16 || bs % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)g.L, (cuuint64_t)g.B};
  cuuint64_t strides[2] = {(cuuint64_t)ps, (cuuint64_t)bs};
  cuuint32_t box[3] = {(cuuint32_t)g.D, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct OutMaps {
  CUtensorMap c, g, gd;
};

template <int D, int LP, bool BIAS>
void launch_fwd2(const CUtensorMap& tm, const OutMaps& om, const void* qkvg, const float* mask, const void* nb, const float* bg,
                 void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, cudaStream_t s) {
  using F = F2<D, LP, BIAS>;
  auto k = attn_fwd_tc2_kernel<D, LP, BIAS>;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, F::TOTAL));
    attr = true;
  }
  const int nqt = (int)((g.L + 127) / 128);
  int ng = num_sms() / ((int)g.H * nqt);
  if (ng > g.B) ng = (int)g.B;
  if (ng < 1) ng = 1;
  const float scale = (float)(1.0 / sqrt((double)D));
  dim3 grid((unsigned)ng, (unsigned)g.H, (unsigned)nqt);
  k<<<grid, F2_THREADS, F::TOTAL, s>>>(tm, om.c, om.g, om.gd, (const bf16*)qkvg, mask, (const bf16*)nb, bg, (bf16*)ctx, (bf16*)gate,
                                       (bf16*)gated, lse, g, scale, ng);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

template <int D, int LP>
void launch_fwd2_b(bool bias, const CUtensorMap& tm, const OutMaps& om, const void* qkvg, const float* mask, const void* nb,
                   const float* bg, void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g,
                   cudaStream_t s) {
  if (bias) launch_fwd2<D, LP, true>(tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd2<D, LP, false>(tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
}

template <int D>
void launch_fwd2_lp(bool bias, const CUtensorMap& tm, const OutMaps& om, const void* qkvg, const float* mask, const void* nb,
                    const float* bg, void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g,
                    cudaStream_t s) {
  if (g.L <= 128) launch_fwd2_b<D, 128>(bias, tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else if (g.L <= 192) launch_fwd2_b<D, 192>(bias, tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd2_b<D, 256>(bias, tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
}

bool fwd2_disabled() {  // EVO_ATTN_FWD2=0: first-generation kernel (A/B measurements); EVO_DISABLE_TC=1
  static const bool v = [] {
    const char* e = getenv("EVO_ATTN_FWD2");
    const char* t = getenv("EVO_DISABLE_TC");
    return (e && e[0] == '0') || (t && t[0] == '1');
  }();
  return v;
}

}  // namespace

// Same coverage as the first-generation kernel (65 <= L <= 256, D = 16 / 32,
// bf16): a problem's forward and backward must agree on which logits path
// formed the saved statistics' row max.
bool attn_fwd_tc2_try(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx, void* gate,
                      void* gated, float* lse, const AttnGeom& g, int dtype, cudaStream_t s) {
  if (fwd2_disabled() || dtype != EVO_BF16) return false;
  if (!(g.D == 16 || g.D == 32) || g.L > 256 || g.L < 65) return false;
  if (g.B > (1ll << 31) || (g.ld % 8) != 0) return false;
  if (((uintptr_t)ctx | (uintptr_t)gate | (uintptr_t)gated | (uintptr_t)lse) & 15) return false;
  CUtensorMap tm;
  OutMaps om;
  if (!qkvg_map(&tm, qkvg, g) || !out_map(&om.c, ctx, g) || !out_map(&om.g, gate, g) || !out_map(&om.gd, gated, g))
    return false;
  const bool bias = nb != nullptr;
  if (g.D == 16) launch_fwd2_lp<16>(bias, tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  else launch_fwd2_lp<32>(bias, tm, om, qkvg, mask, nb, bg, ctx, gate, gated, lse, g, s);
  return true;
}

}  // namespace evo

#ifdef EVO_F2_TRACE
extern "C" int evo_f2_trace_read(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, evo::g_f2_trace, sizeof(long long) * n);
}
#endif
