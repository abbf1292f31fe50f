// Gated attention core backward on the 5th-generation tensor cores (tcgen05 +
// TMEM), bf16 storage / fp32 accumulation -- the closure of
// src/attention.py:178-221.  Forward: attention_tc_fwd.cu.
//
// One CTA per (batch group, head, query tile), 16 warps, looping over the
// batches of its group with double-buffered cp.async staging; the pair-bias
// tile of the CTA's query rows is the same for every batch, so it is staged
// into shared memory once:
//   per 64-key sub-chunk: S = Q K^T and dP = dO V^T on the tensor core,
//   P = exp2(logits*log2e - m) / l and dS = P (dP - D) from TMEM, the bias
//   gradient accumulated in TMEM across the whole batch group (deterministic,
//   no atomics), P / dS written to shared memory;
//   per 128-key chunk: dQ += dS K, dK = dS^T Q, dV = P^T dO on the tensor
//   core (MN-major operand descriptors read the same shared tiles
//   transposed), drained to HBM.
// With two query tiles (L <= 256) both add their dK/dV into slices the prep
// kernel zeroed, by bf16x8 reduction stores: two addends onto zero give the
// same bits in either arrival order.  More query tiles or key windows write
// partials that a combine kernel adds in fixed order.
#include "common.cuh"
#include "reduce.cuh"
#include "attn_geom.cuh"
#include "tc_common.cuh"

namespace evo {

#ifdef EVO_BWD_TRACE
// phase timestamps of CTA (0, 0, 0): softmax warps 0 / 15 and the MMA warp
// (tools/bwd_trace.py; a -DEVO_BWD_TRACE build from tools/build_trace.py --
// its extra registers spill, so read phases relative to each other)
__device__ long long g_bwd_trace[8192];
#define BT(base, slot) do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0) g_bwd_trace[(base) + (slot)] = clock64(); } while (0)
#else
#define BT(base, slot) do {} while (0)
#endif

bool colsum_vec(void* x, int xdt, int64_t ldx, const void* h, void* y, int ydt, float* out,
                int accumulate, void* ws, int64_t rows, int64_t C, int mode, cudaStream_t s);

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void st_zero16(void* p) {
  *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
}

__device__ __forceinline__ void bf16x8_to_f(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

template <int LP>
struct TmemCols {
  static constexpr int value = LP <= 32 ? 32 : (LP <= 64 ? 64 : (LP <= 128 ? 128 : 256));
};

// ============================================================================
// ============================================================================
// backward
// ============================================================================

template <int D, int LP>
struct BwdSmem {
  static constexpr int STAGE = 2 * 128 * D * 2 + 2 * LP * D * 2 + LP * 4;  // Q, dO, K, V, Mb
  static constexpr int q = 0;                        // + stage offset
  static constexpr int o = 128 * D * 2;
  static constexpr int k = o + 128 * D * 2;
  static constexpr int v = k + LP * D * 2;
  static constexpr int mb = v + LP * D * 2;
  static constexpr int p = 2 * STAGE;                // [128 x 128] bf16 (one 128-key chunk)
  static constexpr int ds = p + 128 * 128 * 2;
  static constexpr int bar = ds + 128 * 128 * 2;
  static constexpr int bias = bar + 128;             // [128 x LP] bf16, 16-B chunks XOR-swizzled by row
  static constexpr int total = bias + 128 * LP * 2;
};

// byte offset of (row r, 16-B chunk c) in the swizzled bias tile: the chunk
// index is XORed with r & 7, so the 32 rows a warp reads at one column land in
// 8 different bank groups (no padding needed, which keeps the D=32 / L=256
// variant double-buffered inside 227 KB)
template <int LP>
__device__ __forceinline__ int bias_off(int r, int c) {
  return r * LP * 2 + ((c ^ (r & 7)) << 4);
}

// the CTA's bias rows nb[h, q0 + r, :] -> smem [128][LP] (zero padded)
template <int LP>
__device__ __forceinline__ void stage_bias_tile(uint8_t* sB, const bf16* nb, int64_t h, int q0, int k0, int L,
                                                int tid, int nthreads) {
  constexpr int CPR = LP / 8;
  const bool vec_ok = (L % 8) == 0;
  for (int e = tid; e < 128 * CPR; e += nthreads) {
    const int r = e / CPR, c = e % CPR;
    bf16* dst = reinterpret_cast<bf16*>(sB + bias_off<LP>(r, c));
    const int q = q0 + r, kk = k0 + c * 8;
    if (q < L && vec_ok && kk + 8 <= L) {
      tc::cp_async16(dst, nb + ((size_t)h * L + q) * L + kk);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        dst[u] = (q < L && kk + u < L) ? nb[((size_t)h * L + q) * L + kk + u] : __float2bfloat16(0.f);
    }
  }
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  tc::tmem_st16u(taddr, reinterpret_cast<const uint32_t(&)[16]>(v));
}
__device__ __forceinline__ void tmem_zero(uint32_t taddr) {
  float z[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) z[e] = 0.f;
  tmem_st16(taddr, z);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// 8 bf16 added into global memory at L2 (round-to-nearest).  Used only where
// exactly two addends meet a zeroed destination, so the result does not depend
// on their arrival order (0 + a + b == 0 + b + a: fp addition commutes)
__device__ __forceinline__ void red_add_bf16x8(void* p, const uint4& v) {
  asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

template <int D, int LP>
__device__ __forceinline__ void bwd_stage(uint8_t* st, const bf16* qkvg, const bf16* dctx,
                                          const float* mbias, const AttnGeom& g, int64_t b,
                                          int64_t h, int q0, int tid, int k0 = 0) {
  using SM = BwdSmem<D, LP>;
  constexpr int DC = D / 8;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  bf16* sQ = reinterpret_cast<bf16*>(st + SM::q);
  bf16* sO = reinterpret_cast<bf16*>(st + SM::o);
  bf16* sK = reinterpret_cast<bf16*>(st + SM::k);
  bf16* sV = reinterpret_cast<bf16*>(st + SM::v);
  float* sMb = reinterpret_cast<float*>(st + SM::mb);
  for (int e = tid; e < 128 * DC; e += 512) {
    const int r = e / DC, c = e % DC;
    const int off = ((r >> 3) * DC + c) * 64 + (r & 7) * 8;
    if (q0 + r < L) {
      const int64_t t = g.tok(b, q0 + r);
      tc::cp_async16(sQ + off, qkvg + t * g.ld + h * D + c * 8);
      tc::cp_async16(sO + off, dctx + t * HD + h * D + c * 8);
    } else {
      st_zero16(sQ + off);
      st_zero16(sO + off);
    }
  }
  for (int e = tid; e < LP * DC; e += 512) {
    const int j = e / DC, c = e % DC;
    const int off = ((j >> 3) * DC + c) * 64 + (j & 7) * 8;
    if (k0 + j < L) {
      const bf16* src = qkvg + g.tok(b, k0 + j) * g.ld + HD + h * D + c * 8;
      tc::cp_async16(sK + off, src);
      tc::cp_async16(sV + off, src + HD);
    } else {
      st_zero16(sK + off);
      st_zero16(sV + off);
    }
  }
  for (int j = tid; j < LP; j += 512)
    if (k0 + j < L)
      tc::cp_async4(sMb + j, mbias + b * L + k0 + j);  // precomputed (m - 1) * 1e9 * log2(e)
    else
      sMb[j] = -INFINITY;
}

// advance a shared-memory descriptor by a byte offset (the start-address
// field holds addr >> 4 in its low 14 bits; shared addresses stay < 256 KB)
__device__ __forceinline__ uint64_t dadd(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }

// S = Q K^T and dP = dO V^T for the 64 keys at koff (one elected lane of the
// calling warp issues; completion arrives on bar)
template <int D>
__device__ __forceinline__ void issue_sdp(uint32_t st, int koff, uint32_t tbase, uint32_t c_s, uint32_t c_dp,
                                          uint64_t* bar, int q_off, int o_off, int k_off, int v_off) {
  constexpr int DC = D / 8;
  const uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
  const uint64_t aq = tc::sdesc(st + q_off, 128, DC * 128);
  const uint64_t ao = tc::sdesc(st + o_off, 128, DC * 128);
  const uint64_t bk = tc::sdesc(st + k_off + (koff / 8) * DC * 128, 128, DC * 128);
  const uint64_t bv = tc::sdesc(st + v_off + (koff / 8) * DC * 128, 128, DC * 128);
#pragma unroll
  for (int k = 0; k < D / 16; ++k) {
    tc::mma_bf16_ss_w(tbase + c_s, dadd(aq, k * 256), dadd(bk, k * 256), idesc, k > 0 ? 1u : 0u);
    tc::mma_bf16_ss_w(tbase + c_dp, dadd(ao, k * 256), dadd(bv, k * 256), idesc, k > 0 ? 1u : 0u);
  }
  tc::mma_commit_w(bar);
}

// Warp-specialised, software-pipelined backward (17 warps, one CTA per SM).
//
// Warp 16 issues every tcgen05.mma; warps 0..15 run the softmax backward
// (TMEM lane quarter = warp & 3, 16-key column group = warp >> 2).  They talk
// through four mbarriers only -- no CTA-wide barrier inside the batch loop:
//   barS    (MMA -> softmax)  S/dP of sub-chunk j are in TMEM
//   barSf   (softmax -> MMA)  all 16 warps copied S/dP(j) out (and, at a batch
//                              boundary, the next batch's staging landed):
//                              the MMA warp issues S/dP(j+1) into the same
//                              columns, overlapping the softmax of j
//   barPdS  (softmax -> MMA)  P/dS of a 128-key chunk are in shared memory and
//                              the previous chunk's dK/dV/dQ are drained
//   barKV   (MMA -> softmax)  dQ/dK/dV of the chunk are complete
// The dQ/dK/dV MMAs of chunk c run while the softmax warps compute the first
// sub-chunk of c+1; they are drained (and batch b-1's staging buffer is
// refilled with batch b+1 by cp.async) just before P/dS of c+1 are stored.
// The bias gradient is accumulated in TMEM across the whole batch group.
// (A 32-key, double-buffered-S/dP variant with 8 or 16 softmax warps was
// measured slower: its per-sub-chunk handshake latency dominates.)
template <int D, int LP, bool BIAS>
__global__ void __launch_bounds__(544, 1) attn_bwd_tc_kernel(
    const bf16* __restrict__ qkvg, const bf16* __restrict__ dctx, const float* __restrict__ mbias,
    const bf16* __restrict__ nb, const float* __restrict__ lse, const float* __restrict__ Dvec,
    bf16* __restrict__ dqkvg, bf16* __restrict__ kvpart, float* __restrict__ dnb_part,
    AttnGeom g, float scale, int NG, bf16* __restrict__ qpart, int NKW, int kv_red) {
  using SM = BwdSmem<D, LP>;
  constexpr int DC = D / 8;
  constexpr int NKC = LP / 128;
  constexpr int NSUB = LP / 64;
  constexpr int NCW = 16;  // softmax warps
  constexpr uint32_t C_S = 0, C_DP = 64, C_DQ = 128, C_DK = 128 + D, C_DV = 128 + 2 * D, C_DB = 256;
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sP = reinterpret_cast<bf16*>(smem + SM::p);
  bf16* sdS = reinterpret_cast<bf16*>(smem + SM::ds);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::bar);  // [0] S, [1] KV
  uint64_t* bar2 = bar + 2;                                      // [0] Sf, [1] PdS
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x;
  const int64_t h = blockIdx.y;
  // CTA = (batch group, head, query tile, key window of LP keys); rows longer than
  // 256 keys use several windows, whose dQ partials (and the dK/dV partials of
  // query tiles > 0) are combined afterwards in fixed order
  const int qt = blockIdx.z / NKW, kw = blockIdx.z % NKW;
  const int q0 = qt * 128, k0 = kw * LP;
  const int64_t Ttok = g.B * g.L;
  const int L = (int)g.L;
  const int64_t HD = g.H * D;
  const int64_t b_lo = (g.B * grp) / NG, b_hi = (g.B * (grp + 1)) / NG;

  const int quarter = warp & 3, cg = (warp >> 2) & 3;
  const int row = quarter * 32 + lane;
  const int i = q0 + row;
  const bool valid = i < L && warp < NCW;

  if (warp == NCW) tc::tmem_alloc<512>(slot);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&bar2[0], NCW);
    tc::mbar_init(&bar2[1], NCW);
  }
  if (warp < NCW) {
    if (BIAS) stage_bias_tile<LP>(smem + SM::bias, nb, h, q0, k0, L, tid, 512);
    if (b_lo < b_hi) bwd_stage<D, LP>(smem, qkvg, dctx, mbias, g, b_lo, h, q0, tid, k0);
    cp_async_commit();
    cp_async_wait0();
    tc::fence_proxy_async();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *slot;
  const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16);

  if (warp == NCW) {
    // ======================= MMA issuer =======================
    const int64_t nsub = (b_hi - b_lo) * NSUB;
    const uint32_t s0 = tc::smem_u32(smem);
    uint32_t phSf = 0, phP = 0;
    const uint32_t id_q = tc::idesc_bf16(128, D, false, true);
    const uint32_t id_kv = tc::idesc_bf16(128, D, true, true);
    const uint64_t a_dq = tc::sdesc(tc::smem_u32(sdS), 128, 16 * 128);
    const uint64_t a_ds = tc::sdesc(tc::smem_u32(sdS), 16 * 128, 128);
    const uint64_t a_p = tc::sdesc(tc::smem_u32(sP), 16 * 128, 128);
    if (nsub > 0) issue_sdp<D>(s0, 0, tbase, C_S, C_DP, &bar[0], SM::q, SM::o, SM::k, SM::v);
#pragma unroll 1
    for (int64_t j = 0; j < nsub; ++j) {
      const int sj = (int)(j % NSUB);
      const uint32_t st = s0 + (uint32_t)((j / NSUB) & 1) * SM::STAGE;
      const int tb = 2048 + 8 * (int)(j & 127);
      BT(tb, 0);
      tc::mbar_wait(&bar2[0], phSf);
      phSf ^= 1;
      tc::fence_after();
      BT(tb, 1);
      if (j + 1 < nsub) {
        const int sj2 = (int)((j + 1) % NSUB);
        const uint32_t st2 = s0 + (uint32_t)(((j + 1) / NSUB) & 1) * SM::STAGE;
        issue_sdp<D>(st2, sj2 * 64, tbase, C_S, C_DP, &bar[0], SM::q, SM::o, SM::k, SM::v);
      }
      BT(tb, 2);
      if (sj & 1) {
        const int kc = sj >> 1;
        tc::mbar_wait(&bar2[1], phP);
        phP ^= 1;
        tc::fence_after();
        BT(tb, 3);
        // dQ += dS Kc ; dK = dS^T Q ; dV = P^T dO   (chunk of 128 keys)
        const uint64_t b_k = tc::sdesc(st + SM::k + (kc * 16) * DC * 128, DC * 128, 128);
        const uint64_t b_q = tc::sdesc(st + SM::q, DC * 128, 128);
        const uint64_t b_o = tc::sdesc(st + SM::o, DC * 128, 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          tc::mma_bf16_ss_w(tbase + C_DQ, dadd(a_dq, k * 256), dadd(b_k, k * 2 * DC * 128), id_q,
                            (kc > 0 || k > 0) ? 1u : 0u);
          tc::mma_bf16_ss_w(tbase + C_DK, dadd(a_ds, k * 4096), dadd(b_q, k * 2 * DC * 128), id_kv,
                            k > 0 ? 1u : 0u);
          tc::mma_bf16_ss_w(tbase + C_DV, dadd(a_p, k * 4096), dadd(b_o, k * 2 * DC * 128), id_kv,
                            k > 0 ? 1u : 0u);
        }
        tc::mma_commit_w(&bar[1]);
        BT(tb, 4);
      }
    }
  } else if (b_lo < b_hi) {
    // ======================= softmax backward =======================
    if (BIAS) {
#pragma unroll
      for (int c = 0; c < LP / 4; c += 16) tmem_zero(tl + C_DB + cg * (LP / 4) + c);
    }
    uint32_t phS = 0, phKV = 0;
    bool kv_pending = false;
    int64_t pend_b = b_lo;
    int pend_c = 0;
    // (1/rowsum is folded into dO' and D' by the prep kernel)
    auto row_consts = [&](int64_t b, float& m2, float& Dv) {
      const int64_t bh = b * g.H + h;
      m2 = valid ? lse[2 * (bh * L + i)] : INFINITY;  // P' = 0 on rows beyond L
      Dv = valid ? Dvec[g.tok(b, i) * g.H + h] : 0.f;
    };
    float m2, Dv, m2n = 0.f, Dvn = 0.f;
    row_consts(b_lo, m2, Dv);
    // batch b_lo + 1 into the second buffer (nothing has read it yet)
    if (b_lo + 1 < b_hi) bwd_stage<D, LP>(smem + SM::STAGE, qkvg, dctx, mbias, g, b_lo + 1, h, q0, tid, k0);
    cp_async_commit();

    // drain dK / dV of chunk c of batch b: lanes = keys, cg -> (dK|dV, column half);
    // ``mid`` runs while the TMEM load is in flight
    auto drain_kv = [&](int64_t b, int c, auto&& mid) {
      const int key = k0 + c * 128 + row;
      const int region = cg >> 1, chalf = cg & 1;
      constexpr int DH = D / 2;
      float vv[DH];
      const uint32_t col = (region ? C_DV : C_DK) + chalf * DH;
      if constexpr (DH == 16) tc::tmem_ld16(tl + col, vv);
      else tc::tmem_ld8(tl + col, vv);
      mid();
      tc::wait_ld();
      if (key < L) {
        const float sc = region ? 1.0f : scale;
        uint32_t pk[DH / 2];
#pragma unroll
        for (int e = 0; e < DH; e += 2) pk[e / 2] = tc::pack_bf16(vv[e] * sc, vv[e + 1] * sc);
        const int64_t t = g.tok(b, key);
        bf16* dst = (qt == 0 || kv_red) ? dqkvg + t * g.ld + (1 + region) * HD + h * D + chalf * DH
                                        : kvpart + (qt - 1) * Ttok * 2 * HD + t * 2 * HD + region * HD + h * D + chalf * DH;
        if (kv_red) {
          // two query tiles: both add into the zeroed dK/dV slices (no combine pass)
#pragma unroll
          for (int k = 0; k < DH / 8; ++k)
            red_add_bf16x8(dst + 8 * k, make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]));
        } else {
#pragma unroll
          for (int k = 0; k < DH / 8; ++k)
            reinterpret_cast<uint4*>(dst)[k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
        }
      }
    };
    // dQ of batch b: the TMEM load (dq_issue) and, after a tcgen05.wait::ld, the
    // store (dq_store) -- split so the load can overlap other work
    constexpr int DQ = D / 4;
    auto dq_issue = [&](float (&vv)[DQ]) {
      if constexpr (DQ == 8) tc::tmem_ld8(tl + C_DQ + cg * DQ, vv);
      else tmem_ld4(tl + C_DQ + cg * DQ, vv);
    };
    auto dq_store = [&](int64_t b, const float (&vv)[DQ]) {
      if (valid) {
        const int64_t t = g.tok(b, i);
        bf16* dst = (kw == 0) ? dqkvg + t * g.ld + h * D + cg * DQ
                              : qpart + (kw - 1) * Ttok * HD + t * HD + h * D + cg * DQ;
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < DQ; e += 2) pk[e / 2] = tc::pack_bf16(vv[e] * scale, vv[e + 1] * scale);
        if constexpr (DQ == 8)
          *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        else
          *reinterpret_cast<uint2*>(dst) = make_uint2(pk[0], pk[1]);
      }
    };
    auto drain_dq = [&](int64_t b) {
      float vv[DQ];
      dq_issue(vv);
      tc::wait_ld();
      dq_store(b, vv);
    };

#pragma unroll 1
    for (int64_t b = b_lo; b < b_hi; ++b) {
      const int buf = (int)((b - b_lo) & 1);
      const float* sMb = reinterpret_cast<const float*>(smem + buf * SM::STAGE + SM::mb);
      const bool has_next = b + 1 < b_hi;
      if (has_next) row_consts(b + 1, m2n, Dvn);  // consumed at the next batch
      const float2 nm2 = make_float2(-m2, -m2), nD2 = make_float2(-Dv, -Dv);
#pragma unroll 1
      for (int sj = 0; sj < NSUB; ++sj) {
        const int kc = sj >> 1, sub = sj & 1;
        const bool last_in_batch = sj == NSUB - 1;
        const int c0 = sj * 64 + cg * 16;  // this thread's 16 key columns
        uint32_t braw[8];
        if (BIAS) {
          const uint4 u0 = *reinterpret_cast<const uint4*>(smem + SM::bias + bias_off<LP>(row, c0 >> 3));
          const uint4 u1 = *reinterpret_cast<const uint4*>(smem + SM::bias + bias_off<LP>(row, (c0 >> 3) + 1));
          braw[0] = u0.x, braw[1] = u0.y, braw[2] = u0.z, braw[3] = u0.w;
          braw[4] = u1.x, braw[5] = u1.y, braw[6] = u1.z, braw[7] = u1.w;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) braw[e] = 0u;
        }
        float mbv[16];
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(sMb + c0 + e);
          mbv[e] = t4.x, mbv[e + 1] = t4.y, mbv[e + 2] = t4.z, mbv[e + 3] = t4.w;
        }
        // ---- S/dP(j) out of TMEM, then hand the columns back ----
        const int tb = (warp == 0 ? 0 : (warp == NCW - 1 ? 4096 : 6144)) + 16 * (int)(((b - b_lo) * NSUB + sj) & 127);
        BT(tb, 0);
        tc::mbar_wait(&bar[0], phS);
        phS ^= 1;
        tc::fence_after();
        BT(tb, 1);
        float s[16], dp[16], acc[16];
        tc::tmem_ld16(tl + C_S + cg * 16, s);
        tc::tmem_ld16(tl + C_DP + cg * 16, dp);
        // the previous sub-chunk's bias-gradient store completed while this
        // thread waited for S/dP (waiting right after the store was a stall)
        if (BIAS) tc::wait_st();
        if (BIAS) tc::tmem_ld16(tl + C_DB + c0, acc);
        tc::wait_ld();
        if (last_in_batch && has_next) {
          // batch b+1's staging: each thread waits for its own copies, then a
          // barrier over the 16 softmax warps makes every thread's copies (the
          // key-mask row is read by all of them) visible before batch b+1 starts
          cp_async_wait0();
          tc::fence_proxy_async();
          asm volatile("bar.sync 1, 512;" ::: "memory");
        }
        tc::fence_before();
        tc::mbar_arrive_warp(&bar2[0]);
        BT(tb, 2);
        // ---- P, dS, bias gradient ----
        uint32_t pp[8], pd[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float2 x = tc::logit2(make_float2(s[e], s[e + 1]), tc::bf16x2_f2(braw[e / 2]),
                                      make_float2(mbv[e], mbv[e + 1]), scale);
          const float2 xd = __fadd2_rn(x, nm2);
          const float2 p = make_float2(tc::ex2(xd.x), tc::ex2(xd.y));
          const float2 d = __fmul2_rn(p, __fadd2_rn(make_float2(dp[e], dp[e + 1]), nD2));
          if (BIAS) {
            const float2 a = __fadd2_rn(make_float2(acc[e], acc[e + 1]), d);
            acc[e] = a.x, acc[e + 1] = a.y;
          }
          pp[e / 2] = tc::pack_bf16(p.x, p.y);
          pd[e / 2] = tc::pack_bf16(d.x, d.y);
        }
        if (BIAS) tmem_st16(tl + C_DB + c0, acc);
        BT(tb, 3);
        // ---- P / dS tile [128 q x 128 k]: core (row/8, kcol/8) at ((row/8)*16 + kcol/8)*128 B ----
        // (stored once the previous chunk's dQ/dK/dV MMAs, which read the tile, are complete)
        auto store_pds = [&]() {
          const int kcol = sub * 64 + cg * 16;
#pragma unroll
          for (int qd = 0; qd < 2; ++qd) {
            const int off = ((row >> 3) * 16 + (kcol >> 3) + qd) * 64 + (row & 7) * 8;
            *reinterpret_cast<uint4*>(sP + off) = make_uint4(pp[4 * qd], pp[4 * qd + 1], pp[4 * qd + 2], pp[4 * qd + 3]);
            *reinterpret_cast<uint4*>(sdS + off) = make_uint4(pd[4 * qd], pd[4 * qd + 1], pd[4 * qd + 2], pd[4 * qd + 3]);
          }
        };
        bool pds_stored = false;
        // ---- previous chunk's dQ/dK/dV: wait, drain, recycle its staging ----
        if (sub == 0 && kv_pending) {
          tc::mbar_wait(&bar[1], phKV);
          phKV ^= 1;
          tc::fence_after();
          BT(tb, 4);
          // this sub-chunk's P / dS go to shared memory while the dK/dV load is
          // in flight; at a batch boundary also the dQ load and the prefetch of
          // batch b+1 into batch b-1's buffer (every MMA that read it is complete)
          if (pend_c == NKC - 1) {
            float vq[DQ];
            // (the prefetch inside the load window measured faster for one key
            // chunk per batch -- col 105 -> 97 us -- and slower for two -- tri
            // 197.5 -> 200 us -- so with two it follows the dQ store)
            auto stage_next = [&] {
              if (has_next)
                bwd_stage<D, LP>(smem + (buf ^ 1) * SM::STAGE, qkvg, dctx, mbias, g, b + 1, h, q0, tid, k0);
              cp_async_commit();
            };
            drain_kv(pend_b, pend_c, [&] {
              dq_issue(vq);
              store_pds();
              if (NKC == 1) stage_next();
            });
            dq_store(pend_b, vq);
            if (NKC > 1) stage_next();
          } else {
            drain_kv(pend_b, pend_c, store_pds);
          }
          pds_stored = true;
          kv_pending = false;
          BT(tb, 5);
        }
        if (!pds_stored) store_pds();
        BT(tb, 6);
        if (sub == 1) {
          tc::fence_proxy_async();
          tc::fence_before();
          tc::mbar_arrive_warp(&bar2[1]);
          BT(tb, 7);
          kv_pending = true;
          pend_b = b;
          pend_c = kc;
        }
      }
      m2 = m2n, Dv = Dvn;
    }
    // ---- last chunk's dQ/dK/dV ----
    if (kv_pending) {
      tc::mbar_wait(&bar[1], phKV);
      tc::fence_after();
      drain_kv(pend_b, pend_c, [] {});
      drain_dq(pend_b);
    }
  } else if (BIAS) {  // empty batch group: zero bias-gradient partial
#pragma unroll
    for (int c = 0; c < LP / 4; c += 16) tmem_zero(tl + C_DB + cg * (LP / 4) + c);
    tc::wait_st();
  }
  // ---- bias-gradient partial of this batch group ----
  if (BIAS && warp < NCW) {
    tc::wait_st();
    constexpr int PER = LP / 4;
#pragma unroll 1
    for (int c = 0; c < PER; c += 16) {
      float vv[16];
      tc::tmem_ld16(tl + C_DB + cg * PER + c, vv);
      tc::wait_ld();
      if (valid) {
        float* dst = dnb_part + (((size_t)grp * g.H + h) * L + i) * L + k0 + cg * PER + c;
        const int j0 = k0 + cg * PER + c;
        if ((L % 4) == 0 && j0 + 16 <= L) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            reinterpret_cast<float4*>(dst)[k] = make_float4(vv[4 * k], vv[4 * k + 1], vv[4 * k + 2], vv[4 * k + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (j0 + e < L) dst[e] = vv[e];
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == NCW) tc::tmem_dealloc<512>(tbase);
}

// token-major, 8 channels per thread: dctx = dgated*gate (bf16, the dO the
// MMAs read), d(g) = dgated*ctx*gate*(1-gate), Dvec[t, h] = sum_k dO*ctx
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_prep_tc_kernel(
    const bf16* __restrict__ ctx, const bf16* __restrict__ gate, const bf16* __restrict__ dgated,
    bf16* __restrict__ dqkvg, bf16* __restrict__ dctx, float* __restrict__ Dvec, int64_t T, int H,
    int64_t ld, const float* __restrict__ mask, int64_t msb, int64_t msl, float* __restrict__ mbias,
    int64_t B, int64_t L, int64_t sb, int64_t sl, const float* __restrict__ lse, float* __restrict__ gpart,
    int zero_kv) {
  // key-mask bias of every (batch, key), [b][l] contiguous, in the log2
  // domain of the softmax: (m - 1) * 1e9 * log2(e)  (src/attention.py:151)
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B * L;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / L, l = e % L;
    mbias[e] = (mask[b * msb + l * msl] - 1.0f) * tc::MASK_BIAS_L2;
  }
  constexpr int G = D / 8;  // threads per head
  const int64_t HD8 = (int64_t)H * D / 8;
  const int64_t n = T * HD8;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  // gate-bias gradient: this thread's 8 columns (c8 is fixed per thread when
  // HD8 divides the block size -- checked by the host) summed over its tokens,
  // as the stored bf16 d(gate) values
  float gs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  // two items per thread and iteration, all loads issued before the math
  // (memory-level parallelism; one item per iteration ran at ~2/3 of HBM)
  constexpr int PU = 2;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += step * PU) {
    uint4 rdg[PU], rgv[PU], rcv[PU];
    float rl[PU];
#pragma unroll
    for (int q = 0; q < PU; ++q) {
      const int64_t e = base + q * step + threadIdx.x;
      rl[q] = 0.f;
      if (e < n) {
        // dO is pre-scaled by this row's 1/rowsum (the backward kernel then
        // works with the unnormalised P' = exp2(x - m):  dS = P' (dP' - D'),
        // dV = P'^T dO' -- one multiply per score fewer; fully-masked rows stay
        // uniform since P' = 1 there and 1/l = 1/L)
        const int64_t t = e / HD8;
        const int c8 = (int)(e % HD8);
        const int64_t bq = sl == 1 ? t / sb : t % sl, lq = sl == 1 ? t % sb : t / sl;
        rl[q] = lse[2 * ((bq * H + c8 / G) * L + lq) + 1];
        const int64_t c = t * (HD8 * 8) + c8 * 8;
        rdg[q] = *reinterpret_cast<const uint4*>(dgated + c);
        rgv[q] = *reinterpret_cast<const uint4*>(gate + c);
        rcv[q] = *reinterpret_cast<const uint4*>(ctx + c);
      }
    }
#pragma unroll
    for (int q = 0; q < PU; ++q) {
      const int64_t e = base + q * step + threadIdx.x;
      const bool act = e < n;
      const int64_t t = act ? e / HD8 : 0;
      const int c8 = act ? (int)(e % HD8) : 0;
      float dsum = 0.f;
      if (act) {
        const int64_t c = t * (HD8 * 8) + c8 * 8;
        float dg[8], gv[8], cv[8];
        bf16x8_to_f(rdg[q], dg);
        bf16x8_to_f(rgv[q], gv);
        bf16x8_to_f(rcv[q], cv);
        uint32_t pc[4], pg[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const float d0 = dg[u] * gv[u] * rl[q], d1 = dg[u + 1] * gv[u + 1] * rl[q];
          const float g0 = dg[u] * cv[u] * gv[u] * (1.0f - gv[u]);
          const float g1 = dg[u + 1] * cv[u + 1] * gv[u + 1] * (1.0f - gv[u + 1]);
          const __nv_bfloat162 dq = __floats2bfloat162_rn(d0, d1);
          dsum += __bfloat162float(dq.x) * cv[u] + __bfloat162float(dq.y) * cv[u + 1];
          pc[u / 2] = *reinterpret_cast<const uint32_t*>(&dq);
          pg[u / 2] = tc::pack_bf16(g0, g1);
          const float2 gr = tc::bf16x2_f2(pg[u / 2]);
          gs[u] += gr.x;
          gs[u + 1] += gr.y;
        }
        *reinterpret_cast<uint4*>(dctx + c) = make_uint4(pc[0], pc[1], pc[2], pc[3]);
        *reinterpret_cast<uint4*>(dqkvg + t * ld + 3 * HD8 * 8 + c8 * 8) = make_uint4(pg[0], pg[1], pg[2], pg[3]);
        if (zero_kv) {  // the dK / dV slices the backward's two query tiles add into
          st_zero16(dqkvg + t * ld + HD8 * 8 + c8 * 8);
          st_zero16(dqkvg + t * ld + 2 * HD8 * 8 + c8 * 8);
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      if (act && (c8 % G) == 0) Dvec[t * H + c8 / G] = dsum;
    }
  }
  if (gpart) {
    // block partial of the gate-bias gradient: threads tid, tid + HD8, ...
    // share column chunk tid % HD8; summed in thread order
    __shared__ float red[256 * 8];
#pragma unroll
    for (int u = 0; u < 8; ++u) red[threadIdx.x * 8 + u] = gs[u];
    __syncthreads();
    for (int c = threadIdx.x; c < HD8 * 8; c += blockDim.x) {
      const int c8 = c / 8, u = c % 8;
      float acc = 0.f;
      for (int t = c8; t < (int)blockDim.x; t += (int)HD8) acc += red[t * 8 + u];
      gpart[(int64_t)blockIdx.x * HD8 * 8 + c] = acc;
    }
  }
}

// dqkvg[:, 0:HD] += sum_w qpart[w] (key windows > 0), dqkvg[:, HD:3HD] += sum_q kvpart[q]
// (query tiles > 0); fixed addend order
__global__ void attn_part_combine_kernel(bf16* __restrict__ dqkvg, const bf16* __restrict__ qpart, int nq,
                                         const bf16* __restrict__ kvpart, int nkv, int64_t T, int64_t ld,
                                         int64_t HD) {
  const int64_t per_row = 3 * HD / 8;
  const int64_t n = T * per_row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / per_row, c = (e % per_row) * 8;
    const bool isq = c < HD;
    if (isq ? nq == 0 : nkv == 0) continue;
    uint4* d = reinterpret_cast<uint4*>(dqkvg + t * ld + c);
    float a[8], bq[8];
    bf16x8_to_f(*d, a);
    const int np = isq ? nq : nkv;
    for (int k = 0; k < np; ++k) {
      const uint4 p = isq ? *reinterpret_cast<const uint4*>(qpart + ((int64_t)k * T + t) * HD + c)
                          : *reinterpret_cast<const uint4*>(kvpart + ((int64_t)k * T + t) * 2 * HD + c - HD);
      bf16x8_to_f(p, bq);
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += bq[u];
    }
    uint32_t o[4];
#pragma unroll
    for (int u = 0; u < 8; u += 2) o[u / 2] = tc::pack_bf16(a[u], a[u + 1]);
    *d = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// dqkvg[:, HD:3HD] += kvpart   (query tile 1's dK/dV partial)
__global__ void attn_kv_combine_kernel(bf16* __restrict__ dqkvg, const bf16* __restrict__ kvpart,
                                       int64_t T, int64_t ld, int64_t HD) {
  const int64_t per_row = 2 * HD / 8;
  const int64_t n = T * per_row;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / per_row, c = (e % per_row) * 8;
    uint4* d = reinterpret_cast<uint4*>(dqkvg + t * ld + HD + c);
    const uint4 p = *reinterpret_cast<const uint4*>(kvpart + t * 2 * HD + c);
    float a[8], bq[8];
    bf16x8_to_f(*d, a);
    bf16x8_to_f(p, bq);
    uint32_t o[4];
#pragma unroll
    for (int u = 0; u < 8; u += 2) o[u / 2] = tc::pack_bf16(a[u] + bq[u], a[u + 1] + bq[u + 1]);
    *d = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// dnb[e] (+)= sum over batch groups of the partials (fixed group order)
__global__ void attn_dnb_reduce_kernel(const float* __restrict__ part, float* __restrict__ dnb,
                                       int64_t n, int NG, int accumulate) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int gi = 0; gi < NG; ++gi) acc += part[gi * n + e];
    dnb[e] = accumulate ? dnb[e] + acc : acc;
  }
}

template <typename T>
__global__ void colsum_slice_kernel(const T* __restrict__ x, int64_t ld, int64_t off,
                                    float* __restrict__ partials, int64_t rows, int64_t C) {
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) acc += to_f(x[r * ld + off + c]);
    partials[blockIdx.x * C + c] = acc;
  }
}

bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_DISABLE_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

struct BwdPlan {
  int NQT, NG, LP, NKW, kv_red;
  int64_t off_dctx, off_dvec, off_mb, off_kv, off_q, off_part, off_cols, total;
};

BwdPlan bwd_plan(const AttnGeom& g) {
  BwdPlan p{};
  p.LP = g.L <= 128 ? 128 : 256;
  if (const char* e = getenv("EVO_ATTN_BWD_LP")) {  // key-window width sweeps (128 or 256)
    const int f = atoi(e);
    if (f == 128 || f == 256) p.LP = f;
  }
  p.NQT = (int)((g.L + 127) / 128);
  p.NKW = (int)((g.L + p.LP - 1) / p.LP);
  int per = (int)(g.H * p.NQT * p.NKW);
  int ng = num_sms() / (per > 0 ? per : 1);
  if (ng < 1) ng = 1;
  if (ng > g.B) ng = (int)g.B;
  p.NG = ng;
  // two query tiles over one key window: dK/dV by reduction stores into slices
  // the prep kernel zeroed (order-independent with two addends) instead of a
  // partial plane and a combine pass (EVO_ATTN_KV_RED=0 restores the latter)
  static int kvr = -1;
  if (kvr < 0) {
    const char* e = getenv("EVO_ATTN_KV_RED");
    kvr = (e && e[0] == '0') ? 0 : 1;
  }
  p.kv_red = (kvr == 1 && p.NQT == 2 && p.NKW == 1) ? 1 : 0;
  const int64_t T = g.B * g.L;  // tokens covered by the problem set
  const int64_t HD = g.H * g.D;
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  p.off_dctx = 0;
  p.off_dvec = p.off_dctx + al(T * HD * 2);
  p.off_mb = p.off_dvec + al(g.B * g.H * g.L * 4);
  p.off_kv = p.off_mb + al(g.B * g.L * 4);
  p.off_q = p.off_kv + (int64_t)(p.NQT - 1) * al(T * 2 * HD * 2);
  p.off_part = p.off_q + (int64_t)(p.NKW - 1) * al(T * HD * 2);
  p.off_cols = p.off_part + al((int64_t)p.NG * g.H * g.L * g.L * 4);
  p.total = p.off_cols + al((int64_t)(EVO_PARTIAL_BLOCKS > 8 * num_sms() ? EVO_PARTIAL_BLOCKS : 8 * num_sms()) * HD * 4);
  return p;
}

bool bwd_supported(const AttnGeom& g, int dtype) {
  if (tc_disabled() || dtype != EVO_BF16) return false;
  if (!(g.D == 16 || g.D == 32) || g.L > 1024 || g.L < 65) return false;
  if ((g.ld % 8) != 0) return false;
  return true;
}

template <int D, int LP, bool BIAS>
void launch_bwd(const void* qkvg, const bf16* dctx, const float* mask, const void* nb,
                const float* lse, const float* Dvec, void* dqkvg, bf16* kvpart, float* part,
                const AttnGeom& g, const BwdPlan& p, cudaStream_t s, bf16* qpart) {
  using SM = BwdSmem<D, LP>;
  auto k = attn_bwd_tc_kernel<D, LP, BIAS>;
  static bool attr = false;
  if (!attr) {
    EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::total));
    attr = true;
  }
  dim3 grid((unsigned)p.NG, (unsigned)g.H, (unsigned)(p.NQT * p.NKW));
  const float scale = (float)(1.0 / sqrt((double)D));
  k<<<grid, 544, SM::total, s>>>((const bf16*)qkvg, dctx, mask, (const bf16*)nb, lse, Dvec,
                                 (bf16*)dqkvg, kvpart, part, g, scale, p.NG, qpart, p.NKW, p.kv_red);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

template <int D>
void launch_bwd_d(bool bias, int LP, const void* qkvg, const bf16* dctx, const float* mask,
                  const void* nb, const float* lse, const float* Dvec, void* dqkvg, bf16* kvpart,
                  float* part, const AttnGeom& g, const BwdPlan& p, cudaStream_t s, bf16* qpart) {
  if (LP == 128) {
    if (bias) launch_bwd<D, 128, true>(qkvg, dctx, mask, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
    else launch_bwd<D, 128, false>(qkvg, dctx, mask, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
  } else {
    if (bias) launch_bwd<D, 256, true>(qkvg, dctx, mask, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
    else launch_bwd<D, 256, false>(qkvg, dctx, mask, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
  }
}

}  // namespace
int64_t attn_bwd_tc_workspace(const AttnGeom& g, int dtype) {
  if (!bwd_supported(g, dtype)) return 0;
  return bwd_plan(g).total;
}

bool attn_bwd_tc_try(const void* qkvg, const float* mask, const void* nb, const void* ctx,
                     const void* gate, const void* dgated, const float* lse, void* dqkvg,
                     float* dnb, float* dbg, int accumulate, void* ws, size_t ws_bytes,
                     const AttnGeom& g, int dtype, cudaStream_t s) {
  if (!bwd_supported(g, dtype)) return false;
  if (((uintptr_t)qkvg | (uintptr_t)dqkvg | (uintptr_t)ctx | (uintptr_t)gate | (uintptr_t)dgated) & 15)
    return false;
  const BwdPlan p = bwd_plan(g);
  EVO_REQUIRE((int64_t)ws_bytes >= p.total, EVO_ERR_ARG, "attn_bwd: workspace too small");
  uint8_t* w = (uint8_t*)ws;
  bf16* dctx = (bf16*)(w + p.off_dctx);
  float* Dvec = (float*)(w + p.off_dvec);
  bf16* kvpart = (bf16*)(w + p.off_kv);
  bf16* qpart = (bf16*)(w + p.off_q);
  float* part = (float*)(w + p.off_part);
  float* cols = (float*)(w + p.off_cols);
  float* mbias = (float*)(w + p.off_mb);
  const int64_t T = g.B * g.L, HD = g.H * g.D;
  const int64_t nthr = T * HD / 8;
  const unsigned pgrid = (unsigned)imin64((nthr + 255) / 256, (int64_t)num_sms() * 8);
  // the gate-bias column sums ride on the prep kernel when each thread keeps
  // one column chunk (HD / 8 divides the 256-thread block)
  const bool gfuse = dbg != nullptr && (256 % (HD / 8)) == 0 && pgrid <= (unsigned)(8 * num_sms());
  float* gpart = gfuse ? partial_buffer(cols, (size_t)pgrid * HD * 4) : nullptr;
  {
    if (g.D == 16)
      attn_bwd_prep_tc_kernel<16><<<pgrid, 256, 0, s>>>((const bf16*)ctx, (const bf16*)gate,
                                                         (const bf16*)dgated, (bf16*)dqkvg, dctx,
                                                         Dvec, T, (int)g.H, g.ld, mask, g.msb, g.msl,
                                                         mbias, g.B, g.L, g.sb, g.sl, lse, gpart, p.kv_red);
    else
      attn_bwd_prep_tc_kernel<32><<<pgrid, 256, 0, s>>>((const bf16*)ctx, (const bf16*)gate,
                                                         (const bf16*)dgated, (bf16*)dqkvg, dctx,
                                                         Dvec, T, (int)g.H, g.ld, mask, g.msb, g.msl,
                                                         mbias, g.B, g.L, g.sb, g.sl, lse, gpart, p.kv_red);
    EVO_LAUNCH_CHECK();
  }
  if (gfuse) finalize_partials(gpart, (int)pgrid, HD, dbg, accumulate, s);
  const bool bias = nb != nullptr && dnb != nullptr;
  if (g.D == 16)
    launch_bwd_d<16>(bias, p.LP, qkvg, dctx, mbias, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
  else
    launch_bwd_d<32>(bias, p.LP, qkvg, dctx, mbias, nb, lse, Dvec, dqkvg, kvpart, part, g, p, s, qpart);
  if (p.NKW > 1 || p.NQT > 2) {
    attn_part_combine_kernel<<<cdiv(T * 3 * HD / 8, 256), 256, 0, s>>>((bf16*)dqkvg, qpart, p.NKW - 1, kvpart,
                                                                        p.NQT - 1, T, g.ld, HD);
    EVO_LAUNCH_CHECK();
  } else if (p.NQT > 1 && !p.kv_red) {
    attn_kv_combine_kernel<<<cdiv(T * 2 * HD / 8, 256), 256, 0, s>>>((bf16*)dqkvg, kvpart, T, g.ld, HD);
    EVO_LAUNCH_CHECK();
  }
  if (bias) {
    const int64_t n = g.H * g.L * g.L;
    attn_dnb_reduce_kernel<<<cdiv(n, 256), 256, 0, s>>>(part, dnb, n, p.NG, accumulate);
    EVO_LAUNCH_CHECK();
  }
  int slice = 0;
  if (!gfuse && !colsum_vec((bf16*)dqkvg + 3 * HD, EVO_BF16, g.ld, nullptr, nullptr, EVO_BF16, dbg, accumulate,
                            cols, T, HD, 0, s)) {
    const unsigned pg = partial_grid(T);
    colsum_slice_kernel<bf16><<<pg, 256, 0, s>>>((const bf16*)dqkvg, g.ld, 3 * HD, cols, T, HD);
    EVO_LAUNCH_CHECK();
    finalize_partials(cols, pg, HD, dbg, accumulate, s);
    slice = 1;
  }
  // prep, the combine pass, the bias-gradient reduction, the column-slice
  // sum (the main kernel, colsum_vec and finalize_partials count themselves)
  count_launch(1 + (p.NKW > 1 || (p.NQT > 1 && !p.kv_red)) + bias + slice);
  return true;
}

}  // namespace evo

#ifdef EVO_BWD_TRACE
extern "C" int evo_bwd_trace_read(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, evo::g_bwd_trace, sizeof(long long) * n);
}
#endif
