// Bulk-copy-staged row streams for the bandwidth-bound glue kernels.
//
// The register-staged glue kernels (glue.cu) keep one or two rows per thread
// in flight and run at ~25% occupancy (their per-column accumulators cost
// registers), which leaves them latency-bound near 3 TB/s.  Here each block
// owns a contiguous range of rows and streams it through an NST-deep ring of
// shared-memory stages filled by 1-D bulk copies (cp.async.bulk, TMA engine,
// mbarrier transaction counts): the bytes in flight no longer depend on
// registers or occupancy, and the compute warps only ever read shared memory.
//
// LayerNorm backward (src/tensor.py:190-208):
//   dx = dres + inv * (dxh - mean(dxh) - xh * mean(dxh * xh)),  dxh = dy * g
// with the dgamma / dbeta (and optional colsum(dx)) partials per block, the
// same partial layout as ln_bwd_vec ([dgamma C | dbeta C | colsum(dx) C]).
#include <cstdlib>

#include "common.cuh"
#include "reduce.cuh"
#include "tc_common.cuh"
#include "vec.cuh"

namespace evo {
namespace {

constexpr int ST = 256;  // compute threads per block; one more warp is the bulk-copy producer

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

template <int C, typename TX, typename TD, int NST>
struct LnbStream {
  static constexpr int LANES = C / 8 < 32 ? C / 8 : 32;  // lanes per row, 8 columns per lane chunk
  static constexpr int CH = C / (8 * LANES);
  static constexpr int RPW = 32 / LANES;
  static constexpr int RS = (ST / 32) * RPW;              // rows per stage: one per lane group
  static constexpr int XB = RS * C * (int)sizeof(TX);
  static constexpr int DB = RS * C * (int)sizeof(TD);
  static constexpr int RB = RS * C * 4;
  static constexpr int SB = RS * 4;
  static constexpr int STAGE = ((XB + DB + RB + 2 * SB) + 127) / 128 * 128;
  static constexpr int RED = (ST / LANES) * 3 * C * 4;    // end-of-kernel partial reduction
  static constexpr int BYTES = (NST * STAGE > RED ? NST * STAGE : RED) + 2 * NST * 8;
};

template <int C, typename TX, typename TD, int NST>
__global__ void __launch_bounds__(ST + 32) ln_bwd_stream_kernel(
    const TX* __restrict__ x, const TD* __restrict__ dy, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* dres, float* dx,
    __nv_bfloat16* __restrict__ dx16, float* __restrict__ partials, int64_t rows, int want_dxsum) {
  using M = LnbStream<C, TX, TD, NST>;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (M::BYTES - 2 * NST * 8));  // stage full
  uint64_t* emp = bar + NST;                                                    // stage free
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int l = lane % M::LANES, gi = lane / M::LANES;
  const int rr = warp * M::RPW + gi;  // this lane group's row within a stage
  const int64_t nstage = (rows + M::RS - 1) / M::RS;
  const int64_t s0 = nstage * blockIdx.x / gridDim.x, s1 = nstage * (blockIdx.x + 1) / gridDim.x;
  const int n = (int)(s1 - s0);

  auto issue = [&](int it) {
    const int s = it % NST;
    const int64_t r0 = (s0 + it) * M::RS;
    const int nr = (int)(rows - r0 < M::RS ? rows - r0 : M::RS);
    uint8_t* st = sm + s * M::STAGE;
    const uint32_t xb = nr * C * sizeof(TX), db = nr * C * sizeof(TD), rb = nr * C * 4, sb = nr * 4;
    mbar_expect_tx(&bar[s], xb + db + (dres ? rb : 0) + 2 * sb);
    bulk_g2s(st, x + r0 * C, xb, &bar[s]);
    bulk_g2s(st + M::XB, dy + r0 * C, db, &bar[s]);
    if (dres) bulk_g2s(st + M::XB + M::DB, dres + r0 * C, rb, &bar[s]);
    bulk_g2s(st + M::XB + M::DB + M::RB, mean + r0, sb, &bar[s]);
    bulk_g2s(st + M::XB + M::DB + M::RB + M::SB, rstd + r0, sb, &bar[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&bar[s], 1);
      tc::mbar_init(&emp[s], ST / 32);
    }
  }
  __syncthreads();
  if (warp == ST / 32) {
    // producer: refill stage s once all compute warps released it
    if (lane == 0) {
      for (int it = 0; it < n; ++it) {
        const int s = it % NST;
        if (it >= NST) tc::mbar_wait(&emp[s], (uint32_t)(((it / NST) - 1) & 1));
        issue(it);
      }
    }
    return;
  }
  float dg[M::CH][8], db[M::CH][8], dsx[M::CH][8], gg[M::CH][8];
#pragma unroll
  for (int k = 0; k < M::CH; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      dg[k][e] = db[k][e] = dsx[k][e] = 0.f;
      gg[k][e] = g[(k * M::LANES + l) * 8 + e];
    }

  for (int it = 0; it < n; ++it) {
    const int s = it % NST;
    const int64_t r0 = (s0 + it) * M::RS;
    const int nr = (int)(rows - r0 < M::RS ? rows - r0 : M::RS);
    tc::mbar_wait(&bar[s], (uint32_t)((it / NST) & 1));
    const uint8_t* st = sm + s * M::STAGE;
    // lane groups past the stage's last row run on row 0 with zero weight, so
    // every lane of a warp takes part in the group shuffles
    const bool act = rr < nr;
    const int rq = act ? rr : 0;
    const float w = act ? 1.f : 0.f;
    {
      const TX* sx = reinterpret_cast<const TX*>(st) + rq * C;
      const TD* sdy = reinterpret_cast<const TD*>(st + M::XB) + rq * C;
      const float* sres = reinterpret_cast<const float*>(st + M::XB + M::DB) + rq * C;
      const float mu = reinterpret_cast<const float*>(st + M::XB + M::DB + M::RB)[rq];
      const float inv = reinterpret_cast<const float*>(st + M::XB + M::DB + M::RB + M::SB)[rq];
      float xh[M::CH][8], dxh[M::CH][8], o[M::CH][8];
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 8;
        ld8(sx + c0, xh[k]);
        ld8(sdy + c0, dxh[k]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = dxh[k][e] * w;
          xh[k][e] = (xh[k][e] - mu) * inv;
          dxh[k][e] = d * gg[k][e];
          dg[k][e] += d * xh[k][e];
          db[k][e] += d;
          s1 += dxh[k][e];
          s2 += dxh[k][e] * xh[k][e];
        }
      }
      const float m1 = group_sum<M::LANES>(s1) / (float)C, m2 = group_sum<M::LANES>(s2) / (float)C;
      const int64_t r = r0 + rq;
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 8;
        if (dres) {
          ld8(sres + c0, o[k]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) o[k][e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          o[k][e] += inv * (dxh[k][e] - m1 - xh[k][e] * m2);
          dsx[k][e] += w * o[k][e];
        }
        if (act) {
          st8(dx + r * C + c0, o[k]);
          if (dx16) st8(dx16 + r * C + c0, o[k]);
        }
      }
    }
    tc::mbar_arrive_warp(&emp[s]);  // this warp is done with stage s
  }
  // per-column partials: lane groups -> shared memory -> one row per block (the
  // stage ring is reused: every stage was consumed, no copy is in flight)
  asm volatile("bar.sync 1, %0;" ::"r"(ST) : "memory");
  float* red = reinterpret_cast<float*>(sm);
  const int grp = tid / M::LANES;
  float* mine = red + grp * 3 * C;
#pragma unroll
  for (int k = 0; k < M::CH; ++k) {
    const int c0 = (k * M::LANES + l) * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      mine[c0 + e] = dg[k][e];
      mine[C + c0 + e] = db[k][e];
      mine[2 * C + c0 + e] = dsx[k][e];
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(ST) : "memory");
  const int W = want_dxsum ? 3 * C : 2 * C;
  for (int c = tid; c < W; c += ST) {
    float acc = 0.f;
    for (int q = 0; q < ST / M::LANES; ++q) acc += red[q * 3 * C + c];
    partials[(int64_t)blockIdx.x * 3 * C + c] = acc;
  }
}


// Pair-bias backward (src/model.py:312-317 differentiated): per pair token t,
//   dP[h] = dnb[h, t] (swap_xy: the transposed plane position),
//   dzl = dP . w^T,  dz += LN_bwd(dzl),  dw += zl (x) dP,  dgamma / dbeta += ...
// One warp per token (4 channels per lane, C = 128), TPW tokens per warp and
// stage; z, dz, the LN statistics and (without swap) the H dnb planes of a
// stage arrive by bulk copy.  Partial row per block: [dw C*H | dgamma C | dbeta C].
constexpr int PB_CW = 4;  // compute warps per pair-bias block

template <int NST, int TPW_ = 4>
struct PbbStream {
  static constexpr int C = 128, HM = 8, TPW = TPW_;
  static constexpr int RS = PB_CW * TPW;  // tokens per stage
  static constexpr int ZB = RS * C * 2, DZB = RS * C * 4, SB = RS * 4, NBB = HM * RS * 4;
  static constexpr int STAGE = ((ZB + DZB + 2 * SB + NBB) + 127) / 128 * 128;
  static constexpr int W = C * HM + 3 * C;  // [dw | dgamma | dbeta | colsum(dz) (optional)]
  static constexpr int RED = PB_CW * W * 4;
  static constexpr int BYTES = (NST * STAGE > RED ? NST * STAGE : RED) + 2 * NST * 8;
};

template <int NST, int TPW_, int MINB>
__global__ void __launch_bounds__(PB_CW * 32 + 32, MINB) pair_bias_bwd_stream_kernel(
    const __nv_bfloat16* __restrict__ z, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ g, const float* __restrict__ bln, const float* __restrict__ w,
    const float* __restrict__ dnb, int swap_xy, float* dz, float* __restrict__ partials, int64_t NI,
    int64_t NJ, int H, __nv_bfloat16* __restrict__ dz16, int want_dzsum) {
  using M = PbbStream<NST, TPW_>;
  constexpr int C = M::C;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (M::BYTES - 2 * NST * 8));
  uint64_t* emp = bar + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t NT = NI * NJ;
  const int64_t nstage = (NT + M::RS - 1) / M::RS;
  const int64_t s0 = nstage * blockIdx.x / gridDim.x, s1 = nstage * (blockIdx.x + 1) / gridDim.x;
  const int n = (int)(s1 - s0);

  auto issue = [&](int it) {
    const int s = it % NST;
    const int64_t t0 = (s0 + it) * M::RS;
    const int nt = (int)(NT - t0 < M::RS ? NT - t0 : M::RS);
    uint8_t* st = sm + s * M::STAGE;
    const uint32_t zb = nt * C * 2, dzb = nt * C * 4, sb = nt * 4;
    mbar_expect_tx(&bar[s], zb + dzb + 2 * sb + (swap_xy ? 0 : H * sb));
    bulk_g2s(st, z + t0 * C, zb, &bar[s]);
    bulk_g2s(st + M::ZB, dz + t0 * C, dzb, &bar[s]);
    bulk_g2s(st + M::ZB + M::DZB, mean + t0, sb, &bar[s]);
    bulk_g2s(st + M::ZB + M::DZB + M::SB, rstd + t0, sb, &bar[s]);
    if (!swap_xy)
      for (int h = 0; h < H; ++h)
        bulk_g2s(st + M::ZB + M::DZB + 2 * M::SB + h * M::SB, dnb + h * NT + t0, sb, &bar[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&bar[s], 1);
      tc::mbar_init(&emp[s], PB_CW);
    }
  }
  __syncthreads();
  if (warp == PB_CW) {
    if (lane == 0) {
      for (int it = 0; it < n; ++it) {
        const int s = it % NST;
        if (it >= NST) tc::mbar_wait(&emp[s], (uint32_t)(((it / NST) - 1) & 1));
        issue(it);
      }
    }
    return;
  }
  // this lane's 4 channels: LN affine, w_bias rows, accumulators
  const int c0 = lane * 4;
  // this lane's 4 channels as two pairs on the paired fp32 pipes (FFMA2):
  // w2[j][hh] = w[c0+2j .. c0+2j+1, hh], dw2[e][q] = dw[c0+e, 2q .. 2q+1]
  float2 gg2[2], bb2[2], dgs2[2], dbs2[2], w2[2][M::HM], dw2[4][M::HM / 2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    gg2[j] = make_float2(g[c0 + 2 * j], g[c0 + 2 * j + 1]);
    bb2[j] = make_float2(bln[c0 + 2 * j], bln[c0 + 2 * j + 1]);
    dgs2[j] = dbs2[j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int hh = 0; hh < M::HM; ++hh)
      w2[j][hh] = hh < H ? make_float2(w[(c0 + 2 * j) * H + hh], w[(c0 + 2 * j + 1) * H + hh])
                         : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int q = 0; q < M::HM / 2; ++q) dw2[e][q] = make_float2(0.f, 0.f);
  // column sums of the updated dz (the next module's output-bias gradient)
  float2 dzs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int it = 0; it < n; ++it) {
    const int s = it % NST;
    const int64_t t0 = (s0 + it) * M::RS;
    const int nt = (int)(NT - t0 < M::RS ? NT - t0 : M::RS);
    const uint8_t* st = sm + s * M::STAGE;
    // swap_xy: this warp's dP values straight from global (transposed plane)
    float dpg[M::TPW];
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      const int tt = warp * M::TPW + u;
      dpg[u] = 0.f;
      if (swap_xy && tt < nt && lane < H) {
        const int64_t t = t0 + tt, x = t / NJ, y = t % NJ;
        dpg[u] = dnb[((int64_t)lane * NJ + y) * NI + x];
      }
    }
    tc::mbar_wait(&bar[s], (uint32_t)((it / NST) & 1));
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      const int tt = warp * M::TPW + u;
      if (tt < nt) {  // warp-uniform
      float dpm = dpg[u];
      if (!swap_xy && lane < H)
        dpm = reinterpret_cast<const float*>(st + M::ZB + M::DZB + 2 * M::SB + lane * M::SB)[tt];
      float dP[M::HM];
#pragma unroll
      for (int hh = 0; hh < M::HM; ++hh) dP[hh] = __shfl_sync(0xffffffffu, dpm, hh);
      const float mu = reinterpret_cast<const float*>(st + M::ZB + M::DZB)[tt];
      const float inv = reinterpret_cast<const float*>(st + M::ZB + M::DZB + M::SB)[tt];
      const uint2 zr = *reinterpret_cast<const uint2*>(st + (tt * C + c0) * 2);
      const float4 dzr = *reinterpret_cast<const float4*>(st + M::ZB + (tt * C + c0) * 4);
      const float2 mu2 = make_float2(-mu * inv, -mu * inv), inv2 = make_float2(inv, inv);
      // xh = (z - mu) * inv = z * inv - mu * inv ; zl = xh * g + b
      const float2 xh2[2] = {__ffma2_rn(tc::bf16x2_f2(zr.x), inv2, mu2), __ffma2_rn(tc::bf16x2_f2(zr.y), inv2, mu2)};
      float2 dzl2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int hh = 0; hh < M::HM; ++hh) {
        const float2 p2 = make_float2(dP[hh], dP[hh]);
        dzl2[0] = __ffma2_rn(p2, w2[0][hh], dzl2[0]);
        dzl2[1] = __ffma2_rn(p2, w2[1][hh], dzl2[1]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float2 zl2 = __ffma2_rn(xh2[j], gg2[j], bb2[j]);
        const float zl[2] = {zl2.x, zl2.y};
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const float2 z2 = make_float2(zl[e2], zl[e2]);
#pragma unroll
          for (int q = 0; q < M::HM / 2; ++q)
            dw2[2 * j + e2][q] = __ffma2_rn(z2, make_float2(dP[2 * q], dP[2 * q + 1]), dw2[2 * j + e2][q]);
        }
        dgs2[j] = __ffma2_rn(dzl2[j], xh2[j], dgs2[j]);
        dbs2[j] = __fadd2_rn(dbs2[j], dzl2[j]);
      }
      const float2 dxh2[2] = {__fmul2_rn(dzl2[0], gg2[0]), __fmul2_rn(dzl2[1], gg2[1])};
      const float s1 = (dxh2[0].x + dxh2[0].y) + (dxh2[1].x + dxh2[1].y);
      const float2 t2 = __ffma2_rn(dxh2[0], xh2[0], __fmul2_rn(dxh2[1], xh2[1]));
      const float s2 = t2.x + t2.y;
      const float m1 = group_sum<32>(s1) / (float)C, m2 = group_sum<32>(s2) / (float)C;
      // dz += inv * (dxh - m1 - xh * m2)
      const float2 nm1 = make_float2(-m1, -m1), nm2 = make_float2(-m2, -m2);
      const float2 o0 = __ffma2_rn(inv2, __ffma2_rn(xh2[0], nm2, __fadd2_rn(dxh2[0], nm1)), make_float2(dzr.x, dzr.y));
      const float2 o1 = __ffma2_rn(inv2, __ffma2_rn(xh2[1], nm2, __fadd2_rn(dxh2[1], nm1)), make_float2(dzr.z, dzr.w));
      *reinterpret_cast<float4*>(dz + (t0 + tt) * C + c0) = make_float4(o0.x, o0.y, o1.x, o1.y);
      if (dz16)  // the next module's bf16 operand
        *reinterpret_cast<uint2*>(dz16 + (t0 + tt) * C + c0) =
            make_uint2(tc::pack_bf16(o0.x, o0.y), tc::pack_bf16(o1.x, o1.y));
      if (want_dzsum) {
        dzs2[0] = __fadd2_rn(dzs2[0], o0);
        dzs2[1] = __fadd2_rn(dzs2[1], o1);
      }
      }
    }
    tc::mbar_arrive_warp(&emp[s]);
  }
  asm volatile("bar.sync 1, %0;" ::"r"(PB_CW * 32) : "memory");
  float* red = reinterpret_cast<float*>(sm);
  float* mine = red + warp * M::W;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
#pragma unroll
    for (int hh = 0; hh < M::HM; ++hh)
      if (hh < H) mine[(c0 + e) * H + hh] = (hh & 1) ? dw2[e][hh / 2].y : dw2[e][hh / 2].x;
    mine[C * H + c0 + e] = (e & 1) ? dgs2[e / 2].y : dgs2[e / 2].x;
    mine[C * H + C + c0 + e] = (e & 1) ? dbs2[e / 2].y : dbs2[e / 2].x;
    mine[C * H + 2 * C + c0 + e] = (e & 1) ? dzs2[e / 2].y : dzs2[e / 2].x;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(PB_CW * 32) : "memory");
  const int Wd = C * H + (want_dzsum ? 3 : 2) * C;
  for (int c = tid; c < Wd; c += PB_CW * 32) {
    float acc = 0.f;
    for (int q = 0; q < PB_CW; ++q) acc += red[q * M::W + c];
    partials[(int64_t)blockIdx.x * Wd + c] = acc;
  }
}


// LayerNorm forward (src/tensor.py:173-188): y = (x - mean) * rstd * g + b in the
// output dtype, plus the row statistics.  Warp-per-row (C = 256) or two rows per
// warp (C = 128), TPW row steps per warp and stage; x arrives by bulk copy.
template <int C, typename TY, int NST>
struct LnfStream {
  static constexpr int LANES = C / 8 < 32 ? C / 8 : 32;
  static constexpr int RPW = 32 / LANES;
  static constexpr int TPW = 4;
  static constexpr int RS = (ST / 32) * RPW * TPW;
  static constexpr int STAGE = (RS * C * 2 + 127) / 128 * 128;
  static constexpr int BYTES = NST * STAGE + 2 * NST * 8;
};

template <int C, typename TY, int NST>
__global__ void __launch_bounds__(ST + 32) ln_fwd_stream_kernel(const __nv_bfloat16* __restrict__ x,
                                                                const float* __restrict__ g,
                                                                const float* __restrict__ b, TY* __restrict__ y,
                                                                float* __restrict__ mean, float* __restrict__ rstd,
                                                                int64_t rows, float eps) {
  using M = LnfStream<C, TY, NST>;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NST * M::STAGE);
  uint64_t* emp = bar + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int l = lane % M::LANES, gi = lane / M::LANES;
  const int64_t nstage = (rows + M::RS - 1) / M::RS;
  const int64_t s0 = nstage * blockIdx.x / gridDim.x, s1 = nstage * (blockIdx.x + 1) / gridDim.x;
  const int n = (int)(s1 - s0);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&bar[s], 1);
      tc::mbar_init(&emp[s], ST / 32);
    }
  }
  __syncthreads();
  if (warp == ST / 32) {
    if (lane == 0) {
      for (int it = 0; it < n; ++it) {
        const int s = it % NST;
        if (it >= NST) tc::mbar_wait(&emp[s], (uint32_t)(((it / NST) - 1) & 1));
        const int64_t r0 = (s0 + it) * M::RS;
        const int nr = (int)(rows - r0 < M::RS ? rows - r0 : M::RS);
        mbar_expect_tx(&bar[s], nr * C * 2);
        bulk_g2s(sm + s * M::STAGE, x + r0 * C, nr * C * 2, &bar[s]);
      }
    }
    return;
  }
  float gg[8], bb[8];
  ld8(g + l * 8, gg);
  ld8(b + l * 8, bb);
  for (int it = 0; it < n; ++it) {
    const int s = it % NST;
    const int64_t r0 = (s0 + it) * M::RS;
    const int nr = (int)(rows - r0 < M::RS ? rows - r0 : M::RS);
    tc::mbar_wait(&bar[s], (uint32_t)((it / NST) & 1));
    const __nv_bfloat16* st = reinterpret_cast<const __nv_bfloat16*>(sm + s * M::STAGE);
    float v[M::TPW][8];
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      const int rr = (warp * M::TPW + u) * M::RPW + gi;
      ld8(st + (rr < nr ? rr : 0) * C + l * 8, v[u]);
    }
    tc::mbar_arrive_warp(&emp[s]);  // the stage is in registers
    float mu[M::TPW], inv[M::TPW];
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      float sum = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) sum += v[u][e];
      mu[u] = group_sum<M::LANES>(sum) / (float)C;
    }
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      float q = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[u][e] - mu[u];
        q += d * d;
      }
      inv[u] = rsqrtf(group_sum<M::LANES>(q) / (float)C + eps);
    }
#pragma unroll
    for (int u = 0; u < M::TPW; ++u) {
      const int rr = (warp * M::TPW + u) * M::RPW + gi;
      if (rr < nr) {
        const int64_t r = r0 + rr;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[u][e] - mu[u]) * inv[u] * gg[e] + bb[e];
        st8(y + r * C + l * 8, o);
        if (l == 0) {
          if (mean) mean[r] = mu[u];
          if (rstd) rstd[r] = inv[u];
        }
      }
    }
  }
}

}  // namespace

// Returns false (caller falls back) for shapes this path does not cover.
bool ln_bwd_stream(const void* x, int xdt, const void* dy, int dydt, const float* mean, const float* rstd,
                   const float* g, const float* dres, float* dx, __nv_bfloat16* dx16, float* dgamma,
                   float* dbeta, float* dxsum, int accumulate, void* ws, int64_t rows, int64_t C,
                   int64_t ws_blocks, cudaStream_t s) {
  static const bool off = [] {
    const char* e = getenv("EVO_GLUE_STREAM");
    return e && e[0] == '0';
  }();
  if (off || (C != 128 && C != 256) || xdt != EVO_BF16 || (rows % 4) != 0 || rows < 4096) return false;
  const uintptr_t al = (uintptr_t)x | (uintptr_t)dy | (uintptr_t)dx | (uintptr_t)dres | (uintptr_t)dx16 |
                       (uintptr_t)mean | (uintptr_t)rstd;
  if (al & 15) return false;
  constexpr int NST = 4;
  const int64_t want = 2 * (int64_t)num_sms();
  const unsigned grid = (unsigned)(want < ws_blocks ? want : ws_blocks);
  bool done = false;
  auto go = [&](auto cc, auto td) {
    constexpr int CC = decltype(cc)::value;
    using TD = typename decltype(td)::type;
    using M = LnbStream<CC, __nv_bfloat16, TD, NST>;
    auto k = ln_bwd_stream_kernel<CC, __nv_bfloat16, TD, NST>;
    static bool attr = false;
    if (!attr) {
      EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, M::BYTES));
      attr = true;
    }
    k<<<grid, ST + 32, M::BYTES, s>>>((const __nv_bfloat16*)x, (const TD*)dy, mean, rstd, g, dres, dx, dx16,
                                      (float*)ws, rows, dxsum != nullptr);
    done = true;
  };
  struct F32 { using type = float; };
  struct B16 { using type = __nv_bfloat16; };
  if (C == 256 && dydt == EVO_F32) go(std::integral_constant<int, 256>{}, F32{});
  else if (C == 128 && dydt == EVO_F32) go(std::integral_constant<int, 128>{}, F32{});
  else if (C == 256 && dydt == EVO_BF16) go(std::integral_constant<int, 256>{}, B16{});
  else if (C == 128 && dydt == EVO_BF16) go(std::integral_constant<int, 128>{}, B16{});
  if (!done) return false;
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials((const float*)ws, grid, C, dgamma, accumulate, s, 3 * C);
  finalize_partials((const float*)ws + C, grid, C, dbeta, accumulate, s, 3 * C);
  if (dxsum) finalize_partials((const float*)ws + 2 * C, grid, C, dxsum, 0, s, 3 * C);
  return true;
}

}  // namespace evo

namespace evo {

bool pair_bias_bwd_stream_ok(const void* z, int dt, const void* dz, const void* dz16, const float* mean,
                             const float* rstd, const float* dnb, int64_t NI, int64_t NJ, int64_t C, int64_t H) {
  static const bool off = [] {
    const char* e = getenv("EVO_GLUE_STREAM");
    return e && e[0] == '0';
  }();
  const int64_t NT = NI * NJ;
  if (off || C != 128 || H > 8 || dt != EVO_BF16 || (NT % 4) != 0 || NT < 4096) return false;
  return ((((uintptr_t)z | (uintptr_t)dz | (uintptr_t)mean | (uintptr_t)rstd | (uintptr_t)dnb) & 15) == 0 &&
          (((uintptr_t)dz16) & 7) == 0);
}

bool pair_bias_bwd_stream(const void* z, int dt, const float* mean, const float* rstd, const float* g,
                          const float* bln, const float* w, const float* dnb, int swap, float* dz, float* dg,
                          float* db, float* dw, int accumulate, void* ws, int64_t NI, int64_t NJ, int64_t C,
                          int64_t H, int64_t ws_blocks, cudaStream_t s, __nv_bfloat16* dz16, float* dzsum) {
  if (!pair_bias_bwd_stream_ok(z, dt, dz, dz16, mean, rstd, dnb, NI, NJ, C, H)) return false;
  // tokens per warp and stage x resident blocks per SM; sweep knob
  // EVO_PBB_CFG = "<tpw><minb>" (tools/time_glue.py: 43 45.9 us, 23 47.3,
  // 24 55.9 (spills), 82 38.4-39.7, 162 43.3, 161 50.6, 81 46.6 -- more
  // tokens in flight per warp beat more resident warps)
  static const int cfg = [] {
    const char* e = getenv("EVO_PBB_CFG");
    return e ? atoi(e) : 82;
  }();
  auto launch = [&](auto kern, int bytes, int minb) {
    static bool attr_done[16] = {};
    const int key = (cfg % 16) & 15;
    if (!attr_done[key]) {
      EVO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      attr_done[key] = true;
    }
    const int64_t want = minb * (int64_t)num_sms();
    const unsigned grid = (unsigned)(want < ws_blocks ? want : ws_blocks);
    kern<<<grid, PB_CW * 32 + 32, bytes, s>>>((const __nv_bfloat16*)z, mean, rstd, g, bln, w, dnb, swap, dz,
                                               (float*)ws, NI, NJ, (int)H, dz16, dzsum != nullptr);
    return grid;
  };
  unsigned grid;
  constexpr int NST = 4;
  if (cfg == 24) grid = launch(pair_bias_bwd_stream_kernel<NST, 2, 4>, PbbStream<NST, 2>::BYTES, 4);
  else if (cfg == 23) grid = launch(pair_bias_bwd_stream_kernel<NST, 2, 3>, PbbStream<NST, 2>::BYTES, 3);
  else if (cfg == 82) grid = launch(pair_bias_bwd_stream_kernel<NST, 8, 2>, PbbStream<NST, 8>::BYTES, 2);
  else if (cfg == 162) grid = launch(pair_bias_bwd_stream_kernel<2, 16, 2>, PbbStream<2, 16>::BYTES, 2);
  else if (cfg == 161) grid = launch(pair_bias_bwd_stream_kernel<3, 16, 1>, PbbStream<3, 16>::BYTES, 1);
  else if (cfg == 81) grid = launch(pair_bias_bwd_stream_kernel<6, 8, 1>, PbbStream<6, 8>::BYTES, 1);
  else grid = launch(pair_bias_bwd_stream_kernel<NST, 4, 3>, PbbStream<NST, 4>::BYTES, 3);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  const int64_t W = C * H + (dzsum ? 3 : 2) * C;
  finalize_partials((const float*)ws, grid, C * H, dw, accumulate, s, W);
  finalize_partials((const float*)ws + C * H, grid, C, dg, accumulate, s, W);
  finalize_partials((const float*)ws + C * H + C, grid, C, db, accumulate, s, W);
  if (dzsum) finalize_partials((const float*)ws + C * H + 2 * C, grid, C, dzsum, 0, s, W);
  return true;
}

}  // namespace evo

namespace evo {

bool ln_fwd_stream(const void* x, int xdt, const float* g, const float* b, void* y, int ydt, float* mean,
                   float* rstd, int64_t rows, int64_t C, float eps, cudaStream_t s) {
  static const bool off = [] {
    const char* e = getenv("EVO_GLUE_STREAM");
    return e && e[0] == '0';
  }();
  if (off || (C != 128 && C != 256) || xdt != EVO_BF16 || rows < 4096) return false;
  if (((uintptr_t)x | (uintptr_t)y) & 15) return false;
  constexpr int NST = 4;
  // resident blocks per SM (EVO_LNF_BPS sweep, tools/time_glue.py: 1 -> 7.7 us,
  // 2 -> 7.1 us, 3 -> 9.1 us at the pair shape)
  static const int bps = [] {
    const char* e = getenv("EVO_LNF_BPS");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= 3 ? v : 2;
  }();
  const unsigned grid = (unsigned)(bps * num_sms());
  bool done = false;
  auto go = [&](auto cc, auto ty) {
    constexpr int CC = decltype(cc)::value;
    using TY = typename decltype(ty)::type;
    using M = LnfStream<CC, TY, NST>;
    auto k = ln_fwd_stream_kernel<CC, TY, NST>;
    static bool attr = false;
    if (!attr) {
      EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, M::BYTES));
      attr = true;
    }
    k<<<grid, ST + 32, M::BYTES, s>>>((const __nv_bfloat16*)x, g, b, (TY*)y, mean, rstd, rows, eps);
    done = true;
  };
  struct F32 { using type = float; };
  struct B16 { using type = __nv_bfloat16; };
  if (C == 256 && ydt == EVO_BF16) go(std::integral_constant<int, 256>{}, B16{});
  else if (C == 128 && ydt == EVO_BF16) go(std::integral_constant<int, 128>{}, B16{});
  else if (C == 256 && ydt == EVO_F32) go(std::integral_constant<int, 256>{}, F32{});
  else if (C == 128 && ydt == EVO_F32) go(std::integral_constant<int, 128>{}, F32{});
  if (!done) return false;
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

}  // namespace evo
