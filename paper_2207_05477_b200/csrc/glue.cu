// Vectorised bandwidth-bound glue: LayerNorm fwd/bwd, bias/residual/ReLU
// epilogues, deterministic column sums, pair-bias projection, OPM re-layout.
//
// Design rules (HBM-bound, B200): every access is a 16-byte vector (8
// channels of one token row); a row is spread over C/8 lanes so a warp covers
// 32/(C/8) rows per iteration; blocks own contiguous row ranges (DRAM page
// locality); reductions over rows go through per-block partials reduced in a
// fixed order (reduce.cuh) -- no atomics, bitwise reproducible.
// These kernels serve the storage dtypes of the engine (bf16 or fp32 rows)
// whenever C is a power of two in [32, 1024]; other widths use the scalar
// kernels in layernorm.cu / api.cu / pair_bias.cu / opm.cu.
#include <algorithm>

#include "common.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace evo {

namespace {

constexpr int GT = 256;  // threads per block for all glue kernels

inline bool pow2_width(int64_t C) { return C >= 32 && C <= 1024 && (C & (C - 1)) == 0; }

// Streaming kernels (no partials) take up to 16 blocks per SM so every warp
// has its loads in flight at once; kernels writing per-block partials are
// capped at PARTIAL_PER_SM blocks per SM (bounded partial rows).
constexpr int PARTIAL_PER_SM = 2;
constexpr int EW_UNROLL = 4;          // 16-B vectors per thread in flight in the elementwise kernels
constexpr int PB_PARTIAL_PER_SM = 3;  // pair-bias backward: partial rows for up to 3 blocks per SM
inline unsigned glue_grid(int64_t rows, int rows_per_iter, int per_sm = 16) {
  int64_t want = (rows + rows_per_iter - 1) / rows_per_iter;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (want > cap) want = cap;
  return (unsigned)(want > 0 ? want : 1);
}

// 16 channels (two 16-B chunks) per lane: the per-row shuffle reductions are
// amortised over twice the elements of an 8-channel mapping
template <int C>
struct RowMap {
  static constexpr int LANES = (C / 16) < 2 ? 2 : ((C / 16) < 32 ? (C / 16) : 32);  // lanes per row
  static constexpr int CH = C / (8 * LANES);                                        // 8-chunks per lane
  static constexpr int RPW = 32 / LANES;                      // rows per warp
  static constexpr int GROUPS = GT / LANES;                   // rows per block iteration
};

// ---------------------------------------------------------------------------
// LayerNorm forward

// rows a thread group keeps in flight per iteration: every load of the U rows
// is issued before the first reduction, so each thread has U x 16 B (bf16) or
// U x 32 B (fp32) outstanding -- what HBM3e needs to stay busy at 2048
// threads per SM
template <int C>
struct Unroll {
  static constexpr int value = RowMap<C>::CH >= 4 ? 1 : 4 / RowMap<C>::CH;
};

template <int C, typename TX, typename TY>
__global__ void __launch_bounds__(GT) ln_fwd_vec_kernel(const TX* __restrict__ x,
                                                        const float* __restrict__ g,
                                                        const float* __restrict__ b,
                                                        TY* __restrict__ y, float* __restrict__ mean,
                                                        float* __restrict__ rstd, int64_t rows, float eps) {
  using M = RowMap<C>;
  constexpr int U = Unroll<C>::value;
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  float gg[M::CH][8], bb[M::CH][8];  // this lane's affine parameters, loaded once
#pragma unroll
  for (int k = 0; k < M::CH; ++k) {
    ld8(g + (k * M::LANES + l) * 8, gg[k]);
    ld8(b + (k * M::LANES + l) * 8, bb[k]);
  }
  // block-uniform trip count: the row groups of a warp always shuffle together
  for (int64_t rb = blockIdx.x * (int64_t)(M::GROUPS * U); rb < rows;
       rb += (int64_t)gridDim.x * M::GROUPS * U) {
    float v[U][M::CH][8];
    int64_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rr = rb + u * M::GROUPS + grp;
      r[u] = rr < rows ? rr : rows - 1;
#pragma unroll
      for (int k = 0; k < M::CH; ++k) ld8(x + r[u] * C + (k * M::LANES + l) * 8, v[u][k]);
    }
    float mu[U], inv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[u][k][e];
      mu[u] = group_sum<M::LANES>(s) / (float)C;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[u][k][e] - mu[u];
          q += d * d;
        }
      inv[u] = rsqrtf(group_sum<M::LANES>(q) / (float)C + eps);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool act = rb + u * M::GROUPS + grp < rows;
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 8;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[u][k][e] - mu[u]) * inv[u] * gg[k][e] + bb[k][e];
        if (act) st8(y + r[u] * C + c0, o);
      }
      if (act && l == 0) {
        if (mean) mean[r[u]] = mu[u];
        if (rstd) rstd[r[u]] = inv[u];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// LayerNorm backward: dx = dres + LN'(dy); optional bf16 copy of dx and column
// sums of dx (the next module's output-bias gradient); dgamma/dbeta partials.
// partial layout per block: [dgamma C | dbeta C | colsum(dx) C]

template <int C, typename TX, typename TD>
__global__ void __launch_bounds__(GT) ln_bwd_vec_kernel(
    const TX* __restrict__ x, const TD* __restrict__ dy, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* dres, float* dx,
    __nv_bfloat16* __restrict__ dx16, float* __restrict__ partials, int64_t rows, int want_dxsum) {
  using M = RowMap<C>;
  extern __shared__ float sm[];  // [GROUPS][3C]
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  const int64_t r0 = (rows * blockIdx.x) / gridDim.x, r1 = (rows * (blockIdx.x + 1)) / gridDim.x;
  float dg[M::CH][8], db[M::CH][8], dsx[M::CH][8], gg[M::CH][8];
#pragma unroll
  for (int k = 0; k < M::CH; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      dg[k][e] = db[k][e] = dsx[k][e] = 0.f;
      gg[k][e] = g[(k * M::LANES + l) * 8 + e];
    }
  constexpr int U = M::CH == 1 ? 2 : 1;  // rows in flight per thread group
  for (int64_t rb = r0; rb < r1; rb += M::GROUPS * U) {
    int64_t r[U];
    float w[U], mu[U], inv[U];
    float xh[U][M::CH][8], dxh[U][M::CH][8], o[U][M::CH][8];
    // issue every load of the U rows first (x, dy, dres), then reduce
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool act = rb + u * M::GROUPS + grp < r1;
      r[u] = act ? rb + u * M::GROUPS + grp : r1 - 1;
      w[u] = act ? 1.f : 0.f;
      mu[u] = mean[r[u]];
      inv[u] = rstd[r[u]];
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 8;
        ld8(x + r[u] * C + c0, xh[u][k]);
        ld8(dy + r[u] * C + c0, dxh[u][k]);
        if (dres) {
          ld8(dres + r[u] * C + c0, o[u][k]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) o[u][k][e] = 0.f;
        }
      }
    }
    float m1[U], m2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = dxh[u][k][e] * w[u];
          xh[u][k][e] = (xh[u][k][e] - mu[u]) * inv[u];
          dxh[u][k][e] = d * gg[k][e];
          dg[k][e] += d * xh[u][k][e];
          db[k][e] += d;
          s1 += dxh[u][k][e];
          s2 += dxh[u][k][e] * xh[u][k][e];
        }
      m1[u] = group_sum<M::LANES>(s1) / (float)C;
      m2[u] = group_sum<M::LANES>(s2) / (float)C;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          o[u][k][e] += inv[u] * (dxh[u][k][e] - m1[u] - xh[u][k][e] * m2[u]);
          dsx[k][e] += w[u] * o[u][k][e];
        }
        if (w[u] != 0.f) {
          st8(dx + r[u] * C + c0, o[u][k]);
          if (dx16) st8(dx16 + r[u] * C + c0, o[u][k]);
        }
      }
    }
  }
  float* mine = sm + grp * 3 * C;
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
  __syncthreads();
  const int W = want_dxsum ? 3 * C : 2 * C;
  for (int c = threadIdx.x; c < W; c += GT) {
    float acc = 0.f;
    for (int q = 0; q < M::GROUPS; ++q) acc += sm[q * 3 * C + c];
    partials[(int64_t)blockIdx.x * 3 * C + c] = acc;
  }
}

// ---------------------------------------------------------------------------
// column sums (bias gradients), with optional ReLU-backward mask and cast copy
// MODE 0: v = x;  MODE 1: v = x * (h > 0), written back into x

template <typename TX, typename TY, int MODE>
__global__ void __launch_bounds__(GT) colsum_vec_kernel(TX* x, int64_t ldx, const TX* __restrict__ h,
                                                        TY* __restrict__ y, float* __restrict__ partials,
                                                        int64_t rows, int C) {
  extern __shared__ float sm[];  // [RPB][C]
  const int TPR = C / 8;
  const int RPB = GT / TPR;
  const int ct = threadIdx.x % TPR, rg = threadIdx.x / TPR;
  const int64_t r0 = (rows * blockIdx.x) / gridDim.x, r1 = (rows * (blockIdx.x + 1)) / gridDim.x;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  constexpr int U = 4;  // rows in flight per thread: all loads before any store
  for (int64_t rb = r0 + rg; rb < r1; rb += (int64_t)RPB * U) {
    Vec8<TX> vx[U], vh[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = rb + (int64_t)u * RPB;
      if (r < r1) {
        ldv8(x + r * ldx + ct * 8, vx[u]);
        if (MODE == 1) ldv8(h + r * C + ct * 8, vh[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = rb + (int64_t)u * RPB;
      if (r >= r1) continue;  // rows ascend with u: acc sees rows in order
      float v[8];
      cvt8(vx[u], v);
      if (MODE == 1) {
        float hv[8];
        cvt8(vh[u], hv);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = hv[e] > 0.f ? v[e] : 0.f;
        st8(x + r * ldx + ct * 8, v);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
      if (y) st8(y + r * C + ct * 8, v);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) sm[rg * C + ct * 8 + e] = acc[e];
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += GT) {
    float a = 0.f;
    for (int q = 0; q < RPB; ++q) a += sm[q * C + c];
    partials[(int64_t)blockIdx.x * C + c] = a;
  }
}

// ---------------------------------------------------------------------------
// elementwise epilogues

template <typename TR, typename TY, typename TO>
__global__ void __launch_bounds__(GT) bias_residual_vec_kernel(const TR* __restrict__ res,
                                                               const TY* __restrict__ y,
                                                               const float* __restrict__ bias,
                                                               TO* __restrict__ out, int64_t n8, int C8) {
  constexpr int U = EW_UNROLL;
  for (int64_t e0 = blockIdx.x * (int64_t)(GT * U) + threadIdx.x; e0 < n8; e0 += (int64_t)gridDim.x * GT * U) {
    Vec8<TY> vy[U];
    Vec8<TR> vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * GT;
      if (e < n8) {
        ldv8(y + e * 8, vy[u]);
        if (res) ldv8(res + e * 8, vr[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * GT;
      if (e >= n8) continue;
      const int c0 = (int)(e % C8) * 8;
      float v[8];
      cvt8(vy[u], v);
      if (bias) {
        float bv[8];
        ld8(bias + c0, bv);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += bv[k];
      }
      if (res) {
        float r[8];
        cvt8(vr[u], r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = r[k] + v[k];
      }
      st8(out + e * 8, v);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(GT) bias_relu_vec_kernel(T* __restrict__ y, const float* __restrict__ bias,
                                                           int64_t n8, int C8) {
  constexpr int U = EW_UNROLL;
  for (int64_t e0 = blockIdx.x * (int64_t)(GT * U) + threadIdx.x; e0 < n8; e0 += (int64_t)gridDim.x * GT * U) {
    Vec8<T> vy[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * GT;
      if (e < n8) ldv8(y + e * 8, vy[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * GT;
      if (e >= n8) continue;
      const int c0 = (int)(e % C8) * 8;
      float v[8], bv[8];
      cvt8(vy[u], v);
      if (bias) {
        ld8(bias + c0, bv);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) bv[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = fmaxf(v[k] + bv[k], 0.f);
      st8(y + e * 8, v);
    }
  }
}

// ---------------------------------------------------------------------------
// pair bias: nb[h, x, y] (or [h, y, x]) = LN(z[x, y]) . w[:, h]
//
// A token row is spread over PB_LANES lanes with 4 channels each (8-byte bf16
// / 16-byte fp32 accesses), so a lane's slice of w (4 channels x 8 heads) and,
// in the backward, of dw stay in registers at ~100 registers per thread; two
// tokens per row group are in flight per iteration.  The 8 per-head dot
// products are reduced across the row group by a halving butterfly (8 -> 4
// -> 2 -> 1 values per lane, then plain sums): 9 shuffles per token instead
// of 8 full reductions.

template <int C>
struct PbMap {
  static constexpr int LANES = (C / 4) < 32 ? (C / 4) : 32;  // lanes per token
  static constexpr int CH = C / (4 * LANES);                  // 4-channel chunks per lane
  static constexpr int GROUPS = GT / LANES;                   // tokens per block iteration
  static constexpr int U = 2;                                 // tokens in flight per row group
};

// p[h]: this lane's partial dot product for head h.  Returns the sum over the
// row group's LANES lanes for head pb_head<LANES>(l).
template <int LANES>
__device__ __forceinline__ float head_reduce8(const float (&p)[8], int l) {
  static_assert(LANES >= 8, "head butterfly needs >= 8 lanes per token");
  float q4[4], q2[2];
  {
    const bool hi = (l & (LANES / 2)) != 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      q4[j] = (hi ? p[j + 4] : p[j]) + __shfl_xor_sync(0xffffffffu, hi ? p[j] : p[j + 4], LANES / 2);
  }
  {
    const bool hi = (l & (LANES / 4)) != 0;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      q2[j] = (hi ? q4[j + 2] : q4[j]) + __shfl_xor_sync(0xffffffffu, hi ? q4[j] : q4[j + 2], LANES / 4);
  }
  const bool hi = (l & (LANES / 8)) != 0;
  float q = (hi ? q2[1] : q2[0]) + __shfl_xor_sync(0xffffffffu, hi ? q2[0] : q2[1], LANES / 8);
#pragma unroll
  for (int o = LANES / 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  return q;
}
template <int LANES>
__device__ __forceinline__ int pb_head(int l) {
  return ((l & (LANES / 2)) ? 4 : 0) | ((l & (LANES / 4)) ? 2 : 0) | ((l & (LANES / 8)) ? 1 : 0);
}

template <int C, typename T>
__global__ void __launch_bounds__(GT) pair_bias_fwd_vec_kernel(
    const T* __restrict__ z, const float* __restrict__ g, const float* __restrict__ b,
    const float* __restrict__ w, T* __restrict__ nb, float* __restrict__ mean,
    float* __restrict__ rstd, int64_t NI, int64_t NJ, int H, int swap_xy) {
  using M = PbMap<C>;
  constexpr int U = M::U;
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  float gg[M::CH][4], bb[M::CH][4], wr[M::CH][4][8];
#pragma unroll
  for (int k = 0; k < M::CH; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = (k * M::LANES + l) * 4 + e;
      gg[k][e] = g[c];
      bb[k][e] = b[c];
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) wr[k][e][hh] = hh < H ? w[c * H + hh] : 0.f;
    }
  const int hme = pb_head<M::LANES>(l);
  const bool writer = (l & (M::LANES / 8 - 1)) == 0 && hme < H;
  const int64_t NT = NI * NJ;
  for (int64_t tb = blockIdx.x * (int64_t)(M::GROUPS * U); tb < NT; tb += (int64_t)gridDim.x * M::GROUPS * U) {
    float v[U][M::CH][4];
    int64_t t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t tt = tb + u * M::GROUPS + grp;
      t[u] = tt < NT ? tt : NT - 1;
#pragma unroll
      for (int k = 0; k < M::CH; ++k) ld4(z + t[u] * C + (k * M::LANES + l) * 4, v[u][k]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) s += v[u][k][e];
      const float mu = group_sum<M::LANES>(s) / (float)C;
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float d = v[u][k][e] - mu;
          q += d * d;
        }
      const float inv = rsqrtf(group_sum<M::LANES>(q) / (float)C + 1e-5f);
      float p[8];
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) p[hh] = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float zl = (v[u][k][e] - mu) * inv * gg[k][e] + bb[k][e];
#pragma unroll
          for (int hh = 0; hh < 8; ++hh) p[hh] = fmaf(zl, wr[k][e][hh], p[hh]);
        }
      const float mine = head_reduce8<M::LANES>(p, l);
      const bool act = tb + u * M::GROUPS + grp < NT;
      if (act && writer) {
        const int64_t x = t[u] / NJ, y = t[u] % NJ;
        const int64_t o = swap_xy ? ((int64_t)hme * NJ + y) * NI + x : ((int64_t)hme * NI + x) * NJ + y;
        nb[o] = from_f<T>(mine);
      }
      if (act && l == 0) {
        mean[t[u]] = mu;
        rstd[t[u]] = inv;
      }
    }
  }
}

// partial layout per block: [dw (C*H) | dgamma (C) | dbeta (C)]
template <int C, typename T>
__global__ void __launch_bounds__(GT) pair_bias_bwd_vec_kernel(
    const T* __restrict__ z, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ g, const float* __restrict__ bln, const float* __restrict__ w,
    const float* __restrict__ dnb, int swap_xy, float* __restrict__ dz,
    float* __restrict__ partials, int64_t NI, int64_t NJ, int H) {
  using M = PbMap<C>;
  constexpr int U = M::U;
  extern __shared__ float red[];  // [GROUPS][C*H + 2C]
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  float gg[M::CH][4], bb[M::CH][4], wr[M::CH][4][8], dw[M::CH][4][8], dgs[M::CH][4], dbs[M::CH][4];
#pragma unroll
  for (int k = 0; k < M::CH; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = (k * M::LANES + l) * 4 + e;
      gg[k][e] = g[c];
      bb[k][e] = bln[c];
      dgs[k][e] = dbs[k][e] = 0.f;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        wr[k][e][hh] = hh < H ? w[c * H + hh] : 0.f;
        dw[k][e][hh] = 0.f;
      }
    }
  const int base = (threadIdx.x & 31) - l;  // first lane of this row group
  const int64_t NT = NI * NJ;
  const int64_t t0 = (NT * blockIdx.x) / gridDim.x, t1 = (NT * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tb = t0; tb < t1; tb += M::GROUPS * U) {
    int64_t t[U];
    bool act[U];
    float dpm[U], mu[U], inv[U];
    float v[U][M::CH][4], o[U][M::CH][4];
    // every load of the U tokens first: z, dz, dnb, statistics
#pragma unroll
    for (int u = 0; u < U; ++u) {
      act[u] = tb + u * M::GROUPS + grp < t1;
      t[u] = act[u] ? tb + u * M::GROUPS + grp : t1 - 1;
      const int64_t x = t[u] / NJ, y = t[u] % NJ;
      dpm[u] = 0.f;
      if (act[u] && l < H) {  // inactive groups carry dP = 0: no contribution anywhere
        const int64_t od = swap_xy ? ((int64_t)l * NJ + y) * NI + x : ((int64_t)l * NI + x) * NJ + y;
        dpm[u] = dnb[od];
      }
      mu[u] = mean[t[u]];
      inv[u] = rstd[t[u]];
#pragma unroll
      for (int k = 0; k < M::CH; ++k) {
        const int c0 = (k * M::LANES + l) * 4;
        ld4(z + t[u] * C + c0, v[u][k]);
        if (act[u]) {
          ld4(dz + t[u] * C + c0, o[u][k]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) o[u][k][e] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float dP[8];
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) dP[hh] = __shfl_sync(0xffffffffu, dpm[u], base + hh);
      float xh[M::CH][4], dxh[M::CH][4];
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < M::CH; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          xh[k][e] = (v[u][k][e] - mu[u]) * inv[u];
          const float zl = xh[k][e] * gg[k][e] + bb[k][e];
          float dzl = 0.f;
#pragma unroll
          for (int hh = 0; hh < 8; ++hh) {
            dzl = fmaf(dP[hh], wr[k][e][hh], dzl);
            dw[k][e][hh] = fmaf(zl, dP[hh], dw[k][e][hh]);
          }
          dgs[k][e] += dzl * xh[k][e];
          dbs[k][e] += dzl;
          dxh[k][e] = dzl * gg[k][e];
          s1 += dxh[k][e];
          s2 += dxh[k][e] * xh[k][e];
        }
      const float m1 = group_sum<M::LANES>(s1) / (float)C, m2 = group_sum<M::LANES>(s2) / (float)C;
      if (act[u]) {
#pragma unroll
        for (int k = 0; k < M::CH; ++k) {
#pragma unroll
          for (int e = 0; e < 4; ++e) o[u][k][e] += inv[u] * (dxh[k][e] - m1 - xh[k][e] * m2);
          st4(dz + t[u] * C + (k * M::LANES + l) * 4, o[u][k]);
        }
      }
    }
  }
  const int W = C * H + 2 * C;
  float* mine = red + grp * W;
#pragma unroll
  for (int k = 0; k < M::CH; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = (k * M::LANES + l) * 4 + e;
#pragma unroll
      for (int hh = 0; hh < 8; ++hh)
        if (hh < H) mine[c * H + hh] = dw[k][e][hh];
      mine[C * H + c] = dgs[k][e];
      mine[C * H + C + c] = dbs[k][e];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += GT) {
    float acc = 0.f;
    for (int q = 0; q < M::GROUPS; ++q) acc += red[q * W + c];
    partials[(int64_t)blockIdx.x * W + c] = acc;
  }
}

// ---------------------------------------------------------------------------
// OPM re-layout: outn[i*R + j, p*k + q] = num[i*k + p, j*k + q] * rec[i*R + j]
// block per (i, tile of JT consecutive j); k = 32 staged through shared memory

constexpr int OPM_K = 32, OPM_JT = 8;

template <typename TI, typename TO, bool FWD>
__global__ void __launch_bounds__(GT) opm_relayout_kernel(const TI* __restrict__ src,
                                                          const float* __restrict__ rec,
                                                          TO* __restrict__ dst, int64_t R) {
  constexpr int K = OPM_K, JT = OPM_JT;
  __shared__ float tile[K][JT * K + 4];  // [p][jj*K + q]
  const int64_t i = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * JT;
  const int64_t Rk = R * K;
  if (FWD) {
    // read num rows i*K + p, columns j0*K .. (j0+JT)*K  (coalesced)
    for (int e = threadIdx.x; e < K * JT * K / 8; e += GT) {
      const int p = e / (JT * K / 8), c8 = e % (JT * K / 8);
      float v[8];
      ld8(src + (i * K + p) * Rk + j0 * K + c8 * 8, v);
#pragma unroll
      for (int u = 0; u < 8; ++u) tile[p][c8 * 8 + u] = v[u];
    }
    __syncthreads();
    // write JT output rows of K*K
    for (int e = threadIdx.x; e < JT * K * K / 8; e += GT) {
      const int jj = e / (K * K / 8), w8 = e % (K * K / 8);
      const int p = (w8 * 8) / K, q0 = (w8 * 8) % K;
      const float r = rec[i * R + j0 + jj];
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = tile[p][jj * K + q0 + u] * r;
      st8(dst + (i * R + j0 + jj) * (K * K) + w8 * 8, v);
    }
  } else {
    // read JT rows of doutn [K*K] (coalesced), scale, write back as num rows
    for (int e = threadIdx.x; e < JT * K * K / 8; e += GT) {
      const int jj = e / (K * K / 8), w8 = e % (K * K / 8);
      const int p = (w8 * 8) / K, q0 = (w8 * 8) % K;
      const float r = rec[i * R + j0 + jj];
      float v[8];
      ld8(src + (i * R + j0 + jj) * (K * K) + w8 * 8, v);
#pragma unroll
      for (int u = 0; u < 8; ++u) tile[p][jj * K + q0 + u] = v[u] * r;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < K * JT * K / 8; e += GT) {
      const int p = e / (JT * K / 8), c8 = e % (JT * K / 8);
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = tile[p][c8 * 8 + u];
      st8(dst + (i * K + p) * Rk + j0 * K + c8 * 8, v);
    }
  }
}

// ---------------------------------------------------------------------------
// column-block packing of the four attention projections:
//   pack:   dst[c, s*N + j] = src_s[c*N + j]          (Wq|Wk|Wv|Wg -> [C, 4N])
//   unpack: dst_s[c*N + j]  = src[c, s*N + j]          ([C, 4N] grad -> 4 slots)
// one launch handles up to PACK_MAX matrices (descriptor table as a parameter)

constexpr int PACK_MAX = 64;
struct PackDesc {
  const void* src[4];
  void* dst[4];
  int64_t C, N;
  int ns;  // matrices per group (2 or 4)
};
struct PackBatch {
  int n, dtype_src, dtype_dst, unpack;
  PackDesc d[PACK_MAX];
};

template <typename TS, typename TD>
__global__ void __launch_bounds__(GT) pack_cols_kernel(const __grid_constant__ PackBatch pb) {
  const PackDesc& d = pb.d[blockIdx.y];
  const int64_t n = d.C * d.ns * d.N;
  for (int64_t e = blockIdx.x * (int64_t)GT + threadIdx.x; e < n; e += (int64_t)gridDim.x * GT) {
    const int64_t c = e / (d.ns * d.N), r = e % (d.ns * d.N);
    const int s = (int)(r / d.N);
    const int64_t j = r % d.N;
    if (!pb.unpack)
      reinterpret_cast<TD*>(d.dst[0])[e] = from_f<TD>(to_f(reinterpret_cast<const TS*>(d.src[s])[c * d.N + j]));
    else
      reinterpret_cast<TD*>(d.dst[s])[c * d.N + j] = from_f<TD>(to_f(reinterpret_cast<const TS*>(d.src[0])[e]));
  }
}

// the same with 8 consecutive columns per thread (16-byte / 32-byte vector
// accesses, 32-bit index math): N % 8 == 0 and 16-byte aligned bases
template <typename TS, typename TD>
__global__ void __launch_bounds__(GT) pack_cols8_kernel(const __grid_constant__ PackBatch pb) {
  const PackDesc& d = pb.d[blockIdx.y];
  const int N8 = (int)(d.N / 8), row8 = d.ns * N8, n8 = (int)d.C * row8;
  for (int e = blockIdx.x * GT + threadIdx.x; e < n8; e += gridDim.x * GT) {
    const int c = e / row8, r = e - c * row8;
    const int s = r / N8, j = (r - s * N8) * 8;
    float v[8];
    if (!pb.unpack) {
      ld8(reinterpret_cast<const TS*>(d.src[s]) + (int64_t)c * d.N + j, v);
      st8(reinterpret_cast<TD*>(d.dst[0]) + (int64_t)e * 8, v);
    } else {
      ld8(reinterpret_cast<const TS*>(d.src[0]) + (int64_t)e * 8, v);
      st8(reinterpret_cast<TD*>(d.dst[s]) + (int64_t)c * d.N + j, v);
    }
  }
}

// rec[i, j] = 1 / (sum_s m[s, i0 + i] m[s, j] + 1e-3)   (block per local row i; exact
// integer sums).  i0 > 0: the rows of one DAP shard (src/model.py:351-378 sharded)
__global__ void __launch_bounds__(GT) opm_rec_vec_kernel_(const float* __restrict__ mask,
                                                         float* __restrict__ rec, int64_t S, int64_t R,
                                                         int64_t i0) {
  extern __shared__ float mi[];  // [S]
  const int64_t i = blockIdx.x;
  for (int64_t s = threadIdx.x; s < S; s += GT) mi[s] = mask[s * R + i0 + i];
  __syncthreads();
  for (int64_t j = threadIdx.x; j < R; j += GT) {
    float acc = 0.f;
    for (int64_t s = 0; s < S; ++s) acc += mi[s] * mask[s * R + j];
    rec[i * R + j] = 1.0f / (acc + 1e-3f);
  }
}

template <int C, typename TX>
void ln_fwd_dispatch_y(const void* x, const float* g, const float* b, void* y, int ydt, float* mean,
                       float* rstd, int64_t rows, float eps, cudaStream_t s) {
  using M = RowMap<C>;
  unsigned grid = glue_grid(rows, M::GROUPS * Unroll<C>::value);
  EVO_DISPATCH_T(ydt, TY, {
    ln_fwd_vec_kernel<C, TX, TY><<<grid, GT, 0, s>>>((const TX*)x, g, b, (TY*)y, mean, rstd, rows, eps);
  });
}

#define POW2_C_DISPATCH(C, CC, ...)                                \
  do {                                                             \
    switch (C) {                                                   \
      case 32: { constexpr int CC = 32; __VA_ARGS__; } break;      \
      case 64: { constexpr int CC = 64; __VA_ARGS__; } break;      \
      case 128: { constexpr int CC = 128; __VA_ARGS__; } break;    \
      case 256: { constexpr int CC = 256; __VA_ARGS__; } break;    \
      case 512: { constexpr int CC = 512; __VA_ARGS__; } break;    \
      case 1024: { constexpr int CC = 1024; __VA_ARGS__; } break;  \
      default: return false;                                       \
    }                                                              \
  } while (0)

inline bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace

void pack_cols(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N, int n,
               int sdt, int ddt, int unpack, cudaStream_t s, int ns) {
  for (int i0 = 0; i0 < n; i0 += PACK_MAX) {
    PackBatch pb{};
    pb.n = n - i0 < PACK_MAX ? n - i0 : PACK_MAX;
    pb.dtype_src = sdt;
    pb.dtype_dst = ddt;
    pb.unpack = unpack;
    int64_t maxe = 0;
    for (int k = 0; k < pb.n; ++k) {
      const int i = i0 + k;
      for (int q = 0; q < ns; ++q) {
        pb.d[k].src[q] = unpack ? src[i] : src[ns * i + q];
        pb.d[k].dst[q] = unpack ? dst[ns * i + q] : dst[i];
      }
      pb.d[k].C = C[i];
      pb.d[k].N = N[i];
      pb.d[k].ns = ns;
      maxe = std::max<int64_t>(maxe, C[i] * ns * N[i]);
    }
    bool v8 = maxe < (1ll << 31);
    for (int k = 0; k < pb.n && v8; ++k) {
      v8 = pb.d[k].N % 8 == 0;
      for (int q = 0; q < ns; ++q) v8 = v8 && al16(pb.d[k].src[unpack ? 0 : q]) && al16(pb.d[k].dst[unpack ? q : 0]);
    }
    if (v8) {
      dim3 grid((unsigned)std::min<int64_t>((maxe / 8 + GT - 1) / GT, 1024), (unsigned)pb.n);
      EVO_DISPATCH_T(sdt, TS, EVO_DISPATCH_T(ddt, TD, { pack_cols8_kernel<TS, TD><<<grid, GT, 0, s>>>(pb); }));
      EVO_LAUNCH_CHECK();
      count_launch(1);
      continue;
    }
    dim3 grid((unsigned)std::min<int64_t>((maxe + GT - 1) / GT, 1024), (unsigned)pb.n);
    EVO_DISPATCH_T(sdt, TS, EVO_DISPATCH_T(ddt, TD, { pack_cols_kernel<TS, TD><<<grid, GT, 0, s>>>(pb); }));
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
}

// ============================================================================
// entry points used by the C ABI wrappers (return false -> scalar fallback)

bool ln_fwd_stream(const void* x, int xdt, const float* g, const float* b, void* y, int ydt, float* mean,
                   float* rstd, int64_t rows, int64_t C, float eps, cudaStream_t s);

bool ln_fwd_vec(const void* x, int xdt, const float* g, const float* b, void* y, int ydt,
                float* mean, float* rstd, int64_t rows, int64_t C, float eps, cudaStream_t s) {
  if (!pow2_width(C) || !al16(x) || !al16(y)) return false;
  if (ln_fwd_stream(x, xdt, g, b, y, ydt, mean, rstd, rows, C, eps, s)) return true;
  POW2_C_DISPATCH(C, CC, EVO_DISPATCH_T(xdt, TX, {
    ln_fwd_dispatch_y<CC, TX>(x, g, b, y, ydt, mean, rstd, rows, eps, s);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool ln_bwd_stream(const void* x, int xdt, const void* dy, int dydt, const float* mean, const float* rstd,
                   const float* g, const float* dres, float* dx, __nv_bfloat16* dx16, float* dgamma,
                   float* dbeta, float* dxsum, int accumulate, void* ws, int64_t rows, int64_t C,
                   int64_t ws_blocks, cudaStream_t s);

int64_t ln_bwd_vec_ws(int64_t C) { return (int64_t)num_sms() * PARTIAL_PER_SM * 3 * C * 4; }

bool ln_bwd_vec(const void* x, int xdt, const void* dy, int dydt, const float* mean, const float* rstd,
                const float* g, const float* dres, float* dx, __nv_bfloat16* dx16, float* dgamma,
                float* dbeta, float* dxsum, int accumulate, void* ws, int64_t rows, int64_t C,
                cudaStream_t s) {
  if (!pow2_width(C) || !al16(x) || !al16(dy) || !al16(dx) || (dres && !al16(dres)) ||
      (dx16 && !al16(dx16)))
    return false;
  ws = partial_buffer(ws, ln_bwd_vec_ws(C));
  if (ln_bwd_stream(x, xdt, dy, dydt, mean, rstd, g, dres, dx, dx16, dgamma, dbeta, dxsum, accumulate, ws,
                    rows, C, (int64_t)num_sms() * PARTIAL_PER_SM, s))
    return true;
  unsigned grid = 0;
  POW2_C_DISPATCH(C, CC, {
    using M = RowMap<CC>;
    grid = glue_grid(rows, M::GROUPS * 2, PARTIAL_PER_SM);
    const size_t smem = (size_t)M::GROUPS * 3 * CC * sizeof(float);
    EVO_DISPATCH_T(xdt, TX, EVO_DISPATCH_T(dydt, TD, {
      auto k = ln_bwd_vec_kernel<CC, TX, TD>;
      if (smem > 48 * 1024)
        EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k<<<grid, GT, smem, s>>>((const TX*)x, (const TD*)dy, mean, rstd, g, dres, dx, dx16,
                               (float*)ws, rows, dxsum != nullptr);
    }));
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials((const float*)ws, grid, C, dgamma, accumulate, s, 3 * C);
  finalize_partials((const float*)ws + C, grid, C, dbeta, accumulate, s, 3 * C);
  if (dxsum) finalize_partials((const float*)ws + 2 * C, grid, C, dxsum, 0, s, 3 * C);
  return true;
}

int64_t colsum_vec_ws(int64_t C) { return (int64_t)num_sms() * PARTIAL_PER_SM * C * 4; }

// mode 0: plain colsum (+ optional cast copy y); mode 1: relu-backward in place
bool colsum_vec(void* x, int xdt, int64_t ldx, const void* h, void* y, int ydt, float* out,
                int accumulate, void* ws, int64_t rows, int64_t C, int mode, cudaStream_t s) {
  if (!pow2_width(C) || C > 2048 || !al16(x) || (ldx % 8) != 0 || (y && !al16(y)) || (h && !al16(h)))
    return false;
  const int TPR = (int)(C / 8);
  if (TPR > GT) return false;
  ws = partial_buffer(ws, colsum_vec_ws(C));
  const int RPB = GT / TPR;
  unsigned grid = glue_grid(rows, RPB * 2, PARTIAL_PER_SM);
  const size_t smem = (size_t)RPB * C * sizeof(float);
  EVO_DISPATCH_T(xdt, TX, EVO_DISPATCH_T(ydt, TY, {
    if (mode == 1)
      colsum_vec_kernel<TX, TY, 1><<<grid, GT, smem, s>>>((TX*)x, ldx, (const TX*)h, (TY*)y, (float*)ws, rows, (int)C);
    else
      colsum_vec_kernel<TX, TY, 0><<<grid, GT, smem, s>>>((TX*)x, ldx, nullptr, (TY*)y, (float*)ws, rows, (int)C);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials((const float*)ws, grid, C, out, accumulate, s);
  return true;
}

bool bias_residual_vec(const void* res, int rdt, const void* y, int ydt, const float* bias, void* out,
                       int odt, int64_t rows, int64_t C, cudaStream_t s) {
  if ((C % 8) != 0 || !al16(y) || !al16(out) || (res && !al16(res)) || (bias && !al16(bias))) return false;
  const int64_t n8 = rows * C / 8;
  unsigned grid = glue_grid(n8, GT * EW_UNROLL);
  EVO_DISPATCH_T(rdt, TR, EVO_DISPATCH_T(ydt, TY, EVO_DISPATCH_T(odt, TO, {
    bias_residual_vec_kernel<TR, TY, TO><<<grid, GT, 0, s>>>((const TR*)res, (const TY*)y, bias,
                                                             (TO*)out, n8, (int)(C / 8));
  })));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool bias_relu_vec(void* y, int dt, const float* bias, int64_t rows, int64_t C, cudaStream_t s) {
  if ((C % 8) != 0 || !al16(y) || (bias && !al16(bias))) return false;
  const int64_t n8 = rows * C / 8;
  unsigned grid = glue_grid(n8, GT * EW_UNROLL);
  EVO_DISPATCH_T(dt, T, {
    bias_relu_vec_kernel<T><<<grid, GT, 0, s>>>((T*)y, bias, n8, (int)(C / 8));
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool pair_bias_fwd_vec(const void* z, int dt, const float* g, const float* b, const float* w, void* nb,
                       float* mean, float* rstd, int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap,
                       cudaStream_t s) {
  if (!pow2_width(C) || C > 256 || H > 8 || !al16(z)) return false;
  POW2_C_DISPATCH(C, CC, {
    if constexpr (CC <= 256) {
      using M = PbMap<CC>;
      // resident blocks only: each block loads its slice of w once and loops
      unsigned grid = glue_grid(NI * NJ, M::GROUPS * M::U, 3);
      EVO_DISPATCH_T(dt, T, {
        pair_bias_fwd_vec_kernel<CC, T><<<grid, GT, 0, s>>>((const T*)z, g, b, w, (T*)nb, mean, rstd,
                                                            NI, NJ, (int)H, swap);
      });
    } else {
      return false;
    }
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool pair_bias_bwd_stream(const void* z, int dt, const float* mean, const float* rstd, const float* g,
                          const float* bln, const float* w, const float* dnb, int swap, float* dz, float* dg,
                          float* db, float* dw, int accumulate, void* ws, int64_t NI, int64_t NJ, int64_t C,
                          int64_t H, int64_t ws_blocks, cudaStream_t s, __nv_bfloat16* dz16, float* dzsum);

int64_t pair_bias_bwd_vec_ws(int64_t C, int64_t H) {
  return (int64_t)num_sms() * PB_PARTIAL_PER_SM * (C * H + 3 * C) * 4;
}

bool pair_bias_bwd_vec(const void* z, int dt, const float* mean, const float* rstd, const float* g,
                       const float* bln, const float* w, const float* dnb, int swap, float* dz,
                       float* dg, float* db, float* dw, int accumulate, void* ws, int64_t NI,
                       int64_t NJ, int64_t C, int64_t H, cudaStream_t s, __nv_bfloat16* dz16, float* dzsum,
                       bool* fused_out) {
  if (fused_out) *fused_out = false;
  if (!pow2_width(C) || C > 256 || H > 8 || !al16(z) || !al16(dz)) return false;
  ws = partial_buffer(ws, pair_bias_bwd_vec_ws(C, H));
  if (pair_bias_bwd_stream(z, dt, mean, rstd, g, bln, w, dnb, swap, dz, dg, db, dw, accumulate, ws, NI, NJ, C, H,
                           (int64_t)num_sms() * PB_PARTIAL_PER_SM, s, dz16, dzsum)) {
    if (fused_out) *fused_out = true;
    return true;
  }
  unsigned grid = 0;
  POW2_C_DISPATCH(C, CC, {
    if constexpr (CC <= 256) {
      using M = PbMap<CC>;
      grid = glue_grid(NI * NJ, M::GROUPS * M::U, PB_PARTIAL_PER_SM);
      const int W = (int)(CC * H + 2 * CC);
      const size_t smem = (size_t)M::GROUPS * W * sizeof(float);
      EVO_DISPATCH_T(dt, T, {
        auto k = pair_bias_bwd_vec_kernel<CC, T>;
        if (smem > 48 * 1024)
          EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, GT, smem, s>>>((const T*)z, mean, rstd, g, bln, w, dnb, swap, dz, (float*)ws, NI, NJ, (int)H);
      });
    } else {
      return false;
    }
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  const int64_t W = C * H + 2 * C;
  finalize_partials((const float*)ws, grid, C * H, dw, accumulate, s, W);
  finalize_partials((const float*)ws + C * H, grid, C, dg, accumulate, s, W);
  finalize_partials((const float*)ws + C * H + C, grid, C, db, accumulate, s, W);
  return true;
}

void opm_rec_rows(const float* mask, float* rec, int64_t S, int64_t R, int64_t i0, int64_t NI, cudaStream_t s) {
  if (NI * R == 0) return;
  opm_rec_vec_kernel_<<<(unsigned)NI, GT, S * sizeof(float), s>>>(mask, rec, S, R, i0);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

bool opm_norm_vec(bool fwd, const void* src, int sdt, const float* mask, float* rec, void* dst, int ddt,
                  int64_t S, int64_t R, int64_t k, int64_t i0, int64_t NI, cudaStream_t s) {
  if (k != OPM_K || (R % OPM_JT) != 0 || !al16(src) || !al16(dst)) return false;
  if (fwd && mask) {  // mask == nullptr: rec is given
    opm_rec_vec_kernel_<<<(unsigned)NI, GT, S * sizeof(float), s>>>(mask, rec, S, R, i0);
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
  dim3 grid((unsigned)(R / OPM_JT), (unsigned)NI);
  if (NI == 0) return true;
  EVO_DISPATCH_T(sdt, TI, EVO_DISPATCH_T(ddt, TO, {
    if (fwd)
      opm_relayout_kernel<TI, TO, true><<<grid, GT, 0, s>>>((const TI*)src, rec, (TO*)dst, R);
    else
      opm_relayout_kernel<TI, TO, false><<<grid, GT, 0, s>>>((const TI*)src, rec, (TO*)dst, R);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

}  // namespace evo
