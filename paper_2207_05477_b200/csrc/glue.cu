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
inline unsigned glue_grid(int64_t rows, int rows_per_iter, int per_sm = 16) {
  int64_t want = (rows + rows_per_iter - 1) / rows_per_iter;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (want > cap) want = cap;
  return (unsigned)(want > 0 ? want : 1);
}

template <int C>
struct RowMap {
  static constexpr int LANES = (C / 8) < 32 ? (C / 8) : 32;  // lanes per row
  static constexpr int CH = C / (8 * LANES);                  // 8-chunks per lane
  static constexpr int RPW = 32 / LANES;                      // rows per warp
  static constexpr int GROUPS = GT / LANES;                   // rows per block iteration
};

// ---------------------------------------------------------------------------
// LayerNorm forward

template <int C, typename TX, typename TY>
__global__ void __launch_bounds__(GT) ln_fwd_vec_kernel(const TX* __restrict__ x,
                                                        const float* __restrict__ g,
                                                        const float* __restrict__ b,
                                                        TY* __restrict__ y, float* __restrict__ mean,
                                                        float* __restrict__ rstd, int64_t rows, float eps) {
  using M = RowMap<C>;
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  // block-uniform trip count: the row groups of a warp always shuffle together
  for (int64_t rb = blockIdx.x * (int64_t)M::GROUPS; rb < rows; rb += (int64_t)gridDim.x * M::GROUPS) {
    const bool act = rb + grp < rows;
    const int64_t r = act ? rb + grp : rows - 1;
    float v[M::CH][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < M::CH; ++k) {
      ld8(x + r * C + (k * M::LANES + l) * 8, v[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += v[k][e];
    }
    const float mu = group_sum<M::LANES>(s) / (float)C;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < M::CH; ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = v[k][e] - mu;
        q += d * d;
      }
    const float inv = 1.0f / sqrtf(group_sum<M::LANES>(q) / (float)C + eps);
#pragma unroll
    for (int k = 0; k < M::CH; ++k) {
      const int c0 = (k * M::LANES + l) * 8;
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (v[k][e] - mu) * inv * g[c0 + e] + b[c0 + e];
      if (act) st8(y + r * C + c0, o);
    }
    if (act && l == 0) {
      if (mean) mean[r] = mu;
      if (rstd) rstd[r] = inv;
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
  for (int64_t rb = r0; rb < r1; rb += M::GROUPS) {
    const bool act = rb + grp < r1;
    const int64_t r = act ? rb + grp : r1 - 1;
    const float mu = mean[r], inv = rstd[r];
    const float w = act ? 1.f : 0.f;
    float xh[M::CH][8], dxh[M::CH][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < M::CH; ++k) {
      const int c0 = (k * M::LANES + l) * 8;
      float xv[8], d[8];
      ld8(x + r * C + c0, xv);
      ld8(dy + r * C + c0, d);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        d[e] *= w;
        xh[k][e] = (xv[e] - mu) * inv;
        dxh[k][e] = d[e] * gg[k][e];
        dg[k][e] += d[e] * xh[k][e];
        db[k][e] += d[e];
        s1 += dxh[k][e];
        s2 += dxh[k][e] * xh[k][e];
      }
    }
    const float m1 = group_sum<M::LANES>(s1) / (float)C;
    const float m2 = group_sum<M::LANES>(s2) / (float)C;
#pragma unroll
    for (int k = 0; k < M::CH; ++k) {
      const int c0 = (k * M::LANES + l) * 8;
      float o[8];
      if (dres) {
        ld8(dres + r * C + c0, o);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        o[e] += inv * (dxh[k][e] - m1 - xh[k][e] * m2);
        dsx[k][e] += w * o[e];
      }
      if (act) {
        st8(dx + r * C + c0, o);
        if (dx16) st8(dx16 + r * C + c0, o);
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
#pragma unroll 2
  for (int64_t r = r0 + rg; r < r1; r += RPB) {
    float v[8];
    ld8(x + r * ldx + ct * 8, v);
    if (MODE == 1) {
      float hv[8];
      ld8(h + r * C + ct * 8, hv);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = hv[e] > 0.f ? v[e] : 0.f;
      st8(x + r * ldx + ct * 8, v);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += v[e];
    if (y) st8(y + r * C + ct * 8, v);
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
  for (int64_t e = blockIdx.x * (int64_t)GT + threadIdx.x; e < n8; e += (int64_t)gridDim.x * GT) {
    const int c0 = (int)(e % C8) * 8;
    float v[8];
    ld8(y + e * 8, v);
    if (bias) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] += bias[c0 + k];
    }
    if (res) {
      float r[8];
      ld8(res + e * 8, r);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = r[k] + v[k];
    }
    st8(out + e * 8, v);
  }
}

template <typename T>
__global__ void __launch_bounds__(GT) bias_relu_vec_kernel(T* __restrict__ y, const float* __restrict__ bias,
                                                           int64_t n8, int C8) {
  for (int64_t e = blockIdx.x * (int64_t)GT + threadIdx.x; e < n8; e += (int64_t)gridDim.x * GT) {
    const int c0 = (int)(e % C8) * 8;
    float v[8];
    ld8(y + e * 8, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fmaxf(v[k] + (bias ? bias[c0 + k] : 0.f), 0.f);
    st8(y + e * 8, v);
  }
}

// ---------------------------------------------------------------------------
// pair bias: nb[h, x, y] (or [h, y, x]) = LN(z[x, y]) . w[:, h]

template <int C, typename T>
__global__ void __launch_bounds__(GT) pair_bias_fwd_vec_kernel(
    const T* __restrict__ z, const float* __restrict__ g, const float* __restrict__ b,
    const float* __restrict__ w, T* __restrict__ nb, float* __restrict__ mean,
    float* __restrict__ rstd, int64_t R, int H, int swap_xy) {
  using M = RowMap<C>;
  static_assert(M::CH == 1, "pair bias expects C <= 256");
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  const int c0 = l * 8;
  float gg[8], bb[8], wr[8][8];  // this lane's 8 channels x (up to 8) heads, in registers
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    gg[e] = g[c0 + e];
    bb[e] = b[c0 + e];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) wr[e][hh] = hh < H ? w[(c0 + e) * H + hh] : 0.f;
  }
  const int64_t NT = R * R;
  for (int64_t tb = blockIdx.x * (int64_t)M::GROUPS; tb < NT; tb += (int64_t)gridDim.x * M::GROUPS) {
    const bool act = tb + grp < NT;
    const int64_t t = act ? tb + grp : NT - 1;
    float v[8];
    ld8(z + t * C + c0, v);
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) s += v[e];
    const float mu = group_sum<M::LANES>(s) / (float)C;
    float q = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = v[e] - mu;
      q += d * d;
    }
    const float inv = 1.0f / sqrtf(group_sum<M::LANES>(q) / (float)C + 1e-5f);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (v[e] - mu) * inv * gg[e] + bb[e];
    const int64_t x = t / R, y = t % R;
    float mine = 0.f;
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
      if (hh < H) {
        float p = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) p = fmaf(v[e], wr[e][hh], p);
        p = group_sum<M::LANES>(p);
        if (l == hh) mine = p;
      }
    }
    if (act && l < H) {
      const int64_t o = swap_xy ? ((int64_t)l * R + y) * R + x : ((int64_t)l * R + x) * R + y;
      nb[o] = from_f<T>(mine);
    }
    if (act && l == 0) {
      mean[t] = mu;
      rstd[t] = inv;
    }
  }
}

// partial layout per block: [dw (C*H) | dgamma (C) | dbeta (C)]
template <int C, int HM, typename T>
__global__ void __launch_bounds__(GT) pair_bias_bwd_vec_kernel(
    const T* __restrict__ z, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ g, const float* __restrict__ bln, const float* __restrict__ w,
    const float* __restrict__ dnb, int swap_xy, float* __restrict__ dz,
    float* __restrict__ partials, int64_t R, int H) {
  using M = RowMap<C>;
  static_assert(M::CH == 1, "pair bias expects C <= 256");
  extern __shared__ float sm[];  // (unused [C*HM]) then reduction scratch [GROUPS][C*H + 2C]
  float* red = sm + C * HM;
  const int l = threadIdx.x % M::LANES;
  const int grp = threadIdx.x / M::LANES;
  const int c0 = l * 8;
  float gg[8], bb[8], wr[8][HM];  // this lane's channels x heads, in registers
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    gg[e] = g[c0 + e];
    bb[e] = bln[c0 + e];
#pragma unroll
    for (int hh = 0; hh < HM; ++hh) wr[e][hh] = hh < H ? w[(c0 + e) * H + hh] : 0.f;
  }
  float dw[8][HM], dgs[8], dbs[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    dgs[e] = dbs[e] = 0.f;
#pragma unroll
    for (int hh = 0; hh < HM; ++hh) dw[e][hh] = 0.f;
  }
  const int64_t NT = R * R;
  const int64_t t0 = (NT * blockIdx.x) / gridDim.x, t1 = (NT * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tb = t0; tb < t1; tb += M::GROUPS) {
    const bool act = tb + grp < t1;
    const int64_t t = act ? tb + grp : t1 - 1;
    const int64_t x = t / R, y = t % R;
    float dp_mine = 0.f;
    if (act && l < H) {  // inactive groups carry dP = 0: no contribution anywhere
      const int64_t o = swap_xy ? ((int64_t)l * R + y) * R + x : ((int64_t)l * R + x) * R + y;
      dp_mine = dnb[o];
    }
    float dP[HM];
    const int base = (threadIdx.x & 31) - l;  // first lane of this row group
#pragma unroll
    for (int hh = 0; hh < HM; ++hh) dP[hh] = __shfl_sync(0xffffffffu, dp_mine, base + (hh < M::LANES ? hh : 0));
    const float mu = mean[t], inv = rstd[t];
    float v[8];
    ld8(z + t * C + c0, v);
    float xh[8], dxh[8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      xh[e] = (v[e] - mu) * inv;
      const float zl = xh[e] * gg[e] + bb[e];
      float dzl = 0.f;
#pragma unroll
      for (int hh = 0; hh < HM; ++hh) {
        if (hh < H) {
          dzl = fmaf(dP[hh], wr[e][hh], dzl);
          dw[e][hh] = fmaf(zl, dP[hh], dw[e][hh]);
        }
      }
      dgs[e] += dzl * xh[e];
      dbs[e] += dzl;
      dxh[e] = dzl * gg[e];
      s1 += dxh[e];
      s2 += dxh[e] * xh[e];
    }
    const float m1 = group_sum<M::LANES>(s1) / (float)C, m2 = group_sum<M::LANES>(s2) / (float)C;
    if (act) {
      float o[8];
      ld8(dz + t * C + c0, o);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += inv * (dxh[e] - m1 - xh[e] * m2);
      st8(dz + t * C + c0, o);
    }
  }
  const int W = C * H + 2 * C;
  float* mine = red + grp * W;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
#pragma unroll
    for (int hh = 0; hh < HM; ++hh)
      if (hh < H) mine[(c0 + e) * H + hh] = dw[e][hh];
    mine[C * H + c0 + e] = dgs[e];
    mine[C * H + C + c0 + e] = dbs[e];
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
};
struct PackBatch {
  int n, dtype_src, dtype_dst, unpack;
  PackDesc d[PACK_MAX];
};

template <typename TS, typename TD>
__global__ void __launch_bounds__(GT) pack_cols_kernel(const __grid_constant__ PackBatch pb) {
  const PackDesc& d = pb.d[blockIdx.y];
  const int64_t n = d.C * 4 * d.N;
  for (int64_t e = blockIdx.x * (int64_t)GT + threadIdx.x; e < n; e += (int64_t)gridDim.x * GT) {
    const int64_t c = e / (4 * d.N), r = e % (4 * d.N);
    const int s = (int)(r / d.N);
    const int64_t j = r % d.N;
    if (!pb.unpack)
      reinterpret_cast<TD*>(d.dst[0])[e] = from_f<TD>(to_f(reinterpret_cast<const TS*>(d.src[s])[c * d.N + j]));
    else
      reinterpret_cast<TD*>(d.dst[s])[c * d.N + j] = from_f<TD>(to_f(reinterpret_cast<const TS*>(d.src[0])[e]));
  }
}

// rec[i, j] = 1 / (sum_s m[s, i] m[s, j] + 1e-3)   (block per i; exact integer sums)
__global__ void __launch_bounds__(GT) opm_rec_vec_kernel(const float* __restrict__ mask,
                                                         float* __restrict__ rec, int64_t S, int64_t R) {
  extern __shared__ float mi[];  // [S]
  const int64_t i = blockIdx.x;
  for (int64_t s = threadIdx.x; s < S; s += GT) mi[s] = mask[s * R + i];
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
  unsigned grid = glue_grid(rows, M::GROUPS);
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
               int sdt, int ddt, int unpack, cudaStream_t s) {
  for (int i0 = 0; i0 < n; i0 += PACK_MAX) {
    PackBatch pb{};
    pb.n = n - i0 < PACK_MAX ? n - i0 : PACK_MAX;
    pb.dtype_src = sdt;
    pb.dtype_dst = ddt;
    pb.unpack = unpack;
    int64_t maxe = 0;
    for (int k = 0; k < pb.n; ++k) {
      const int i = i0 + k;
      for (int q = 0; q < 4; ++q) {
        pb.d[k].src[q] = unpack ? src[i] : src[4 * i + q];
        pb.d[k].dst[q] = unpack ? dst[4 * i + q] : dst[i];
      }
      pb.d[k].C = C[i];
      pb.d[k].N = N[i];
      maxe = std::max<int64_t>(maxe, C[i] * 4 * N[i]);
    }
    dim3 grid((unsigned)std::min<int64_t>((maxe + GT - 1) / GT, 1024), (unsigned)pb.n);
    EVO_DISPATCH_T(sdt, TS, EVO_DISPATCH_T(ddt, TD, { pack_cols_kernel<TS, TD><<<grid, GT, 0, s>>>(pb); }));
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
}

// ============================================================================
// entry points used by the C ABI wrappers (return false -> scalar fallback)

bool ln_fwd_vec(const void* x, int xdt, const float* g, const float* b, void* y, int ydt,
                float* mean, float* rstd, int64_t rows, int64_t C, float eps, cudaStream_t s) {
  if (!pow2_width(C) || !al16(x) || !al16(y)) return false;
  POW2_C_DISPATCH(C, CC, EVO_DISPATCH_T(xdt, TX, {
    ln_fwd_dispatch_y<CC, TX>(x, g, b, y, ydt, mean, rstd, rows, eps, s);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

int64_t ln_bwd_vec_ws(int64_t C) { return (int64_t)num_sms() * PARTIAL_PER_SM * 3 * C * 4; }

bool ln_bwd_vec(const void* x, int xdt, const void* dy, int dydt, const float* mean, const float* rstd,
                const float* g, const float* dres, float* dx, __nv_bfloat16* dx16, float* dgamma,
                float* dbeta, float* dxsum, int accumulate, void* ws, int64_t rows, int64_t C,
                cudaStream_t s) {
  if (!pow2_width(C) || !al16(x) || !al16(dy) || !al16(dx) || (dres && !al16(dres)) ||
      (dx16 && !al16(dx16)))
    return false;
  ws = partial_buffer(ws, ln_bwd_vec_ws(C));
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
  if ((C % 8) != 0 || !al16(y) || !al16(out) || (res && !al16(res))) return false;
  const int64_t n8 = rows * C / 8;
  unsigned grid = glue_grid(n8, GT * 2);
  EVO_DISPATCH_T(rdt, TR, EVO_DISPATCH_T(ydt, TY, EVO_DISPATCH_T(odt, TO, {
    bias_residual_vec_kernel<TR, TY, TO><<<grid, GT, 0, s>>>((const TR*)res, (const TY*)y, bias,
                                                             (TO*)out, n8, (int)(C / 8));
  })));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool bias_relu_vec(void* y, int dt, const float* bias, int64_t rows, int64_t C, cudaStream_t s) {
  if ((C % 8) != 0 || !al16(y)) return false;
  const int64_t n8 = rows * C / 8;
  unsigned grid = glue_grid(n8, GT * 2);
  EVO_DISPATCH_T(dt, T, {
    bias_relu_vec_kernel<T><<<grid, GT, 0, s>>>((T*)y, bias, n8, (int)(C / 8));
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

bool pair_bias_fwd_vec(const void* z, int dt, const float* g, const float* b, const float* w, void* nb,
                       float* mean, float* rstd, int64_t R, int64_t C, int64_t H, int swap,
                       cudaStream_t s) {
  if (!pow2_width(C) || C > 256 || H > 8 || H > C / 8 || !al16(z)) return false;
  POW2_C_DISPATCH(C, CC, {
    if constexpr (CC <= 256) {
      using M = RowMap<CC>;
      unsigned grid = glue_grid(R * R, M::GROUPS * 4, 2);  // weights live in registers: few blocks
      EVO_DISPATCH_T(dt, T, {
        pair_bias_fwd_vec_kernel<CC, T><<<grid, GT, 0, s>>>((const T*)z, g, b, w, (T*)nb, mean, rstd,
                                                            R, (int)H, swap);
      });
    } else {
      return false;
    }
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  return true;
}

int64_t pair_bias_bwd_vec_ws(int64_t C, int64_t H) {
  return (int64_t)num_sms() * PARTIAL_PER_SM * (C * H + 2 * C) * 4;
}

bool pair_bias_bwd_vec(const void* z, int dt, const float* mean, const float* rstd, const float* g,
                       const float* bln, const float* w, const float* dnb, int swap, float* dz,
                       float* dg, float* db, float* dw, int accumulate, void* ws, int64_t R,
                       int64_t C, int64_t H, cudaStream_t s) {
  if (!pow2_width(C) || C > 256 || H > 8 || H > C / 8 || !al16(z) || !al16(dz)) return false;
  ws = partial_buffer(ws, pair_bias_bwd_vec_ws(C, H));
  unsigned grid = 0;
  POW2_C_DISPATCH(C, CC, {
    if constexpr (CC <= 256) {
      using M = RowMap<CC>;
      grid = glue_grid(R * R, M::GROUPS * 2, PARTIAL_PER_SM);
      const int W = (int)(CC * H + 2 * CC);
      const size_t smem = ((size_t)CC * 8 + (size_t)M::GROUPS * W) * sizeof(float);
      EVO_DISPATCH_T(dt, T, {
        auto k = pair_bias_bwd_vec_kernel<CC, 8, T>;
        if (smem > 48 * 1024)
          EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, GT, smem, s>>>((const T*)z, mean, rstd, g, bln, w, dnb, swap, dz, (float*)ws, R, (int)H);
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

bool opm_norm_vec(bool fwd, const void* src, int sdt, const float* mask, float* rec, void* dst, int ddt,
                  int64_t S, int64_t R, int64_t k, cudaStream_t s) {
  if (k != OPM_K || (R % OPM_JT) != 0 || !al16(src) || !al16(dst)) return false;
  if (fwd) {
    opm_rec_vec_kernel<<<(unsigned)R, GT, S * sizeof(float), s>>>(mask, rec, S, R);
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
  dim3 grid((unsigned)(R / OPM_JT), (unsigned)R);
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
