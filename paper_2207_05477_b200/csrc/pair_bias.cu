// Pair-bias projection for MSA-row and triangle attention (src/model.py:312-317):
//   nb[h, i, j] = LN(z)[i, j, :] . w_bias[:, h]
// One warp per pair token: LayerNorm in registers, the H-wide projection as
// warp reductions, written straight into the transposed bias layout the
// attention kernels read (nb[h, query, key], storage dtype).  Bandwidth-bound: reads
// the pair once (R*R*C storage bytes), writes H*R*R fp32.
//
// Backward fuses dP -> dLN -> LayerNorm backward -> dz (+=) with the
// w_bias / LN-affine gradient partials in one pass over the pair.
#include "common.cuh"
#include "vec.cuh"
#include "tc_common.cuh"
#include <type_traits>
#include "reduce.cuh"

namespace evo {

constexpr int PB_WARPS = 8;
constexpr int PB_HMAX = 16;

template <typename T, int NPL>
__global__ void __launch_bounds__(PB_WARPS * 32) pair_bias_fwd_kernel(
    const T* __restrict__ z, const float* __restrict__ g, const float* __restrict__ b,
    const float* __restrict__ w, T* __restrict__ nb, float* __restrict__ mean,
    float* __restrict__ rstd, int64_t NI, int64_t NJ, int C, int H, int swap_xy) {
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)PB_WARPS + (threadIdx.x >> 5);
  if (t >= NI * NJ) return;
  float v[NPL];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    v[k] = c < C ? to_f(z[t * C + c]) : 0.f;
    s += v[k];
  }
  const float mu = warp_sum(s) / (float)C;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    float d = c < C ? v[k] - mu : 0.f;
    q += d * d;
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / (float)C + 1e-5f);
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    v[k] = c < C ? (v[k] - mu) * inv * g[c] + b[c] : 0.f;
  }
  const int64_t x = t / NJ, y = t % NJ;
  float mine = 0.f;
#pragma unroll
  for (int h = 0; h < PB_HMAX; ++h) {
    if (h < H) {
      float p = 0.f;
#pragma unroll
      for (int k = 0; k < NPL; ++k) {
        int c = lane + 32 * k;
        if (c < C) p = fmaf(v[k], w[c * H + h], p);
      }
      p = warp_sum(p);
      if (lane == h) mine = p;
    }
  }
  if (lane < H) {
    int64_t o = swap_xy ? ((int64_t)lane * NJ + y) * NI + x : ((int64_t)lane * NI + x) * NJ + y;
    nb[o] = from_f<T>(mine);
  }
  if (lane == 0) {
    mean[t] = mu;
    rstd[t] = inv;
  }
}

template <typename T, int NPL>
__global__ void __launch_bounds__(PB_WARPS * 32) pair_bias_bwd_kernel(
    const T* __restrict__ z, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ g, const float* __restrict__ bln, const float* __restrict__ w,
    const float* __restrict__ dnb, int swap_xy, float* __restrict__ dz,
    float* __restrict__ partials, int64_t NI, int64_t NJ, int C, int H) {
  extern __shared__ float sm[];  // [PB_WARPS][C*H + 2C]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = C * H + 2 * C;
  float dw[NPL][PB_HMAX], dg[NPL], db[NPL];
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    dg[k] = db[k] = 0.f;
#pragma unroll
    for (int h = 0; h < PB_HMAX; ++h) dw[k][h] = 0.f;
  }
  for (int64_t t = blockIdx.x * (int64_t)PB_WARPS + warp; t < NI * NJ;
       t += (int64_t)gridDim.x * PB_WARPS) {
    const int64_t x = t / NJ, y = t % NJ;
    float dp = 0.f;
    if (lane < H) {
      int64_t o = swap_xy ? ((int64_t)lane * NJ + y) * NI + x : ((int64_t)lane * NI + x) * NJ + y;
      dp = dnb[o];
    }
    float dP[PB_HMAX];
#pragma unroll
    for (int h = 0; h < PB_HMAX; ++h) dP[h] = __shfl_sync(0xffffffffu, dp, h);
    const float mu = mean[t], inv = rstd[t];
    float xh[NPL], dxh[NPL];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      int c = lane + 32 * k;
      if (c < C) {
        xh[k] = (to_f(z[t * C + c]) - mu) * inv;
        const float zl = xh[k] * g[c] + bln[c];
        float dzl = 0.f;
#pragma unroll
        for (int h = 0; h < PB_HMAX; ++h) {
          if (h < H) {
            dzl = fmaf(dP[h], w[c * H + h], dzl);
            dw[k][h] = fmaf(zl, dP[h], dw[k][h]);
          }
        }
        dg[k] += dzl * xh[k];
        db[k] += dzl;
        dxh[k] = dzl * g[c];
      } else {
        xh[k] = dxh[k] = 0.f;
      }
      s1 += dxh[k];
      s2 += dxh[k] * xh[k];
    }
    const float m1 = warp_sum(s1) / (float)C, m2 = warp_sum(s2) / (float)C;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      int c = lane + 32 * k;
      if (c < C) dz[t * C + c] += inv * (dxh[k] - m1 - xh[k] * m2);
    }
  }
  float* mine = sm + warp * W;
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    if (c < C) {
#pragma unroll
      for (int h = 0; h < PB_HMAX; ++h)
        if (h < H) mine[c * H + h] = dw[k][h];
      mine[C * H + c] = dg[k];
      mine[C * H + C + c] = db[k];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    float acc = 0.f;
    for (int ww = 0; ww < PB_WARPS; ++ww) acc += sm[ww * W + c];
    partials[(int64_t)blockIdx.x * W + c] = acc;
  }
}

#define PB_NPL_DISPATCH(C, NPL, ...)                                          \
  do {                                                                        \
    if ((C) <= 32) { constexpr int NPL = 1; __VA_ARGS__; }                    \
    else if ((C) <= 64) { constexpr int NPL = 2; __VA_ARGS__; }               \
    else if ((C) <= 128) { constexpr int NPL = 4; __VA_ARGS__; }              \
    else if ((C) <= 256) { constexpr int NPL = 8; __VA_ARGS__; }              \
    else throw Error(EVO_ERR_UNSUPPORTED, "pair_bias: C > 256");              \
  } while (0)

bool pair_bias_fwd_vec(const void* z, int dt, const float* g, const float* b, const float* w, void* nb,
                       float* mean, float* rstd, int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap,
                       cudaStream_t s);

// Thread-per-token forward: each thread owns one token row (no cross-lane
// reductions at all), reads it three times from L1 (sum, squared deviation,
// projection), and keeps the 8 head accumulators in registers; LN affine and
// w_bias are broadcast from shared memory.  Threads walk the tokens in output
// order -- for the transposed triangle-end layout (swap) thread i handles token
// (i % NI, i / NI) -- so the 8 head planes of nb are written coalesced.
__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int C, typename T>
struct PbTile {
  static constexpr int ROWB = C * (int)sizeof(T) + 16;  // padded row: 16-B chunk index 17t+k spreads banks
  static constexpr int CPR = C * (int)sizeof(T) / 16;   // 16-B chunks per row
  static constexpr int bytes = 128 * ROWB;
};

// A block owns 128 consecutive output positions: their token rows are staged
// into shared memory with coalesced 16-B cp.async (CPR threads per row), then
// each thread reduces and projects one row from the padded tile.
template <int C, typename T>
__global__ void __launch_bounds__(128) pair_bias_fwd_tpt_kernel(
    const T* __restrict__ z, const float* __restrict__ g, const float* __restrict__ b,
    const float* __restrict__ w, T* __restrict__ nb, float* __restrict__ mean,
    float* __restrict__ rstd, int64_t NI, int64_t NJ, int H, int swap) {
  using TL = PbTile<C, T>;
  extern __shared__ __align__(16) uint8_t tile[];
  __shared__ float4 sw[C][2];   // w[c, 0..7] (zero beyond H)
  const int64_t RR = NI * NJ;
  const int64_t i0 = blockIdx.x * (int64_t)128;
  // stage: chunk k of row r by thread (r * CPR + k) % 128
  for (int e = threadIdx.x; e < 128 * TL::CPR; e += 128) {
    const int r = e / TL::CPR, k = e % TL::CPR;
    const int64_t i = i0 + r;
    if (i < RR) {
      const int64_t tok = swap ? (i % NI) * NJ + i / NI : i;
      tc::cp_async16(tile + r * TL::ROWB + k * 16, reinterpret_cast<const uint8_t*>(z + tok * C) + k * 16);
    }
  }
  tc::cp_async_commit();
  // LayerNorm folded into the projection: with gw = g (x) w and the per-head
  // constants G = sum_c gw[c, :], BW = sum_c b[c] w[c, :],
  //   nb[h] = rstd * (sum_c z_c gw[c, h] - mean * G[h]) + BW[h],
  // so one pass over the row gives the statistics and the head sums together
  __shared__ float sG[8], sBW[8], spart[4][16];
  static_assert(C <= 128 * 4, "one block of 128 threads covers the channels");
  {
    float gsum[8], bsum[8];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) gsum[hh] = bsum[hh] = 0.f;
    for (int e = threadIdx.x; e < C; e += blockDim.x) {
      float t[8];
      const float ge = g[e], be = b[e];
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        const float we = hh < H ? w[e * H + hh] : 0.f;
        t[hh] = ge * we;
        gsum[hh] += t[hh];
        bsum[hh] += be * we;
      }
      sw[e][0] = make_float4(t[0], t[1], t[2], t[3]);
      sw[e][1] = make_float4(t[4], t[5], t[6], t[7]);
    }
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gsum[hh] += __shfl_xor_sync(0xffffffffu, gsum[hh], o);
        bsum[hh] += __shfl_xor_sync(0xffffffffu, bsum[hh], o);
      }
    }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int hh = 0; hh < 8; ++hh) {
        spart[threadIdx.x >> 5][hh] = gsum[hh];
        spart[threadIdx.x >> 5][8 + hh] = bsum[hh];
      }
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const float acc = spart[0][threadIdx.x] + spart[1][threadIdx.x] + spart[2][threadIdx.x] + spart[3][threadIdx.x];
    if (threadIdx.x < 8) sG[threadIdx.x] = acc;
    else sBW[threadIdx.x - 8] = acc;
  }
  tc::cp_async_wait0();
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  if (i >= RR) return;
  const int64_t tok = swap ? (i % NI) * NJ + i / NI : i;
  const uint8_t* row = tile + threadIdx.x * TL::ROWB;
  float s = 0.f, q = 0.f;
  float2 p[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll 2
  for (int c = 0; c < C; c += 8) {
    Vec8<T> v;
    if constexpr (sizeof(T) == 2) {
      v.u = *reinterpret_cast<const uint4*>(row + c * 2);
    } else {
      v.a = *reinterpret_cast<const float4*>(row + c * 4);
      v.b = *reinterpret_cast<const float4*>(row + c * 4 + 16);
    }
    float f[8];
    cvt8(v, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float4 w0 = sw[c + e][0], w1 = sw[c + e][1];
      const float2 z2 = make_float2(f[e], f[e]);
      s += f[e];
      q = fmaf(f[e], f[e], q);
      p[0] = __ffma2_rn(z2, make_float2(w0.x, w0.y), p[0]);
      p[1] = __ffma2_rn(z2, make_float2(w0.z, w0.w), p[1]);
      p[2] = __ffma2_rn(z2, make_float2(w1.x, w1.y), p[2]);
      p[3] = __ffma2_rn(z2, make_float2(w1.z, w1.w), p[3]);
    }
  }
  const float mu = s / (float)C;
  const float inv = rsqrtf(fmaxf(q / (float)C - mu * mu, 0.f) + 1e-5f);
  const float ph[8] = {p[0].x, p[0].y, p[1].x, p[1].y, p[2].x, p[2].y, p[3].x, p[3].y};
#pragma unroll
  for (int hh = 0; hh < 8; ++hh)
    if (hh < H) nb[hh * RR + i] = from_f<T>(fmaf(inv, ph[hh] - mu * sG[hh], sBW[hh]));
  mean[tok] = mu;
  rstd[tok] = inv;
}

bool pair_bias_fwd_tpt(const void* z, int dt, const float* g, const float* b, const float* w, void* nb,
                       float* mean, float* rstd, int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap,
                       cudaStream_t s) {
  if (H > 8 || (C % 8) != 0 || (((uintptr_t)z) & 15) != 0) return false;
  const int64_t RR = NI * NJ;
  const unsigned grid = (unsigned)((RR + 127) / 128);
  bool done = true;
  auto go = [&](auto cc) {
    constexpr int CC = decltype(cc)::value;
    EVO_DISPATCH_T(dt, T, {
      auto k = pair_bias_fwd_tpt_kernel<CC, T>;
      constexpr int SMEM = PbTile<CC, T>::bytes;
      static bool attr = false;
      if (!attr) {
        EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        attr = true;
      }
      k<<<grid, 128, SMEM, s>>>((const T*)z, g, b, w, (T*)nb, mean, rstd, NI, NJ, (int)H, swap);
    });
  };
  if (C == 32) go(std::integral_constant<int, 32>{});
  else if (C == 64) go(std::integral_constant<int, 64>{});
  else if (C == 128) go(std::integral_constant<int, 128>{});
  else if (C == 256) go(std::integral_constant<int, 256>{});
  else done = false;
  if (done) {
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
  return done;
}
bool pair_bias_fwd_mma(const void* z, int dt, const float* g, const float* b, const float* w, void* nb,
                       float* mean, float* rstd, int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap,
                       cudaStream_t s);  // pair_bias_mma.cu
bool ln_pair_bias_fwd_mma(const void* z, int dt, const float* lg, const float* lb, const float* g, const float* b,
                          const float* w, void* xl, void* nb, float* mean, float* rstd, int64_t NI, int64_t NJ,
                          int64_t C, int64_t H, int swap, cudaStream_t s);  // pair_bias_mma.cu
int64_t pair_bias_bwd_vec_ws(int64_t C, int64_t H);
bool pair_bias_bwd_vec(const void* z, int dt, const float* mean, const float* rstd, const float* g,
                       const float* bln, const float* w, const float* dnb, int swap, float* dz,
                       float* dg, float* db, float* dw, int accumulate, void* ws, int64_t NI,
                       int64_t NJ, int64_t C, int64_t H, cudaStream_t s, __nv_bfloat16* dz16, float* dzsum,
                       bool* fused_out);

}  // namespace evo

using namespace evo;

extern "C" {

int evo_pair_bias_fwd_rect(const void* z, int dtype, const float* ln_g, const float* ln_b,
                           const float* w_bias, void* nb, float* mean, float* rstd, int64_t NI,
                           int64_t NJ, int64_t C, int64_t H, int swap_xy, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(H >= 1 && H <= PB_HMAX, EVO_ERR_UNSUPPORTED, "pair_bias: heads must be in [1,16]");
  EVO_REQUIRE(NI >= 0 && NJ >= 0, EVO_ERR_ARG, "pair_bias: negative extent");
  if (NI * NJ == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (pair_bias_fwd_mma(z, dtype, ln_g, ln_b, w_bias, nb, mean, rstd, NI, NJ, C, H, swap_xy, s))
    return EVO_OK;
  if (pair_bias_fwd_tpt(z, dtype, ln_g, ln_b, w_bias, nb, mean, rstd, NI, NJ, C, H, swap_xy, s))
    return EVO_OK;
  if (pair_bias_fwd_vec(z, dtype, ln_g, ln_b, w_bias, nb, mean, rstd, NI, NJ, C, H, swap_xy, s))
    return EVO_OK;
  unsigned grid = cdiv(NI * NJ, PB_WARPS);
  PB_NPL_DISPATCH(C, NPL, EVO_DISPATCH_T(dtype, T, {
    pair_bias_fwd_kernel<T, NPL><<<grid, PB_WARPS * 32, 0, s>>>(
        (const T*)z, ln_g, ln_b, w_bias, (T*)nb, mean, rstd, NI, NJ, (int)C, (int)H, swap_xy);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_ln_pair_bias_fwd(const void* z, int dtype, const float* ln_g, const float* ln_b, const float* bias_ln_g,
                         const float* bias_ln_b, const float* w_bias, void* xl, void* nb, float* mean, float* rstd,
                         int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap_xy, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(NI >= 0 && NJ >= 0 && H >= 1, EVO_ERR_ARG, "ln_pair_bias: bad extents");
  if (NI * NJ == 0) return EVO_OK;
  EVO_REQUIRE(ln_pair_bias_fwd_mma(z, dtype, ln_g, ln_b, bias_ln_g, bias_ln_b, w_bias, xl, nb, mean, rstd, NI, NJ, C,
                                   H, swap_xy, (cudaStream_t)stream),
              EVO_ERR_UNSUPPORTED, "ln_pair_bias: bf16, c_z = 128, H <= 8, >= 4096 tokens only");
  EVO_API_END
}

int evo_pair_bias_fwd(const void* z, int dtype, const float* ln_g, const float* ln_b,
                      const float* w_bias, void* nb, float* mean, float* rstd, int64_t R,
                      int64_t C, int64_t H, int swap_xy, void* stream) {
  return evo_pair_bias_fwd_rect(z, dtype, ln_g, ln_b, w_bias, nb, mean, rstd, R, R, C, H, swap_xy, stream);
}

int64_t evo_pair_bias_bwd_workspace(int64_t C, int64_t H) {
  const int64_t a = (int64_t)EVO_PARTIAL_BLOCKS * (C * H + 2 * C) * 4, b = pair_bias_bwd_vec_ws(C, H);
  return a > b ? a : b;
}

int evo_pair_bias_bwd_rect(const void* z, int dtype, const float* mean, const float* rstd,
                           const float* ln_g, const float* ln_b, const float* w_bias,
                           const float* dnb, int swap_xy, float* dz, float* dln_g,
                           float* dln_b, float* dw_bias, int accumulate, void* ws, int64_t NI,
                           int64_t NJ, int64_t C, int64_t H, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(H >= 1 && H <= PB_HMAX, EVO_ERR_UNSUPPORTED, "pair_bias: heads must be in [1,16]");
  EVO_REQUIRE(ws != nullptr, EVO_ERR_ARG, "pair_bias_bwd: workspace required");
  EVO_REQUIRE(NI >= 0 && NJ >= 0, EVO_ERR_ARG, "pair_bias: negative extent");
  if (NI * NJ == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (pair_bias_bwd_vec(z, dtype, mean, rstd, ln_g, ln_b, w_bias, dnb, swap_xy, dz, dln_g, dln_b,
                        dw_bias, accumulate, ws, NI, NJ, C, H, s, nullptr, nullptr, nullptr))
    return EVO_OK;
  const int64_t want = (NI * NJ + PB_WARPS - 1) / PB_WARPS;
  unsigned grid = (unsigned)(want < EVO_PARTIAL_BLOCKS ? want : EVO_PARTIAL_BLOCKS);
  const int64_t W = C * H + 2 * C;
  size_t smem = (size_t)PB_WARPS * W * sizeof(float);
  float* part = (float*)ws;
  PB_NPL_DISPATCH(C, NPL, EVO_DISPATCH_T(dtype, T, {
    auto k = pair_bias_bwd_kernel<T, NPL>;
    if (smem > 48 * 1024)
      EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, PB_WARPS * 32, smem, s>>>((const T*)z, mean, rstd, ln_g, ln_b, w_bias, dnb,
                                         swap_xy, dz, part, NI, NJ, (int)C, (int)H);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials(part, grid, C * H, dw_bias, accumulate, s, W);
  finalize_partials(part + C * H, grid, C, dln_g, accumulate, s, W);
  finalize_partials(part + C * H + C, grid, C, dln_b, accumulate, s, W);
  EVO_API_END
}

}  // extern "C"
namespace evo {
bool pair_bias_bwd_stream_ok(const void* z, int dt, const void* dz, const void* dz16, const float* mean,
                             const float* rstd, const float* dnb, int64_t NI, int64_t NJ, int64_t C,
                             int64_t H);  // glue_stream.cu
}
extern "C" {

int evo_pair_bias_bwd_ex(const void* z, int dtype, const float* mean, const float* rstd, const float* ln_g,
                         const float* ln_b, const float* w_bias, const float* dnb, int swap_xy, float* dz,
                         float* dln_g, float* dln_b, float* dw_bias, int accumulate, void* ws, int64_t NI, int64_t NJ,
                         int64_t C, int64_t H, void* dz16, float* dzsum, void* stream) {
  if (!dz16 && !dzsum)
    return evo_pair_bias_bwd_rect(z, dtype, mean, rstd, ln_g, ln_b, w_bias, dnb, swap_xy, dz, dln_g, dln_b, dw_bias,
                                  accumulate, ws, NI, NJ, C, H, stream);
  EVO_API_BEGIN
  EVO_REQUIRE(H >= 1 && H <= 8 && ws != nullptr && NI > 0 && NJ > 0, EVO_ERR_ARG, "pair_bias_bwd_ex: bad arguments");
  // decided before any work, so an unsupported call leaves dz untouched
  EVO_REQUIRE(pair_bias_bwd_stream_ok(z, dtype, dz, dz16, mean, rstd, dnb, NI, NJ, C, H), EVO_ERR_UNSUPPORTED,
              "pair_bias_bwd_ex: the fused bf16 copy / column sums need the streamed path "
              "(bf16, c_z = 128, H <= 8, >= 4096 tokens, a multiple of 4)");
  bool fused = false;
  EVO_REQUIRE(pair_bias_bwd_vec(z, dtype, mean, rstd, ln_g, ln_b, w_bias, dnb, swap_xy, dz, dln_g, dln_b, dw_bias,
                                accumulate, ws, NI, NJ, C, H, (cudaStream_t)stream, (__nv_bfloat16*)dz16, dzsum,
                                &fused) &&
                  fused,
              EVO_ERR_UNSUPPORTED, "pair_bias_bwd_ex: the fused bf16 copy / column sums need the streamed path "
                                   "(bf16, c_z = 128, H <= 8, >= 4096 tokens, a multiple of 4)");
  EVO_API_END
}

int evo_pair_bias_bwd(const void* z, int dtype, const float* mean, const float* rstd,
                      const float* ln_g, const float* ln_b, const float* w_bias,
                      const float* dnb, int swap_xy, float* dz, float* dln_g,
                      float* dln_b, float* dw_bias, int accumulate, void* ws, int64_t R,
                      int64_t C, int64_t H, void* stream) {
  return evo_pair_bias_bwd_rect(z, dtype, mean, rstd, ln_g, ln_b, w_bias, dnb, swap_xy, dz, dln_g, dln_b,
                                dw_bias, accumulate, ws, R, R, C, H, stream);
}

}  // extern "C"
