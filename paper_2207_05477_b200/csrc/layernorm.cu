// LayerNorm forward/backward over the channel dim (src/tensor.py:173-208).
// One warp per row; lane l owns channels l, l+32, ... (coalesced).  The
// backward fuses the residual-gradient add and produces deterministic
// per-block partials for dgamma/dbeta.
#include "common.cuh"
#include "reduce.cuh"

namespace evo {

constexpr int LN_WARPS = 8;

template <typename TX, typename TY, int NPL>
__global__ void __launch_bounds__(LN_WARPS * 32) ln_fwd_kernel(
    const TX* __restrict__ x, const float* __restrict__ g, const float* __restrict__ b,
    TY* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int64_t rows, int C,
    float eps) {
  const int lane = threadIdx.x & 31;
  int64_t row = blockIdx.x * (int64_t)LN_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const TX* xr = x + row * C;
  float v[NPL];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    v[k] = c < C ? to_f(xr[c]) : 0.f;
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
  const float var = warp_sum(q) / (float)C;
  const float inv = 1.0f / sqrtf(var + eps);
  TY* yr = y + row * C;
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    if (c < C) yr[c] = from_f<TY>((v[k] - mu) * inv * g[c] + b[c]);
  }
  if (lane == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = inv;
  }
}

template <typename TX, typename TD, int NPL>
__global__ void __launch_bounds__(LN_WARPS * 32) ln_bwd_kernel(
    const TX* __restrict__ x, const TD* __restrict__ dy, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ g, const float* dres, float* dx,
    float* __restrict__ partials, int64_t rows, int C) {
  extern __shared__ float sm[];  // [LN_WARPS][2C]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float dg[NPL], db[NPL], gg[NPL];
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    dg[k] = 0.f;
    db[k] = 0.f;
    int c = lane + 32 * k;
    gg[k] = c < C ? g[c] : 0.f;
  }
  for (int64_t row = blockIdx.x * (int64_t)LN_WARPS + warp; row < rows;
       row += (int64_t)gridDim.x * LN_WARPS) {
    const float mu = mean[row], inv = rstd[row];
    float xh[NPL], dxh[NPL];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      int c = lane + 32 * k;
      float xv = c < C ? to_f(x[row * C + c]) : 0.f;
      float d = c < C ? to_f(dy[row * C + c]) : 0.f;
      xh[k] = c < C ? (xv - mu) * inv : 0.f;
      dxh[k] = d * gg[k];
      dg[k] += d * xh[k];
      db[k] += d;
      s1 += dxh[k];
      s2 += dxh[k] * xh[k];
    }
    const float m1 = warp_sum(s1) / (float)C;
    const float m2 = warp_sum(s2) / (float)C;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      int c = lane + 32 * k;
      if (c < C) {
        float v = inv * (dxh[k] - m1 - xh[k] * m2);
        if (dres) v += dres[row * C + c];
        dx[row * C + c] = v;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    int c = lane + 32 * k;
    if (c < C) {
      sm[warp * 2 * C + c] = dg[k];
      sm[warp * 2 * C + C + c] = db[k];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) {
    float acc = 0.f;
    for (int w = 0; w < LN_WARPS; ++w) acc += sm[w * 2 * C + c];
    partials[blockIdx.x * 2 * C + c] = acc;
  }
}

#define LN_NPL_DISPATCH(C, NPL, ...)                                          \
  do {                                                                        \
    if ((C) <= 32) { constexpr int NPL = 1; __VA_ARGS__; }                    \
    else if ((C) <= 64) { constexpr int NPL = 2; __VA_ARGS__; }               \
    else if ((C) <= 128) { constexpr int NPL = 4; __VA_ARGS__; }              \
    else if ((C) <= 256) { constexpr int NPL = 8; __VA_ARGS__; }              \
    else if ((C) <= 512) { constexpr int NPL = 16; __VA_ARGS__; }             \
    else if ((C) <= 1024) { constexpr int NPL = 32; __VA_ARGS__; }            \
    else throw Error(EVO_ERR_UNSUPPORTED, "layernorm: C > 1024");             \
  } while (0)

// vectorised kernels (glue.cu)
bool ln_fwd_vec(const void* x, int xdt, const float* g, const float* b, void* y, int ydt,
                float* mean, float* rstd, int64_t rows, int64_t C, float eps, cudaStream_t s);
int64_t ln_bwd_vec_ws(int64_t C);
bool ln_bwd_vec(const void* x, int xdt, const void* dy, int dydt, const float* mean, const float* rstd,
                const float* g, const float* dres, float* dx, __nv_bfloat16* dx16, float* dgamma,
                float* dbeta, float* dxsum, int accumulate, void* ws, int64_t rows, int64_t C,
                cudaStream_t s);

}  // namespace evo

using namespace evo;

extern "C" {

int evo_layernorm_fwd(const void* x, int x_dtype, const float* gamma, const float* beta, void* y,
                      int y_dtype, float* mean, float* rstd, int64_t rows, int64_t C, float eps,
                      void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(C > 0, EVO_ERR_ARG, "layernorm: C must be positive");
  if (rows == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (ln_fwd_vec(x, x_dtype, gamma, beta, y, y_dtype, mean, rstd, rows, C, eps, s)) return EVO_OK;
  unsigned grid = cdiv(rows, LN_WARPS);
  LN_NPL_DISPATCH(C, NPL, EVO_DISPATCH_T(x_dtype, TX, EVO_DISPATCH_T(y_dtype, TY, {
    ln_fwd_kernel<TX, TY, NPL><<<grid, LN_WARPS * 32, 0, s>>>(
        (const TX*)x, gamma, beta, (TY*)y, mean, rstd, rows, (int)C, eps);
  })));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int64_t evo_layernorm_bwd_workspace(int64_t rows, int64_t C) {
  (void)rows;
  const int64_t a = (int64_t)EVO_PARTIAL_BLOCKS * 2 * C * 4, b = ln_bwd_vec_ws(C);
  return a > b ? a : b;
}

int evo_layernorm_bwd_ex(const void* x, int x_dtype, const void* dy, int dy_dtype,
                         const float* mean, const float* rstd, const float* gamma,
                         const float* dres, float* dx, void* dx_bf16, float* dxsum,
                         float* dgamma, float* dbeta, int accumulate, void* ws, int64_t rows,
                         int64_t C, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(C > 0 && ws, EVO_ERR_ARG, "layernorm_bwd: bad arguments");
  if (rows == 0) return EVO_OK;
  const bool ok = ln_bwd_vec(x, x_dtype, dy, dy_dtype, mean, rstd, gamma, dres, dx,
                             (__nv_bfloat16*)dx_bf16, dgamma, dbeta, dxsum, accumulate, ws, rows,
                             C, (cudaStream_t)stream);
  EVO_REQUIRE(ok, EVO_ERR_UNSUPPORTED,
              "layernorm_bwd_ex: needs a power-of-two width in [32, 1024] and 16-B aligned rows");
  EVO_API_END
}

int evo_layernorm_bwd(const void* x, int x_dtype, const void* dy, int dy_dtype, const float* mean,
                      const float* rstd, const float* gamma, const float* dres, float* dx,
                      float* dgamma, float* dbeta, int accumulate, void* ws, int64_t rows,
                      int64_t C, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(C > 0 && ws, EVO_ERR_ARG, "layernorm_bwd: bad arguments");
  if (rows == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (ln_bwd_vec(x, x_dtype, dy, dy_dtype, mean, rstd, gamma, dres, dx, nullptr, dgamma, dbeta,
                 nullptr, accumulate, ws, rows, C, s))
    return EVO_OK;
  int64_t want = (rows + LN_WARPS - 1) / LN_WARPS;
  unsigned grid = (unsigned)(want < EVO_PARTIAL_BLOCKS ? want : EVO_PARTIAL_BLOCKS);
  size_t smem = (size_t)LN_WARPS * 2 * C * sizeof(float);
  LN_NPL_DISPATCH(C, NPL, EVO_DISPATCH_T(x_dtype, TX, EVO_DISPATCH_T(dy_dtype, TD, {
    auto k = ln_bwd_kernel<TX, TD, NPL>;
    if (smem > 48 * 1024) EVO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, LN_WARPS * 32, smem, s>>>((const TX*)x, (const TD*)dy, mean, rstd, gamma, dres, dx,
                                         (float*)ws, rows, (int)C);
  })));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials((const float*)ws, grid, C, dgamma, accumulate, s, 2 * C);
  finalize_partials((const float*)ws + C, grid, C, dbeta, accumulate, s, 2 * C);
  EVO_API_END
}

}  // extern "C"
