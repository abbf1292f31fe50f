// Kernels of the unfused gated-attention baseline, ``gated_attention_reference``
// (src/attention.py:78-115): the reference's fine-grained composition with
// materialised [B*S, H, R, R] logits, used as the oracle for the fused
// operator (tests/test_acceptance.py:46-71).  fp32 throughout; the GEMMs are
// the library's (evo_gemm), these are the pieces between them:
//   * softmax over the last dim of the logits after the mask bias
//     (m - 1) * 1e9 and the pair bias are added, in the reference's order
//     (src/attention.py:99-106) -- and its backward w * (g - sum(g * w));
//   * the sigmoid gate and the gated context (:111-113) and their backward;
//   * a fixed-order sum over rows (bias gradients, d(nb) = sum over B*S).
#include "common.cuh"
#include "reduce.cuh"

namespace evo {
namespace {

// one warp per logits row (bs, h, i); R up to a few thousand (strided loop)
__global__ void softmax_masked_rows_kernel(float* __restrict__ x, const float* __restrict__ mask, int64_t msb,
                                           int64_t msl, const float* __restrict__ nb, int64_t BS, int64_t H,
                                           int64_t R) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= BS * H * R) return;
  const int64_t i = row % R, h = (row / R) % H, bs = row / (R * H);
  float* xr = x + row * R;
  const float* nbr = nb ? nb + (h * R + i) * R : nullptr;
  float m = -INFINITY;
  for (int64_t j = lane; j < R; j += 32) {
    float v = xr[j] + (mask[bs * msb + j * msl] - 1.0f) * 1e9f;  // logits + maskbias (:101)
    if (nbr) v += nbr[j];                                         // + nb (:104)
    xr[j] = v;
    m = fmaxf(m, v);
  }
  m = warp_max(m);
  float sum = 0.f;
  for (int64_t j = lane; j < R; j += 32) {
    const float e = expf(xr[j] - m);
    xr[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  for (int64_t j = lane; j < R; j += 32) xr[j] = xr[j] / sum;
}

// g <- w * (g - sum_j g * w), per row
__global__ void softmax_rows_bwd_kernel(const float* __restrict__ w, float* __restrict__ g, int64_t rows,
                                        int64_t R) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* wr = w + row * R;
  float* gr = g + row * R;
  float d = 0.f;
  for (int64_t j = lane; j < R; j += 32) d += gr[j] * wr[j];
  d = warp_sum(d);
  for (int64_t j = lane; j < R; j += 32) gr[j] = wr[j] * (gr[j] - d);
}

__global__ void gate_fwd_kernel(const float* __restrict__ gp, const float* __restrict__ ctx, float* __restrict__ gate,
                                float* __restrict__ gated, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float g = 1.0f / (1.0f + expf(-gp[e]));  // src/tensor.py:290-292
    gate[e] = g;
    gated[e] = ctx[e] * g;
  }
}

__global__ void gate_bwd_kernel(const float* __restrict__ dgated, const float* __restrict__ gate,
                                const float* __restrict__ ctx, float* __restrict__ dctx, float* __restrict__ dgp,
                                int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float g = gate[e], d = dgated[e];
    dctx[e] = d * g;
    dgp[e] = d * ctx[e] * g * (1.0f - g);
  }
}

// out[c] (+)= sum_r x[r, c], rows summed in ascending order (deterministic)
__global__ void sum_rows_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, float* __restrict__ out,
                                int accumulate) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int64_t r = 0; r < rows; ++r) acc += x[r * cols + c];
    out[c] = accumulate ? out[c] + acc : acc;
  }
}

unsigned grid_for(int64_t n, int per_block) {
  const int64_t b = (n + per_block - 1) / per_block;
  return (unsigned)(b < 65535 * 64 ? b : 65535 * 64);
}

}  // namespace
}  // namespace evo

using namespace evo;

extern "C" {

int evo_softmax_masked_rows(float* x, const float* mask, int64_t mask_sb, int64_t mask_sl, const float* nb,
                            int64_t BS, int64_t H, int64_t R, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(BS >= 0 && H > 0 && R > 0 && mask != nullptr, EVO_ERR_ARG, "softmax_masked_rows: bad arguments");
  const int64_t rows = BS * H * R;
  if (rows == 0) return EVO_OK;
  softmax_masked_rows_kernel<<<grid_for(rows, 8), 256, 0, (cudaStream_t)stream>>>(x, mask, mask_sb, mask_sl, nb, BS,
                                                                                  H, R);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_softmax_rows_bwd(const float* w, float* g, int64_t rows, int64_t R, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(rows >= 0 && R > 0, EVO_ERR_ARG, "softmax_rows_bwd: bad extents");
  if (rows == 0) return EVO_OK;
  softmax_rows_bwd_kernel<<<grid_for(rows, 8), 256, 0, (cudaStream_t)stream>>>(w, g, rows, R);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_gate_fwd(const float* gp, const float* ctx, float* gate, float* gated, int64_t n, void* stream) {
  EVO_API_BEGIN
  if (n == 0) return EVO_OK;
  gate_fwd_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(gp, ctx, gate, gated, n);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_gate_bwd(const float* dgated, const float* gate, const float* ctx, float* dctx, float* dgp, int64_t n,
                 void* stream) {
  EVO_API_BEGIN
  if (n == 0) return EVO_OK;
  gate_bwd_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(dgated, gate, ctx, dctx, dgp, n);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_sum_rows(const float* x, int64_t rows, int64_t cols, float* out, int accumulate, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(rows >= 0 && cols >= 0, EVO_ERR_ARG, "sum_rows: bad extents");
  if (cols == 0) return EVO_OK;
  sum_rows_kernel<<<grid_for(cols, 256), 256, 0, (cudaStream_t)stream>>>(x, rows, cols, out, accumulate);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

}  // extern "C"
