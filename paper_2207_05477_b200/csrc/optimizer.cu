// Fused-buffer optimizer tail over the pooled parameter regions
// (src/fusion.py:150-233, the paper's "tensor fusion"):
//   launch 1  evo_sumsq_f64   fp64 sum of squares of the whole grad region
//   launch 2  (finalize of the fp64 partials)
//   launch 3  evo_adam_clip_ema  clip scale + Adam + EMA (+ bf16 shadow) in
//             one vectorised pass over params/grads/adam_m/adam_v/ema.
// The reference's (1, 2, 1, 1) launch budget for (sync, clip, update, EMA)
// becomes 3 kernels in total.  Elementwise arithmetic uses explicit
// round-to-nearest intrinsics (no FMA contraction) in the reference's
// evaluation order, so parameters, moments and EMA are bitwise identical to
// the numpy reference.
#include "common.cuh"
#include "reduce.cuh"

namespace evo {

constexpr int OPT_THREADS = 256;

__global__ void __launch_bounds__(OPT_THREADS) sumsq_kernel(const float* __restrict__ g, int64_t n,
                                                            double* __restrict__ partials) {
  __shared__ double red[OPT_THREADS / 32];
  double acc = 0.0;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = g4[i];
    acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)g[i] * g[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < OPT_THREADS / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

// Also advances the device step counter and looks up this step's Adam bias
// corrections bc = (1 - b1^t, 1 - b2^t) in fp32, tabulated on the host with the
// reference's own expression (src/fusion.py:189-192); past the end of the
// table both corrections have rounded to exactly 1.0f, so clamping is exact.
// Keeping t on the device is what lets a captured CUDA graph replay the step.
__global__ void sumsq_final_kernel(const double* __restrict__ partials, int G, double* out,
                                   int64_t* __restrict__ step, const float* __restrict__ bc_table,
                                   int64_t table_len, float* __restrict__ bc_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < G; ++i) s += partials[i];
    *out = s;
    if (step) {
      const int64_t t = ++*step;
      const int64_t i = (t < table_len ? t : table_len) - 1;
      bc_out[0] = bc_table[i];
      bc_out[1] = bc_table[table_len + i];
    }
  }
}

struct AdamArgs {
  double clip;
  float lr, b1, omb1, b2, omb2, eps, bc1, bc2, decay, omdecay;
};

__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, float& e,
                                         float scale, bool do_scale, const AdamArgs& a) {
  if (do_scale) g = __fmul_rn(g, scale);                                   // fusion.py:181
  m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));                 // :200
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(a.omb2, __fmul_rn(g, g)));   // :201
  const float mh = __fdiv_rn(m, a.bc1);                                    // :202
  const float vh = __fdiv_rn(v, a.bc2);                                    // :203
  const float upd = __fdiv_rn(__fmul_rn(a.lr, mh), __fadd_rn(__fsqrt_rn(vh), a.eps));
  p = __fsub_rn(p, upd);                                                   // :204
  e = __fadd_rn(__fmul_rn(a.decay, e), __fmul_rn(a.omdecay, p));           // :220
}

__global__ void __launch_bounds__(OPT_THREADS) adam_clip_ema_kernel(
    float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
    float* __restrict__ v, float* __restrict__ ema, __nv_bfloat16* __restrict__ pb, int64_t n,
    const double* __restrict__ sumsq, AdamArgs a, const float* __restrict__ bc_dev) {
  if (bc_dev) {  // this step's bias corrections, written by sumsq_final_kernel
    a.bc1 = bc_dev[0];
    a.bc2 = bc_dev[1];
  }
  const double norm = sqrt(*sumsq);
  const bool do_scale = norm > a.clip;
  const float scale = do_scale ? (float)(a.clip / norm) : 1.0f;            // :176-178
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float4 ee = reinterpret_cast<float4*>(ema)[i];
    adam_one(pp.x, gg.x, mm.x, vv.x, ee.x, scale, do_scale, a);
    adam_one(pp.y, gg.y, mm.y, vv.y, ee.y, scale, do_scale, a);
    adam_one(pp.z, gg.z, mm.z, vv.z, ee.z, scale, do_scale, a);
    adam_one(pp.w, gg.w, mm.w, vv.w, ee.w, scale, do_scale, a);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(ema)[i] = ee;
    if (pb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(pp.z, pp.w);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pb)[i] = packed;
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float pp = p[i], mm = m[i], vv = v[i], ee = ema[i];
    adam_one(pp, g[i], mm, vv, ee, scale, do_scale, a);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    ema[i] = ee;
    if (pb) pb[i] = __float2bfloat16_rn(pp);
  }
}

}  // namespace evo

using namespace evo;

extern "C" {

int64_t evo_sumsq_workspace(void) { return 1024 * 8; }

int evo_sumsq_f64(const float* g, int64_t n, double* out, void* ws, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(((uintptr_t)g & 15) == 0, EVO_ERR_ARG, "sumsq: grad region must be 16-B aligned");
  cudaStream_t s = (cudaStream_t)stream;
  int G = num_sms() * 4;
  if (G > 1024) G = 1024;
  sumsq_kernel<<<G, OPT_THREADS, 0, s>>>(g, n, (double*)ws);
  EVO_LAUNCH_CHECK();
  sumsq_final_kernel<<<1, 32, 0, s>>>((const double*)ws, G, out, nullptr, nullptr, 0, nullptr);
  EVO_LAUNCH_CHECK();
  count_launch(2);
  EVO_API_END
}

int evo_sumsq_f64_step(const float* g, int64_t n, double* out, void* ws, int64_t* step,
                       const float* bc_table, int64_t table_len, float* bc_out, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(((uintptr_t)g & 15) == 0, EVO_ERR_ARG, "sumsq: grad region must be 16-B aligned");
  EVO_REQUIRE(step && bc_table && bc_out && table_len >= 1, EVO_ERR_ARG, "sumsq_step: bad step arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int G = num_sms() * 4;
  if (G > 1024) G = 1024;
  sumsq_kernel<<<G, OPT_THREADS, 0, s>>>(g, n, (double*)ws);
  EVO_LAUNCH_CHECK();
  sumsq_final_kernel<<<1, 32, 0, s>>>((const double*)ws, G, out, step, bc_table, table_len, bc_out);
  EVO_LAUNCH_CHECK();
  count_launch(2);
  EVO_API_END
}

namespace {
int adam_launch(float* p, const float* g, float* m, float* v, float* ema, void* p_bf16, int64_t n,
                const double* sumsq, double clip, float lr, float b1, float omb1, float b2, float omb2,
                float eps, float bc1, float bc2, const float* bc_dev, float decay, float omdecay,
                void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE((((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v | (uintptr_t)ema) & 15) == 0,
              EVO_ERR_ARG, "adam: regions must be 16-B aligned");
  EVO_REQUIRE(((uintptr_t)p_bf16 & 7) == 0, EVO_ERR_ARG, "adam: bf16 shadow must be 8-B aligned");
  AdamArgs a{clip, lr, b1, omb1, b2, omb2, eps, bc1, bc2, decay, omdecay};
  int64_t want = (n / 4 + OPT_THREADS - 1) / OPT_THREADS;
  int64_t cap = (int64_t)num_sms() * 8;
  unsigned G = (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
  adam_clip_ema_kernel<<<G, OPT_THREADS, 0, (cudaStream_t)stream>>>(
      p, g, m, v, ema, (__nv_bfloat16*)p_bf16, n, sumsq, a, bc_dev);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}
}  // namespace

int evo_adam_clip_ema(float* p, const float* g, float* m, float* v, float* ema, void* p_bf16,
                      int64_t n, const double* sumsq, double clip, float lr, float b1, float omb1,
                      float b2, float omb2, float eps, float bc1, float bc2, float decay,
                      float omdecay, void* stream) {
  return adam_launch(p, g, m, v, ema, p_bf16, n, sumsq, clip, lr, b1, omb1, b2, omb2, eps, bc1, bc2, nullptr,
                     decay, omdecay, stream);
}

int evo_adam_clip_ema_dev(float* p, const float* g, float* m, float* v, float* ema, void* p_bf16,
                          int64_t n, const double* sumsq, double clip, float lr, float b1, float omb1,
                          float b2, float omb2, float eps, const float* bc, float decay, float omdecay,
                          void* stream) {
  if (!bc) {
    set_error("adam_dev: null bias-correction pointer");
    return EVO_ERR_ARG;
  }
  return adam_launch(p, g, m, v, ema, p_bf16, n, sumsq, clip, lr, b1, omb1, b2, omb2, eps, 1.0f, 1.0f, bc,
                     decay, omdecay, stream);
}

}  // extern "C"
