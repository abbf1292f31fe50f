// Triangle multiplicative update glue (AlphaFold2 Supplementary Alg. 11/12;
// absent from the reference, which lists it only as planner inventory,
// src/planner.py:37-45).  The two contractions o[c] = a[c] b[c]^T (outgoing)
// / a[c]^T b[c] (incoming) are channel-batched [R x R] GEMMs (evo_gemm,
// batched); these kernels produce and consume their channel-major operands:
//   gate_fwd   a = sigmoid(ag + bag) * (ap + bap) * mask, b likewise,
//              token-major projections -> channel-major [ch, R*R]
//   gate_bwd   channel-major da/db -> token-major d(projections)
//   transpose  [rows, cols] <-> [cols, rows] (smem tiled, coalesced both ways)
//   gated residual  out = z + sigmoid(gp + bg) * (y + by) and its backward
#include "common.cuh"
#include "tc_common.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace evo {

namespace {

constexpr int TT = 32;  // tile edge

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + __expf(-x)); }

// proj: [RR, ld] with column blocks [ap | ag | bp | bg] of width ch
template <typename T>
__global__ void __launch_bounds__(256) trimul_gate_fwd_kernel(
    const T* __restrict__ proj, int64_t ld, const float* __restrict__ bap, const float* __restrict__ bag,
    const float* __restrict__ bbp, const float* __restrict__ bbg, const float* __restrict__ mask,
    T* __restrict__ a_cm, T* __restrict__ b_cm, int64_t RR, int ch) {
  __shared__ float ta[TT][TT + 1], tb[TT][TT + 1];
  const int64_t t0 = (int64_t)blockIdx.x * TT;
  const int c0 = blockIdx.y * TT;
  const int tx = threadIdx.x % TT, ty = threadIdx.x / TT;  // 32 x 8
  for (int r = ty; r < TT; r += 8) {
    const int64_t t = t0 + r;
    const int c = c0 + tx;
    float av = 0.f, bv = 0.f;
    if (t < RR && c < ch) {
      const T* row = proj + t * ld;
      const float m = mask[t];
      av = sigm(to_f(row[ch + c]) + bag[c]) * (to_f(row[c]) + bap[c]) * m;
      bv = sigm(to_f(row[3 * ch + c]) + bbg[c]) * (to_f(row[2 * ch + c]) + bbp[c]) * m;
    }
    ta[r][tx] = av;
    tb[r][tx] = bv;
  }
  __syncthreads();
  for (int r = ty; r < TT; r += 8) {
    const int c = c0 + r;
    const int64_t t = t0 + tx;
    if (c < ch && t < RR) {
      a_cm[(int64_t)c * RR + t] = from_f<T>(ta[tx][r]);
      b_cm[(int64_t)c * RR + t] = from_f<T>(tb[tx][r]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) trimul_gate_bwd_kernel(
    const T* __restrict__ proj, int64_t ld, const float* __restrict__ bap, const float* __restrict__ bag,
    const float* __restrict__ bbp, const float* __restrict__ bbg, const float* __restrict__ mask,
    const T* __restrict__ da_cm, const T* __restrict__ db_cm, T* __restrict__ dproj, int64_t RR, int ch) {
  __shared__ float ta[TT][TT + 1], tb[TT][TT + 1];
  const int64_t t0 = (int64_t)blockIdx.x * TT;
  const int c0 = blockIdx.y * TT;
  const int tx = threadIdx.x % TT, ty = threadIdx.x / TT;
  for (int r = ty; r < TT; r += 8) {  // read channel-major rows (coalesced along t)
    const int c = c0 + r;
    const int64_t t = t0 + tx;
    ta[r][tx] = (c < ch && t < RR) ? to_f(da_cm[(int64_t)c * RR + t]) : 0.f;
    tb[r][tx] = (c < ch && t < RR) ? to_f(db_cm[(int64_t)c * RR + t]) : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < TT; r += 8) {  // write token-major rows (coalesced along c)
    const int64_t t = t0 + r;
    const int c = c0 + tx;
    if (t < RR && c < ch) {
      const T* row = proj + t * ld;
      T* drow = dproj + t * 4 * ch;
      const float m = mask[t];
      const float da = ta[tx][r] * m, db = tb[tx][r] * m;
      const float ap = to_f(row[c]) + bap[c], sa = sigm(to_f(row[ch + c]) + bag[c]);
      const float bp = to_f(row[2 * ch + c]) + bbp[c], sb = sigm(to_f(row[3 * ch + c]) + bbg[c]);
      drow[c] = from_f<T>(da * sa);
      drow[ch + c] = from_f<T>(da * ap * sa * (1.0f - sa));
      drow[2 * ch + c] = from_f<T>(db * sb);
      drow[3 * ch + c] = from_f<T>(db * bp * sb * (1.0f - sb));
    }
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) transpose_kernel(const TI* __restrict__ x, TO* __restrict__ y,
                                                        int64_t rows, int64_t cols) {
  __shared__ float t[TT][TT + 1];
  const int64_t r0 = (int64_t)blockIdx.y * TT, c0 = (int64_t)blockIdx.x * TT;
  const int tx = threadIdx.x % TT, ty = threadIdx.x / TT;
  for (int r = ty; r < TT; r += 8)
    t[r][tx] = (r0 + r < rows && c0 + tx < cols) ? to_f(x[(r0 + r) * cols + c0 + tx]) : 0.f;
  __syncthreads();
  for (int r = ty; r < TT; r += 8)
    if (c0 + r < cols && r0 + tx < rows) y[(c0 + r) * rows + r0 + tx] = from_f<TO>(t[tx][r]);
}

// 64 x 64 tiles, 16-byte accesses on both sides: each thread loads two 8-wide
// row chunks, the tile goes through shared memory (fp32, padded), and each
// thread stores two 8-wide chunks of the transposed tile
template <typename TI>
__device__ __forceinline__ void ld8f(const TI* p, float (&f)[8]);
template <>
__device__ __forceinline__ void ld8f<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = tc::bf16x2_f2(w[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void ld8f<float>(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}

template <typename TI>
__global__ void __launch_bounds__(256) transpose_vec_kernel(const TI* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                                            int64_t rows, int64_t cols) {
  __shared__ float t[64][65];
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int idx = threadIdx.x + q * 256, r = idx >> 3, c8 = (idx & 7) * 8;
    float f[8];
    ld8f<TI>(x + (r0 + r) * cols + c0 + c8, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) t[r][c8 + e] = f[e];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int idx = threadIdx.x + q * 256, oc = idx >> 3, r8 = (idx & 7) * 8;  // output row = input column
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = tc::pack_bf16(t[r8 + 2 * k][oc], t[r8 + 2 * k + 1][oc]);
    *reinterpret_cast<uint4*>(y + (c0 + oc) * rows + r0 + r8) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// out = res + sigmoid(gp + bg) * (y + by); g saved
template <typename T>
__global__ void gated_residual_kernel(const T* __restrict__ res, const T* __restrict__ gp, int64_t ld_gp,
                                      const float* __restrict__ bg, const T* __restrict__ y,
                                      const float* __restrict__ by, T* __restrict__ g_out,
                                      T* __restrict__ out, int64_t rows, int64_t C) {
  const int64_t n = rows * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / C, c = e % C;
    const float gv = sigm(to_f(gp[r * ld_gp + c]) + bg[c]);
    g_out[e] = from_f<T>(gv);
    out[e] = from_f<T>(to_f(res[e]) + gv * (to_f(y[e]) + by[c]));
  }
}

// dyb = dout * g ;  dgp = dout * (y + by) * g * (1 - g)
template <typename T>
__global__ void gated_residual_bwd_kernel(const float* __restrict__ dout, const T* __restrict__ g,
                                          const T* __restrict__ y, const float* __restrict__ by,
                                          T* __restrict__ dyb, T* __restrict__ dgp, int64_t rows, int64_t C) {
  const int64_t n = rows * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % C;
    const float d = dout[e], gv = to_f(g[e]);
    dyb[e] = from_f<T>(d * gv);
    dgp[e] = from_f<T>(d * (to_f(y[e]) + by[c]) * gv * (1.0f - gv));
  }
}

// ---- 16-byte vector forms (ch % 32 == 0, RR % 8 == 0, 16-B aligned rows) ----
// A block covers 64 tokens x 32 channels: the token-major side is read /
// written as 8-channel vectors (thread = token, channel group), the
// channel-major side as 8-token vectors, through a transposing smem tile.

template <typename T>
__global__ void __launch_bounds__(256) trimul_gate_fwd_vec_kernel(
    const T* __restrict__ proj, int64_t ld, const float* __restrict__ bap, const float* __restrict__ bag,
    const float* __restrict__ bbp, const float* __restrict__ bbg, const float* __restrict__ mask,
    T* __restrict__ a_cm, T* __restrict__ b_cm, int64_t RR, int ch) {
  __shared__ float sa[32][65], sb[32][65];
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int c0 = blockIdx.y * 32;
  {
    const int tt = threadIdx.x >> 2, cg = threadIdx.x & 3;
    const int64_t t = t0 + tt;
    const int c = c0 + cg * 8;
    float ap[8], ag[8], bp[8], bgv[8];
    if (t < RR) {
      const T* row = proj + t * ld;
      ld8(row + c, ap);
      ld8(row + ch + c, ag);
      ld8(row + 2 * ch + c, bp);
      ld8(row + 3 * ch + c, bgv);
      const float m = mask[t];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sa[cg * 8 + u][tt] = sigm(ag[u] + bag[c + u]) * (ap[u] + bap[c + u]) * m;
        sb[cg * 8 + u][tt] = sigm(bgv[u] + bbg[c + u]) * (bp[u] + bbp[c + u]) * m;
      }
    }
  }
  __syncthreads();
  const int r = threadIdx.x >> 3, seg = threadIdx.x & 7;
  const int64_t tb = t0 + seg * 8;
  if (tb < RR) {  // RR % 8 == 0
    float va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) va[u] = sa[r][seg * 8 + u], vb[u] = sb[r][seg * 8 + u];
    st8(a_cm + (int64_t)(c0 + r) * RR + tb, va);
    st8(b_cm + (int64_t)(c0 + r) * RR + tb, vb);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) trimul_gate_bwd_vec_kernel(
    const T* __restrict__ proj, int64_t ld, const float* __restrict__ bap, const float* __restrict__ bag,
    const float* __restrict__ bbp, const float* __restrict__ bbg, const float* __restrict__ mask,
    const T* __restrict__ da_cm, const T* __restrict__ db_cm, T* __restrict__ dproj, int64_t RR, int ch) {
  __shared__ float sa[32][65], sb[32][65];
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int c0 = blockIdx.y * 32;
  {
    const int r = threadIdx.x >> 3, seg = threadIdx.x & 7;
    const int64_t tb = t0 + seg * 8;
    float va[8], vb[8];
    if (tb < RR) {
      ld8(da_cm + (int64_t)(c0 + r) * RR + tb, va);
      ld8(db_cm + (int64_t)(c0 + r) * RR + tb, vb);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) va[u] = vb[u] = 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) sa[r][seg * 8 + u] = va[u], sb[r][seg * 8 + u] = vb[u];
  }
  __syncthreads();
  const int tt = threadIdx.x >> 2, cg = threadIdx.x & 3;
  const int64_t t = t0 + tt;
  if (t >= RR) return;
  const int c = c0 + cg * 8;
  const T* row = proj + t * ld;
  T* drow = dproj + t * 4 * ch;
  float ap[8], ag[8], bp[8], bgv[8], o0[8], o1[8], o2[8], o3[8];
  ld8(row + c, ap);
  ld8(row + ch + c, ag);
  ld8(row + 2 * ch + c, bp);
  ld8(row + 3 * ch + c, bgv);
  const float m = mask[t];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float da = sa[cg * 8 + u][tt] * m, db = sb[cg * 8 + u][tt] * m;
    const float a_p = ap[u] + bap[c + u], sa_ = sigm(ag[u] + bag[c + u]);
    const float b_p = bp[u] + bbp[c + u], sb_ = sigm(bgv[u] + bbg[c + u]);
    o0[u] = da * sa_;
    o1[u] = da * a_p * sa_ * (1.0f - sa_);
    o2[u] = db * sb_;
    o3[u] = db * b_p * sb_ * (1.0f - sb_);
  }
  st8(drow + c, o0);
  st8(drow + ch + c, o1);
  st8(drow + 2 * ch + c, o2);
  st8(drow + 3 * ch + c, o3);
}

// gated residual, 8 elements of one row per thread
template <typename T>
__global__ void gated_residual_vec_kernel(const T* __restrict__ res, const T* __restrict__ gp, int64_t ld_gp,
                                          const float* __restrict__ bg, const T* __restrict__ y,
                                          const float* __restrict__ by, T* __restrict__ g_out, T* __restrict__ out,
                                          int64_t rows, int64_t C) {
  const int64_t n8 = rows * C / 8;
  for (int64_t e8 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e8 < n8;
       e8 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e8 * 8, r = e / C, c = e % C;
    float rv[8], gv[8], yv[8], go[8], ov[8];
    ld8(res + e, rv);
    ld8(gp + r * ld_gp + c, gv);
    ld8(y + e, yv);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      go[u] = sigm(gv[u] + bg[c + u]);
      ov[u] = rv[u] + go[u] * (yv[u] + by[c + u]);
    }
    st8(g_out + e, go);
    st8(out + e, ov);
  }
}

template <typename T>
__global__ void gated_residual_bwd_vec_kernel(const float* __restrict__ dout, const T* __restrict__ g,
                                              const T* __restrict__ y, const float* __restrict__ by,
                                              T* __restrict__ dyb, T* __restrict__ dgp, int64_t rows, int64_t C) {
  const int64_t n8 = rows * C / 8;
  for (int64_t e8 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e8 < n8;
       e8 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e8 * 8, c = e % C;
    float dv[8], gv[8], yv[8], a[8], b[8];
    ld8(dout + e, dv);
    ld8(g + e, gv);
    ld8(y + e, yv);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = dv[u] * gv[u];
      b[u] = dv[u] * (yv[u] + by[c + u]) * gv[u] * (1.0f - gv[u]);
    }
    st8(dyb + e, a);
    st8(dgp + e, b);
  }
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace
}  // namespace evo

using namespace evo;

extern "C" {

int evo_trimul_gate_fwd(const void* proj, int64_t ld, const float* b_ap, const float* b_ag,
                        const float* b_bp, const float* b_bg, const float* mask, void* a_cm,
                        void* b_cm, int64_t RR, int64_t ch, int dtype, void* stream) {
  EVO_API_BEGIN
  const int64_t es = dtype == EVO_F32 ? 4 : 2;
  if (ch % 32 == 0 && RR % 8 == 0 && (ld * es) % 16 == 0 && al16(proj) && al16(a_cm) && al16(b_cm)) {
    dim3 g2(cdiv(RR, 64), (unsigned)(ch / 32));
    EVO_DISPATCH_T(dtype, T, {
      trimul_gate_fwd_vec_kernel<T><<<g2, 256, 0, (cudaStream_t)stream>>>(
          (const T*)proj, ld, b_ap, b_ag, b_bp, b_bg, mask, (T*)a_cm, (T*)b_cm, RR, (int)ch);
    });
    EVO_LAUNCH_CHECK();
    count_launch(1);
    return EVO_OK;
  }
  dim3 grid(cdiv(RR, TT), cdiv(ch, TT));
  EVO_DISPATCH_T(dtype, T, {
    trimul_gate_fwd_kernel<T><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const T*)proj, ld, b_ap, b_ag, b_bp, b_bg, mask, (T*)a_cm, (T*)b_cm, RR, (int)ch);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_trimul_gate_bwd(const void* proj, int64_t ld, const float* b_ap, const float* b_ag,
                        const float* b_bp, const float* b_bg, const float* mask, const void* da_cm,
                        const void* db_cm, void* dproj, int64_t RR, int64_t ch, int dtype,
                        void* stream) {
  EVO_API_BEGIN
  const int64_t es = dtype == EVO_F32 ? 4 : 2;
  if (ch % 32 == 0 && RR % 8 == 0 && (ld * es) % 16 == 0 && al16(proj) && al16(da_cm) && al16(db_cm) &&
      al16(dproj)) {
    dim3 g2(cdiv(RR, 64), (unsigned)(ch / 32));
    EVO_DISPATCH_T(dtype, T, {
      trimul_gate_bwd_vec_kernel<T><<<g2, 256, 0, (cudaStream_t)stream>>>(
          (const T*)proj, ld, b_ap, b_ag, b_bp, b_bg, mask, (const T*)da_cm, (const T*)db_cm, (T*)dproj, RR,
          (int)ch);
    });
    EVO_LAUNCH_CHECK();
    count_launch(1);
    return EVO_OK;
  }
  dim3 grid(cdiv(RR, TT), cdiv(ch, TT));
  EVO_DISPATCH_T(dtype, T, {
    trimul_gate_bwd_kernel<T><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const T*)proj, ld, b_ap, b_ag, b_bp, b_bg, mask, (const T*)da_cm, (const T*)db_cm, (T*)dproj,
        RR, (int)ch);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_transpose2d(const void* x, int x_dtype, void* y, int y_dtype, int64_t rows, int64_t cols,
                    void* stream) {
  EVO_API_BEGIN
  if (y_dtype == EVO_BF16 && rows % 64 == 0 && cols % 64 == 0 && rows / 64 <= 65535 && al16(x) && al16(y)) {
    dim3 g64((unsigned)(cols / 64), (unsigned)(rows / 64));
    if (x_dtype == EVO_BF16)
      transpose_vec_kernel<__nv_bfloat16><<<g64, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)x,
                                                                                 (__nv_bfloat16*)y, rows, cols);
    else
      transpose_vec_kernel<float><<<g64, 256, 0, (cudaStream_t)stream>>>((const float*)x, (__nv_bfloat16*)y, rows,
                                                                         cols);
    EVO_LAUNCH_CHECK();
    count_launch(1);
    return EVO_OK;
  }
  dim3 grid(cdiv(cols, TT), cdiv(rows, TT));
  EVO_DISPATCH_T(x_dtype, TI, EVO_DISPATCH_T(y_dtype, TO, {
    transpose_kernel<TI, TO><<<grid, 256, 0, (cudaStream_t)stream>>>((const TI*)x, (TO*)y, rows, cols);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_gated_residual(const void* res, const void* gp, int64_t ld_gp, const float* bg, const void* y,
                       const float* by, void* g_out, void* out, int64_t rows, int64_t C, int dtype,
                       void* stream) {
  EVO_API_BEGIN
  const int64_t n = rows * C;
  const int64_t es = dtype == EVO_F32 ? 4 : 2;
  if (C % 8 == 0 && (ld_gp * es) % 16 == 0 && al16(res) && al16(gp) && al16(y) && al16(g_out) && al16(out)) {
    const unsigned g8 = (unsigned)imin64((n / 8 + 255) / 256, (int64_t)num_sms() * 16);
    EVO_DISPATCH_T(dtype, T, {
      gated_residual_vec_kernel<T><<<g8, 256, 0, (cudaStream_t)stream>>>(
          (const T*)res, (const T*)gp, ld_gp, bg, (const T*)y, by, (T*)g_out, (T*)out, rows, C);
    });
    EVO_LAUNCH_CHECK();
    count_launch(1);
    return EVO_OK;
  }
  const unsigned grid = (unsigned)imin64((n + 255) / 256, (int64_t)num_sms() * 16);
  EVO_DISPATCH_T(dtype, T, {
    gated_residual_kernel<T><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const T*)res, (const T*)gp, ld_gp, bg, (const T*)y, by, (T*)g_out, (T*)out, rows, C);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_gated_residual_bwd(const float* dout, const void* g, const void* y, const float* by, void* dyb,
                           void* dgp, int64_t rows, int64_t C, int dtype, void* stream) {
  EVO_API_BEGIN
  const int64_t n = rows * C;
  if (C % 8 == 0 && al16(dout) && al16(g) && al16(y) && al16(dyb) && al16(dgp)) {
    const unsigned g8 = (unsigned)imin64((n / 8 + 255) / 256, (int64_t)num_sms() * 16);
    EVO_DISPATCH_T(dtype, T, {
      gated_residual_bwd_vec_kernel<T><<<g8, 256, 0, (cudaStream_t)stream>>>(
          dout, (const T*)g, (const T*)y, by, (T*)dyb, (T*)dgp, rows, C);
    });
    EVO_LAUNCH_CHECK();
    count_launch(1);
    return EVO_OK;
  }
  const unsigned grid = (unsigned)imin64((n + 255) / 256, (int64_t)num_sms() * 16);
  EVO_DISPATCH_T(dtype, T, {
    gated_residual_bwd_kernel<T><<<grid, 256, 0, (cudaStream_t)stream>>>(
        dout, (const T*)g, (const T*)y, by, (T*)dyb, (T*)dgp, rows, C);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

}  // extern "C"
