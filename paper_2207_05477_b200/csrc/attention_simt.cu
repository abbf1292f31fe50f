// Gated attention core, SIMT fp32-math kernels (src/attention.py:118-233).
//
// This is the FP32_EXACT path used for the fp32 parity configuration
// (tcgen05 kind::tf32 has a 10-bit mantissa, too coarse for rtol 1e-4) and
// for head dims the tensor-core kernel does not cover.  The bf16 hot path
// is attention_tc.cu.
//
// Forward: one thread per query row, keys streamed through shared memory in
// chunks with an online softmax.  Logits are accumulated in the reference
// order ((q.k)*c^-1/2 + (mask-1)*1e9) + nb (src/attention.py:151-156), so a
// fully-masked row comes out uniform exactly as in the reference.
//
// Backward (deterministic, no float atomics):
//   prep : dctx = dgated*gate, d(g) = dgated*ctx*gate*(1-gate), Dvec = rowsum(dctx*ctx)
//   rows : recompute p = exp(s - lse), ds = p*(dctx.v - D); dq; stash p, ds
//   cols : dk = sum_i ds*q, dv = sum_i p*dctx
//   bias : dnb[h] = sum over batches of ds (fixed batch order)
#include "common.cuh"
#include "reduce.cuh"
#include "attn_geom.cuh"

namespace evo {

constexpr int SIMT_QT = 64;  // query rows (threads) per CTA
constexpr int SIMT_KC = 32;  // keys per shared-memory chunk
constexpr float LOG2E = 1.4426950408889634f;
constexpr float MASK_BIAS_L2 = 1.4426950408889634e9f;  // = tc::MASK_BIAS_L2 (tc_common.cuh)


template <typename T, int DM>
__global__ void __launch_bounds__(SIMT_QT) attn_fwd_simt_kernel(
    const T* __restrict__ qkvg, const float* __restrict__ mask, const T* __restrict__ nb,
    const float* __restrict__ bg, T* __restrict__ ctx, T* __restrict__ gate, T* __restrict__ gated,
    float* __restrict__ lse, AttnGeom g, float scale) {
  __shared__ float Ks[SIMT_KC][DM];
  __shared__ float Vs[SIMT_KC][DM];
  __shared__ float Mb[SIMT_KC];
  const int64_t b = blockIdx.z, h = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)SIMT_QT + threadIdx.x;
  const bool active = i < g.L;
  const int64_t HD = g.H * g.D;
  float q[DM], acc[DM];
#pragma unroll
  for (int k = 0; k < DM; ++k) {
    q[k] = (active && k < g.D) ? to_f(qkvg[g.tok(b, i) * g.ld + h * g.D + k]) : 0.f;
    acc[k] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int64_t j0 = 0; j0 < g.L; j0 += SIMT_KC) {
    const int nk = (int)imin64((int64_t)SIMT_KC, g.L - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < SIMT_KC * DM; e += SIMT_QT) {
      int jj = e / DM, k = e % DM;
      float kv = 0.f, vv = 0.f;
      if (jj < nk && k < g.D) {
        const T* row = qkvg + g.tok(b, j0 + jj) * g.ld + h * g.D + k;
        kv = to_f(row[HD]);
        vv = to_f(row[2 * HD]);
      }
      Ks[jj][k] = kv;
      Vs[jj][k] = vv;
    }
    for (int jj = threadIdx.x; jj < SIMT_KC; jj += SIMT_QT)
      Mb[jj] = jj < nk ? (mask[b * g.msb + (j0 + jj) * g.msl] - 1.0f) * (sizeof(T) == 2 ? MASK_BIAS_L2 : 1e9f)
                       : 0.f;
    __syncthreads();
    if (!active) continue;
    float s[SIMT_KC];
    float cmax = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < SIMT_KC; ++jj) {
      if (jj < nk) {
        float d = 0.f;
#pragma unroll
        for (int k = 0; k < DM; ++k) d = fmaf(q[k], Ks[jj][k], d);
        const float nbv = nb ? to_f(nb[(h * g.L + i) * g.L + j0 + jj]) : 0.f;
        float v;
        if constexpr (sizeof(T) == 2) {
          // bf16: the fused order of the tcgen05 kernels, (s c + nb) log2e + mask bias, so
          // a problem's forward and backward form the same logits whichever path runs them
          v = fmaf(fmaf(d, scale, nbv), LOG2E, Mb[jj]);  // Mb already (m - 1) 1e9 log2e
        } else {
          v = __fmul_rn(d, scale);  // fp32 parity path: the reference's order (src/attention.py:151-156)
          v = v + Mb[jj];
          if (nb) v = v + nbv;
          v = __fmul_rn(v, LOG2E);  // softmax in the log2 domain
        }
        s[jj] = v;
        cmax = fmaxf(cmax, v);
      } else {
        s[jj] = -INFINITY;
      }
    }
    const float mn = fmaxf(m, cmax);
    const float alpha = exp2f(m - mn);  // m=-inf on the first chunk -> 0
    l *= alpha;
#pragma unroll
    for (int k = 0; k < DM; ++k) acc[k] *= alpha;
#pragma unroll
    for (int jj = 0; jj < SIMT_KC; ++jj) {
      if (jj < nk) {
        float p = exp2f(s[jj] - mn);
        l += p;
#pragma unroll
        for (int k = 0; k < DM; ++k) acc[k] = fmaf(p, Vs[jj][k], acc[k]);
      }
    }
    m = mn;
  }
  if (!active) return;
  const float invl = 1.0f / l;
  const int64_t t = g.tok(b, i);
#pragma unroll
  for (int k = 0; k < DM; ++k) {
    if (k < g.D) {
      const int64_t c = h * g.D + k;
      float cv = acc[k] * invl;
      float gp = to_f(qkvg[t * g.ld + 3 * HD + c]) + bg[c];
      float gv = 1.0f / (1.0f + expf(-gp));
      ctx[t * HD + c] = from_f<T>(cv);
      gate[t * HD + c] = from_f<T>(gv);
      gated[t * HD + c] = from_f<T>(cv * gv);
    }
  }
  // (row max, 1/sum) instead of one log-sum-exp: at a fully-masked row the
  // logits sit at -1e9 where fp32 cannot resolve m + log(l) (ulp 64).
  lse[2 * ((b * g.H + h) * g.L + i)] = m;
  lse[2 * ((b * g.H + h) * g.L + i) + 1] = invl;
}

// thread per (b, h, l): dctx, d(g pre-activation) and Dvec
template <typename T>
__global__ void attn_bwd_prep_kernel(const T* __restrict__ ctx, const T* __restrict__ gate,
                                     const T* __restrict__ dgated, T* __restrict__ dqkvg,
                                     float* __restrict__ dctx_ws, float* __restrict__ Dvec, AttnGeom g) {
  const int64_t n = g.B * g.H * g.L;
  const int64_t HD = g.H * g.D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e % g.L, h = (e / g.L) % g.H, b = e / (g.L * g.H);
    const int64_t t = g.tok(b, l);
    float dsum = 0.f;
    for (int k = 0; k < g.D; ++k) {
      const int64_t c = t * HD + h * g.D + k;
      float dg = to_f(dgated[c]), gv = to_f(gate[c]), cv = to_f(ctx[c]);
      float dctx = dg * gv;
      float dgp = dg * cv * gv * (1.0f - gv);  // src/attention.py:184-187
      dqkvg[t * g.ld + 3 * HD + h * g.D + k] = from_f<T>(dgp);
      dctx_ws[c] = dctx;
      dsum += dctx * cv;
    }
    Dvec[t * g.H + h] = dsum;
  }
}

// thread per query row: ds, dq; stash p and ds transposed [B,H,Lk,Lq]
template <typename T, int DM>
__global__ void __launch_bounds__(SIMT_QT) attn_bwd_rows_kernel(
    const T* __restrict__ qkvg, const float* __restrict__ mask, const T* __restrict__ nb,
    const float* __restrict__ lse, const float* __restrict__ dctx_ws, const float* __restrict__ Dvec,
    float* __restrict__ Pt, float* __restrict__ dSt, T* __restrict__ dqkvg, AttnGeom g, float scale) {
  __shared__ float Ks[SIMT_KC][DM];
  __shared__ float Vs[SIMT_KC][DM];
  __shared__ float Mb[SIMT_KC];
  const int64_t b = blockIdx.z, h = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)SIMT_QT + threadIdx.x;
  const bool active = i < g.L;
  const int64_t HD = g.H * g.D;
  const int64_t ti = active ? g.tok(b, i) : 0;
  float q[DM], dc[DM], dq[DM];
#pragma unroll
  for (int k = 0; k < DM; ++k) {
    bool ok = active && k < g.D;
    q[k] = ok ? to_f(qkvg[ti * g.ld + h * g.D + k]) : 0.f;
    dc[k] = ok ? dctx_ws[ti * HD + h * g.D + k] : 0.f;
    dq[k] = 0.f;
  }
  const int64_t bh = b * g.H + h;
  const float ls = active ? lse[2 * (bh * g.L + i)] : 0.f;
  const float rl = active ? lse[2 * (bh * g.L + i) + 1] : 0.f;
  const float Dv = active ? Dvec[ti * g.H + h] : 0.f;
  for (int64_t j0 = 0; j0 < g.L; j0 += SIMT_KC) {
    const int nk = (int)imin64((int64_t)SIMT_KC, g.L - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < SIMT_KC * DM; e += SIMT_QT) {
      int jj = e / DM, k = e % DM;
      float kv = 0.f, vv = 0.f;
      if (jj < nk && k < g.D) {
        const T* row = qkvg + g.tok(b, j0 + jj) * g.ld + h * g.D + k;
        kv = to_f(row[HD]);
        vv = to_f(row[2 * HD]);
      }
      Ks[jj][k] = kv;
      Vs[jj][k] = vv;
    }
    for (int jj = threadIdx.x; jj < SIMT_KC; jj += SIMT_QT)
      Mb[jj] = jj < nk ? (mask[b * g.msb + (j0 + jj) * g.msl] - 1.0f) * (sizeof(T) == 2 ? MASK_BIAS_L2 : 1e9f)
                       : 0.f;
    __syncthreads();
    if (!active) continue;
    for (int jj = 0; jj < nk; ++jj) {
      float d = 0.f, dp = 0.f;
#pragma unroll
      for (int k = 0; k < DM; ++k) {
        d = fmaf(q[k], Ks[jj][k], d);
        dp = fmaf(dc[k], Vs[jj][k], dp);
      }
      const float nbv = nb ? to_f(nb[(h * g.L + i) * g.L + j0 + jj]) : 0.f;
      float p;
      if constexpr (sizeof(T) == 2) {
        // fused order (see the forward); x - m is clamped at 0: the saved row max may
        // come from the tcgen05 forward, whose MMA sums the dot products in another order
        const float x = fmaf(fmaf(d, scale, nbv), LOG2E, Mb[jj]);
        p = exp2f(fminf(x - ls, 0.f)) * rl;
      } else {
        float s = __fmul_rn(d, scale);
        s = s + Mb[jj];
        if (nb) s = s + nbv;
        p = exp2f(__fmul_rn(s, LOG2E) - ls) * rl;
      }
      float ds = p * (dp - Dv);
      const int64_t o = (bh * g.L + j0 + jj) * g.L + i;
      Pt[o] = p;
      dSt[o] = ds;
#pragma unroll
      for (int k = 0; k < DM; ++k) dq[k] = fmaf(ds, Ks[jj][k], dq[k]);
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < DM; ++k)
    if (k < g.D) dqkvg[ti * g.ld + h * g.D + k] = from_f<T>(dq[k] * scale);
}

// thread per key column: dk, dv
template <typename T, int DM>
__global__ void __launch_bounds__(SIMT_QT) attn_bwd_cols_kernel(
    const T* __restrict__ qkvg, const float* __restrict__ dctx_ws, const float* __restrict__ Pt,
    const float* __restrict__ dSt, T* __restrict__ dqkvg, AttnGeom g, float scale) {
  __shared__ float Qs[SIMT_KC][DM];
  __shared__ float Cs[SIMT_KC][DM];
  const int64_t b = blockIdx.z, h = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)SIMT_QT + threadIdx.x;
  const bool active = j < g.L;
  const int64_t HD = g.H * g.D;
  const int64_t bh = b * g.H + h;
  float dk[DM], dv[DM];
#pragma unroll
  for (int k = 0; k < DM; ++k) dk[k] = dv[k] = 0.f;
  for (int64_t i0 = 0; i0 < g.L; i0 += SIMT_KC) {
    const int ni = (int)imin64((int64_t)SIMT_KC, g.L - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < SIMT_KC * DM; e += SIMT_QT) {
      int ii = e / DM, k = e % DM;
      float qv = 0.f, cv = 0.f;
      if (ii < ni && k < g.D) {
        int64_t t = g.tok(b, i0 + ii);
        qv = to_f(qkvg[t * g.ld + h * g.D + k]);
        cv = dctx_ws[t * HD + h * g.D + k];
      }
      Qs[ii][k] = qv;
      Cs[ii][k] = cv;
    }
    __syncthreads();
    if (!active) continue;
    const float* prow = Pt + (bh * g.L + j) * g.L + i0;
    const float* drow = dSt + (bh * g.L + j) * g.L + i0;
    for (int ii = 0; ii < ni; ++ii) {
      float p = prow[ii], ds = drow[ii];
#pragma unroll
      for (int k = 0; k < DM; ++k) {
        dk[k] = fmaf(ds, Qs[ii][k], dk[k]);
        dv[k] = fmaf(p, Cs[ii][k], dv[k]);
      }
    }
  }
  if (!active) return;
  const int64_t t = g.tok(b, j);
#pragma unroll
  for (int k = 0; k < DM; ++k) {
    if (k < g.D) {
      dqkvg[t * g.ld + HD + h * g.D + k] = from_f<T>(dk[k] * scale);
      dqkvg[t * g.ld + 2 * HD + h * g.D + k] = from_f<T>(dv[k]);
    }
  }
}

// dnb[h, i, j] (+)= sum_b dSt[b, h, j, i]  (fixed batch order)
__global__ void attn_bwd_bias_kernel(const float* __restrict__ dSt, float* __restrict__ dnb,
                                     int64_t B, int64_t H, int64_t L, int accumulate) {
  const int64_t n = H * L * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % L, i = (e / L) % L, h = e / (L * L);
    const int64_t src = (h * L + j) * L + i;
    float acc = 0.f;
    for (int64_t b = 0; b < B; ++b) acc += dSt[b * n + src];
    dnb[e] = accumulate ? dnb[e] + acc : acc;
  }
}

// colsum over a strided column slice (rows of length ld, columns [off, off+C))
template <typename T>
__global__ void colsum_strided_kernel(const T* __restrict__ x, int64_t ld, int64_t off,
                                      float* __restrict__ partials, int64_t rows, int64_t C) {
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) acc += to_f(x[r * ld + off + c]);
    partials[blockIdx.x * C + c] = acc;
  }
}

#define ATTN_DM_DISPATCH(D, DM, ...)                                      \
  do {                                                                    \
    if ((D) <= 8) { constexpr int DM = 8; __VA_ARGS__; }                  \
    else if ((D) <= 16) { constexpr int DM = 16; __VA_ARGS__; }           \
    else if ((D) <= 32) { constexpr int DM = 32; __VA_ARGS__; }           \
    else if ((D) <= 64) { constexpr int DM = 64; __VA_ARGS__; }           \
    else throw Error(EVO_ERR_UNSUPPORTED, "attention: head dim > 64");    \
  } while (0)

// tcgen05 path (attention_tc.cu); returns false when the shape is not covered.
bool attn_fwd_tc_try(const void* qkvg, const float* mask, const void* nb, const float* bg,
                     void* ctx, void* gate, void* gated, float* lse, const AttnGeom& g, int dtype,
                     cudaStream_t s);
bool attn_bwd_tc_try(const void* qkvg, const float* mask, const void* nb, const void* ctx,
                     const void* gate, const void* dgated, const float* lse, void* dqkvg,
                     float* dnb, float* dbg, int accumulate, void* ws, size_t ws_bytes,
                     const AttnGeom& g, int dtype, cudaStream_t s);
int64_t attn_bwd_tc_workspace(const AttnGeom& g, int dtype);
bool attn_fwd_tc_kb_try(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx,
                        void* gate, void* gated, float* lse, const AttnGeom& g, int dtype, cudaStream_t s);
bool attn_fwd_tc2_try(const void* qkvg, const float* mask, const void* nb, const float* bg, void* ctx, void* gate,
                      void* gated, float* lse, const AttnGeom& g, int dtype, cudaStream_t s);

static AttnGeom make_geom(int64_t B, int64_t L, int64_t H, int64_t D, int64_t sb, int64_t sl,
                          int64_t ld, int64_t msb, int64_t msl) {
  EVO_REQUIRE(B > 0 && L > 0 && H > 0 && D > 0, EVO_ERR_ARG, "attention: non-positive extent");
  EVO_REQUIRE(ld >= 4 * H * D, EVO_ERR_ARG, "attention: ld_qkvg < 4*H*D");
  // the (batch, position) -> token-row map must cover rows 0..B*L-1 exactly (row-major
  // [B, L] or its transpose): the kernels' per-token workspaces are indexed by token row
  EVO_REQUIRE((sb == L && sl == 1) || (sb == 1 && sl == B), EVO_ERR_ARG,
              "attention: token strides must map (b, l) onto rows 0..B*L-1 (sb=L,sl=1 or sb=1,sl=B)");
  AttnGeom g{B, L, H, D, sb, sl, ld, msb, msl};
  return g;
}

static int64_t simt_ws_bytes(const AttnGeom& g) {
  int64_t T = g.B * g.L;
  int64_t n = 2 * g.B * g.H * g.L * g.L + T * g.H * g.D + g.B * g.H * g.L;
  int64_t cols = (int64_t)EVO_PARTIAL_BLOCKS * g.H * g.D;
  return (n + cols) * 4 + 256;
}

}  // namespace evo

using namespace evo;

extern "C" {

int evo_attn_fwd(const void* qkvg, int64_t ld_qkvg, const float* mask, int64_t mask_sb,
                 int64_t mask_sl, const void* nb, const float* bg, void* ctx, void* gate,
                 void* gated, float* lse, int64_t B, int64_t L, int64_t H, int64_t D,
                 int64_t tok_sb, int64_t tok_sl, int dtype, void* stream) {
  EVO_API_BEGIN
  AttnGeom g = make_geom(B, L, H, D, tok_sb, tok_sl, ld_qkvg, mask_sb, mask_sl);
  cudaStream_t s = (cudaStream_t)stream;
  if (attn_fwd_tc2_try(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, dtype, s)) return EVO_OK;
  if (attn_fwd_tc_try(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, dtype, s)) return EVO_OK;
  if (attn_fwd_tc_kb_try(qkvg, mask, nb, bg, ctx, gate, gated, lse, g, dtype, s)) return EVO_OK;
  const float scale = (float)(1.0 / sqrt((double)D));
  dim3 grid(cdiv(L, SIMT_QT), (unsigned)H, (unsigned)B);
  ATTN_DM_DISPATCH(D, DM, EVO_DISPATCH_T(dtype, T, {
    attn_fwd_simt_kernel<T, DM><<<grid, SIMT_QT, 0, s>>>((const T*)qkvg, mask, (const T*)nb, bg, (T*)ctx,
                                                         (T*)gate, (T*)gated, lse, g, scale);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int64_t evo_attn_bwd_workspace(int64_t B, int64_t L, int64_t H, int64_t D, int dtype) {
  AttnGeom g{B, L, H, D, 0, 0, 4 * H * D, 0, 0};
  int64_t a = simt_ws_bytes(g);
  int64_t t = attn_bwd_tc_workspace(g, dtype);
  return a > t ? a : t;
}

int evo_attn_bwd(const void* qkvg, int64_t ld_qkvg, const float* mask, int64_t mask_sb,
                 int64_t mask_sl, const void* nb, const void* ctx, const void* gate,
                 const void* dgated, const float* lse, void* dqkvg, float* dnb, float* dbg,
                 int accumulate, void* ws, size_t ws_bytes, int64_t B, int64_t L, int64_t H,
                 int64_t D, int64_t tok_sb, int64_t tok_sl, int dtype, void* stream) {
  EVO_API_BEGIN
  AttnGeom g = make_geom(B, L, H, D, tok_sb, tok_sl, ld_qkvg, mask_sb, mask_sl);
  cudaStream_t s = (cudaStream_t)stream;
  if (attn_bwd_tc_try(qkvg, mask, nb, ctx, gate, dgated, lse, dqkvg, dnb, dbg, accumulate,
                      ws, ws_bytes, g, dtype, s))
    return EVO_OK;
  EVO_REQUIRE((int64_t)ws_bytes >= simt_ws_bytes(g), EVO_ERR_ARG, "attn_bwd: workspace too small");
  const float scale = (float)(1.0 / sqrt((double)D));
  float* f = (float*)ws;
  const int64_t nP = B * H * L * L;
  float* Pt = f;
  float* dSt = Pt + nP;
  float* dctx_ws = dSt + nP;
  float* Dvec = dctx_ws + B * L * H * D;
  float* partials = Dvec + B * H * L;
  dim3 grid(cdiv(L, SIMT_QT), (unsigned)H, (unsigned)B);
  const int64_t nbhl = B * H * L;
  EVO_DISPATCH_T(dtype, T, {
    attn_bwd_prep_kernel<T><<<cdiv(nbhl, 256), 256, 0, s>>>(
        (const T*)ctx, (const T*)gate, (const T*)dgated, (T*)dqkvg, dctx_ws, Dvec, g);
    EVO_LAUNCH_CHECK();
    ATTN_DM_DISPATCH(D, DM, {
      attn_bwd_rows_kernel<T, DM><<<grid, SIMT_QT, 0, s>>>((const T*)qkvg, mask, (const T*)nb, lse,
                                                           dctx_ws, Dvec, Pt, dSt, (T*)dqkvg, g, scale);
      EVO_LAUNCH_CHECK();
      attn_bwd_cols_kernel<T, DM><<<grid, SIMT_QT, 0, s>>>((const T*)qkvg, dctx_ws, Pt, dSt,
                                                           (T*)dqkvg, g, scale);
      EVO_LAUNCH_CHECK();
    });
    // dbg = colsum of the d(g) slot
    unsigned pg = partial_grid(B * L);
    colsum_strided_kernel<T><<<pg, 256, 0, s>>>((const T*)dqkvg, g.ld, 3 * H * D, partials, B * L, H * D);
    EVO_LAUNCH_CHECK();
    finalize_partials(partials, pg, H * D, dbg, accumulate, s);
  });
  if (dnb) {
    attn_bwd_bias_kernel<<<cdiv(H * L * L, 256), 256, 0, s>>>(dSt, dnb, B, H, L, accumulate);
    EVO_LAUNCH_CHECK();
  }
  count_launch(5);
  EVO_API_END
}

}  // extern "C"
