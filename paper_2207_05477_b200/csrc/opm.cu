// Outer-product-mean glue (src/model.py:351-378) and the squared-mean loss
// (src/harness.py:313-320).  The two contractions of the OPM
// (num = a^T c over the sequence axis, out = outn . W_out) run through
// evo_gemm; these kernels are the bandwidth-bound pieces around them:
//   proj      a = (LN(m).Wl + bl)*mask,  c = (LN(m).Wr + br)*mask
//   norm_fwd  outn[i,j,p*k+q] = num[i*k+p, j*k+q] / (sum_s m_si m_sj + 1e-3)
//   norm_bwd  the inverse re-layout of the gradient
#include "common.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace evo {

template <typename T>
__global__ void opm_proj_kernel(const T* __restrict__ ab, const float* __restrict__ bl,
                                const float* __restrict__ br, const float* __restrict__ mask,
                                T* __restrict__ a, T* __restrict__ c, int64_t SR, int k) {
  const int64_t n = SR * 2 * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / (2 * k);
    const int col = (int)(e % (2 * k));
    const float m = mask[t];
    if (col < k)
      a[t * k + col] = from_f<T>((to_f(ab[e]) + bl[col]) * m);
    else
      c[t * k + col - k] = from_f<T>((to_f(ab[e]) + br[col - k]) * m);
  }
}

// d_ab = [da | dc] * mask, with colsum partials over the 2k columns
template <typename T>
__global__ void opm_proj_bwd_kernel(const T* __restrict__ da, const T* __restrict__ dc,
                                    const float* __restrict__ mask, T* __restrict__ dab,
                                    float* __restrict__ partials, int64_t SR, int k) {
  const int C = 2 * k;
  for (int col = threadIdx.x; col < C; col += blockDim.x) {
    float acc = 0.f;
    for (int64_t t = blockIdx.x; t < SR; t += gridDim.x) {
      float v = col < k ? to_f(da[t * k + col]) : to_f(dc[t * k + col - k]);
      v = v * mask[t];
      dab[t * C + col] = from_f<T>(v);
      acc += v;
    }
    partials[blockIdx.x * C + col] = acc;
  }
}

// Vectorised d_ab = [da | dc] * mask: 8 channels (16 B bf16) per thread, a
// block covers 256 / (2k/8) rows per step, column partials reduced in smem.
template <typename T>
__global__ void __launch_bounds__(256) opm_proj_bwd_vec_kernel(const T* __restrict__ da, const T* __restrict__ dc,
                                                               const float* __restrict__ mask, T* __restrict__ dab,
                                                               float* __restrict__ partials, int64_t SR, int k) {
  extern __shared__ float red[];  // [256][8]
  const int G = 2 * k / 8;        // 8-column groups per row
  const int rows_per = 256 / G;
  const int cg = threadIdx.x % G, rl = threadIdx.x / G;
  const bool act = rl < rows_per;
  const T* src = cg < k / 8 ? da : dc;
  const int sc = (cg < k / 8 ? cg : cg - k / 8) * 8;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (act) {
    for (int64_t t = (int64_t)blockIdx.x * rows_per + rl; t < SR; t += (int64_t)gridDim.x * rows_per) {
      float v[8];
      ld8(src + t * k + sc, v);
      const float m = mask[t];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[e] *= m;
        acc[e] += v[e];
      }
      st8(dab + t * 2 * k + cg * 8, v);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.x * 8 + e] = act ? acc[e] : 0.f;
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * k; c += blockDim.x) {
    const int g = c / 8, e = c % 8;
    float s = 0.f;
    for (int r = 0; r < rows_per; ++r) s += red[(r * G + g) * 8 + e];
    partials[(int64_t)blockIdx.x * 2 * k + c] = s;
  }
}

__global__ void opm_rec_kernel(const float* __restrict__ mask, float* __restrict__ rec, int64_t S,
                               int64_t R, int64_t i0, int64_t NI) {
  const int64_t n = NI * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + e / R, j = e % R;
    float acc = 0.f;
    for (int64_t s = 0; s < S; ++s) acc += mask[s * R + i] * mask[s * R + j];
    rec[e] = 1.0f / (acc + 1e-3f);
  }
}

// one block per (i, j) pair row of outn; thread e = p*k + q
template <typename TI, typename TO>
__global__ void opm_norm_fwd_kernel(const TI* __restrict__ num, const float* __restrict__ rec,
                                    TO* __restrict__ outn, int64_t R, int k) {
  const int64_t ij = blockIdx.x;
  const int64_t i = ij / R, j = ij % R;
  const int64_t Rk = R * k;
  const float r = rec[ij];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int p = e / k, q = e % k;
    outn[ij * k * k + e] = from_f<TO>(to_f(num[(i * k + p) * Rk + j * k + q]) * r);
  }
}

template <typename TI, typename TO>
__global__ void opm_norm_bwd_kernel(const TI* __restrict__ doutn, const float* __restrict__ rec,
                                    TO* __restrict__ dnum, int64_t R, int k) {
  const int64_t ij = blockIdx.x;
  const int64_t i = ij / R, j = ij % R;
  const int64_t Rk = R * k;
  const float r = rec[ij];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int p = e / k, q = e % k;
    dnum[(i * k + p) * Rk + j * k + q] = from_f<TO>(to_f(doutn[ij * k * k + e]) * r);
  }
}

// loss partials: block b sums x^2 over its grid-stride slice; also writes 2*k*x
template <typename T>
__global__ void sq_loss_kernel(const T* __restrict__ x, int64_t n, float k2,
                               float* __restrict__ dx, float* __restrict__ partials) {
  __shared__ float red[32];
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = to_f(x[i]);
    acc += v * v;
    dx[i] = k2 * v;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
  }
}

__global__ void sq_loss_final_kernel(const float* __restrict__ pm, const float* __restrict__ pz,
                                     int G, float km, float kz, float* __restrict__ loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double sm = 0.0, sz = 0.0;
  for (int g = 0; g < G; ++g) {
    sm += pm[g];
    sz += pz[g];
  }
  float lm = (float)sm * km, lz = (float)sz * kz;
  *loss = lm + lz;
}

bool opm_norm_vec(bool fwd, const void* src, int sdt, const float* mask, float* rec, void* dst, int ddt,
                  int64_t S, int64_t R, int64_t k, int64_t i0, int64_t NI, cudaStream_t s);
void opm_rec_rows(const float* mask, float* rec, int64_t S, int64_t R, int64_t i0, int64_t NI, cudaStream_t s);

}  // namespace evo

using namespace evo;

extern "C" {

int evo_opm_proj(const void* ab, const float* bl, const float* br, const float* mask, void* a,
                 void* c, int64_t SR, int64_t k, int dtype, void* stream) {
  EVO_API_BEGIN
  const int64_t n = SR * 2 * k;
  if (n == 0) return EVO_OK;
  unsigned g = (unsigned)imin64((n + 255) / 256, (int64_t)num_sms() * 16);
  EVO_DISPATCH_T(dtype, T, {
    opm_proj_kernel<T><<<g, 256, 0, (cudaStream_t)stream>>>((const T*)ab, bl, br, mask, (T*)a,
                                                            (T*)c, SR, (int)k);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_opm_proj_bwd(const void* da, const void* dc, const float* mask, void* d_ab, float* dbl,
                     float* dbr, int accumulate, void* ws, int64_t SR, int64_t k, int dtype,
                     void* stream) {
  EVO_API_BEGIN
  cudaStream_t s = (cudaStream_t)stream;
  unsigned g = partial_grid(SR);
  ws = partial_buffer(ws, (size_t)g * 2 * k * 4);
  int bs = (int)((2 * k + 31) / 32 * 32);
  if (bs > 256) bs = 256;
  const bool vec = (k % 8) == 0 && 2 * k <= 256 && (((uintptr_t)da | (uintptr_t)dc | (uintptr_t)d_ab) & 15) == 0;
  EVO_DISPATCH_T(dtype, T, {
    if (vec)
      opm_proj_bwd_vec_kernel<T><<<g, 256, 256 * 8 * sizeof(float), s>>>((const T*)da, (const T*)dc, mask,
                                                                          (T*)d_ab, (float*)ws, SR, (int)k);
    else
      opm_proj_bwd_kernel<T><<<g, bs, 0, s>>>((const T*)da, (const T*)dc, mask, (T*)d_ab,
                                              (float*)ws, SR, (int)k);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  finalize_partials((const float*)ws, g, k, dbl, accumulate, s, 2 * k);
  finalize_partials((const float*)ws + k, g, k, dbr, accumulate, s, 2 * k);
  EVO_API_END
}

int evo_opm_norm_fwd_rows(const void* num, int num_dtype, const float* mask, float* rec, void* outn,
                          int out_dtype, int64_t S, int64_t R, int64_t k, int64_t i0, int64_t NI,
                          void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(i0 >= 0 && NI >= 0 && i0 + NI <= R, EVO_ERR_ARG, "opm_norm: row range outside [0, R)");
  if (NI * R == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (opm_norm_vec(true, num, num_dtype, mask, rec, outn, out_dtype, S, R, k, i0, NI, s)) return EVO_OK;
  opm_rec_kernel<<<cdiv(NI * R, 256), 256, 0, s>>>(mask, rec, S, R, i0, NI);
  EVO_LAUNCH_CHECK();
  int bs = (int)(k * k < 256 ? ((k * k + 31) / 32) * 32 : 256);
  EVO_DISPATCH_T(num_dtype, TI, EVO_DISPATCH_T(out_dtype, TO, {
    opm_norm_fwd_kernel<TI, TO><<<(unsigned)(NI * R), bs, 0, s>>>((const TI*)num, rec, (TO*)outn, R, (int)k);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(2);
  EVO_API_END
}

int evo_opm_rec(const float* mask, float* rec, int64_t S, int64_t R, int64_t i0, int64_t NI, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(i0 >= 0 && NI >= 0 && i0 + NI <= R && S * 4 <= 48 * 1024, EVO_ERR_ARG,
              "opm_rec: row range outside [0, R) or S too large");
  opm_rec_rows(mask, rec, S, R, i0, NI, (cudaStream_t)stream);
  EVO_API_END
}

int evo_opm_norm_apply_rows(const void* num, int num_dtype, const float* rec, void* outn, int out_dtype,
                            int64_t R, int64_t k, int64_t NI, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(NI >= 0 && NI <= R, EVO_ERR_ARG, "opm_norm: row count outside [0, R]");
  if (NI * R == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (opm_norm_vec(true, num, num_dtype, nullptr, const_cast<float*>(rec), outn, out_dtype, 0, R, k, 0, NI, s))
    return EVO_OK;
  int bs = (int)(k * k < 256 ? ((k * k + 31) / 32) * 32 : 256);
  EVO_DISPATCH_T(num_dtype, TI, EVO_DISPATCH_T(out_dtype, TO, {
    opm_norm_fwd_kernel<TI, TO><<<(unsigned)(NI * R), bs, 0, s>>>((const TI*)num, rec, (TO*)outn, R, (int)k);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_opm_norm_fwd(const void* num, int num_dtype, const float* mask, float* rec, void* outn,
                     int out_dtype, int64_t S, int64_t R, int64_t k, void* stream) {
  return evo_opm_norm_fwd_rows(num, num_dtype, mask, rec, outn, out_dtype, S, R, k, 0, R, stream);
}

int evo_opm_norm_bwd_rows(const void* doutn, int in_dtype, const float* rec, void* dnum, int out_dtype,
                          int64_t R, int64_t k, int64_t NI, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(NI >= 0 && NI <= R, EVO_ERR_ARG, "opm_norm: row count outside [0, R]");
  if (NI * R == 0) return EVO_OK;
  if (opm_norm_vec(false, doutn, in_dtype, nullptr, const_cast<float*>(rec), dnum, out_dtype, 0, R, k, 0,
                   NI, (cudaStream_t)stream))
    return EVO_OK;
  int bs = (int)(k * k < 256 ? ((k * k + 31) / 32) * 32 : 256);
  EVO_DISPATCH_T(in_dtype, TI, EVO_DISPATCH_T(out_dtype, TO, {
    opm_norm_bwd_kernel<TI, TO><<<(unsigned)(NI * R), bs, 0, (cudaStream_t)stream>>>(
        (const TI*)doutn, rec, (TO*)dnum, R, (int)k);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_opm_norm_bwd(const void* doutn, int in_dtype, const float* rec, void* dnum, int out_dtype,
                     int64_t R, int64_t k, void* stream) {
  return evo_opm_norm_bwd_rows(doutn, in_dtype, rec, dnum, out_dtype, R, k, R, stream);
}

int64_t evo_sq_loss_workspace(void) { return 2 * EVO_PARTIAL_BLOCKS * 4; }

int evo_sq_loss(const void* msa, int64_t n_m, const void* pair, int64_t n_z, int dtype, float km,
                float kz, float* loss, float* dmsa, float* dpair, void* ws, void* stream) {
  EVO_API_BEGIN
  cudaStream_t s = (cudaStream_t)stream;
  float* pm = (float*)ws;
  float* pz = pm + EVO_PARTIAL_BLOCKS;
  const int G = EVO_PARTIAL_BLOCKS;
  EVO_DISPATCH_T(dtype, T, {
    sq_loss_kernel<T><<<G, 256, 0, s>>>((const T*)msa, n_m, 2.0f * km, dmsa, pm);
    EVO_LAUNCH_CHECK();
    sq_loss_kernel<T><<<G, 256, 0, s>>>((const T*)pair, n_z, 2.0f * kz, dpair, pz);
    EVO_LAUNCH_CHECK();
  });
  sq_loss_final_kernel<<<1, 32, 0, s>>>(pm, pz, G, km, kz, loss);
  EVO_LAUNCH_CHECK();
  count_launch(3);
  EVO_API_END
}

}  // extern "C"
