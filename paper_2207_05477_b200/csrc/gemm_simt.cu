// CUDA-core GEMM for the fp32 parity mode (and any operand TMA cannot
// address): true fp32 FFMA accumulation, because tcgen05's kind::tf32 keeps a
// 10-bit mantissa, too coarse for the rtol 1e-4 parity target (SURVEY.md
// section 0.5).  Same contract as the tensor-core GEMM (gemm_tc.cu):
//
//   D[b] = act(alpha * op(A[b]) op(B[b]) + bias) + beta * C[b]      (row-major)
//
// 64 x 64 output tile per 256-thread block, 4 x 4 outputs per thread, K staged
// through shared memory 16 at a time; batch on gridDim.z.
#include "common.cuh"
#include "reduce.cuh"

namespace evo {
namespace {

constexpr int SM_T = 64, SK_T = 16;

template <typename TA>
__device__ __forceinline__ float ldf(const TA* p) {
  return to_f(*p);
}

template <typename TA, typename TD>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int64_t M, int64_t N, int64_t K, const TA* __restrict__ A,
                                                        int64_t lda, int ta, int64_t sa, const TA* __restrict__ B,
                                                        int64_t ldb, int tb, int64_t sb, TD* D, int64_t ldd,
                                                        int64_t sd, float alpha, float beta, const void* Cin,
                                                        int c_f32, int64_t ldc, int64_t sc,
                                                        const float* __restrict__ bias, int relu,
                                                        float* __restrict__ part, int64_t kchunk) {
  __shared__ float As[SK_T][SM_T + 4];
  __shared__ float Bs[SK_T][SM_T + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * SM_T, n0 = (int64_t)blockIdx.x * SM_T;
  // part != nullptr: split-K, blockIdx.z is the split (K range of kchunk), raw
  // sums go to part[z] and splitk_reduce applies the epilogue
  const int64_t z = part ? 0 : blockIdx.z;
  A += z * sa;
  B += z * sb;
  D += z * sd;
  const int64_t kbeg = part ? blockIdx.z * kchunk : 0;
  const int64_t kend = part ? min(K, kbeg + kchunk) : K;
  float acc[4][4] = {};
  for (int64_t k0 = kbeg; k0 < kend; k0 += SK_T) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * 256;
      int m, k;
      if (!ta) {
        m = idx / SK_T;
        k = idx % SK_T;
      } else {
        k = idx / SM_T;
        m = idx % SM_T;
      }
      const int64_t gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gm < M && gk < kend) v = ldf(ta ? A + gk * lda + gm : A + gm * lda + gk);
      As[k][m] = v;
      int n;
      if (!tb) {
        k = idx / SM_T;
        n = idx % SM_T;
      } else {
        n = idx / SK_T;
        k = idx % SK_T;
      }
      const int64_t gn = n0 + n, gk2 = k0 + k;
      float w = 0.f;
      if (gn < N && gk2 < kend) w = ldf(tb ? B + gn * ldb + gk2 : B + gk2 * ldb + gn);
      Bs[k][n] = w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SK_T; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      if (part) {
        part[blockIdx.z * M * N + m * N + n] = acc[i][j];
        continue;
      }
      float v = alpha * acc[i][j];
      if (bias) v += bias[n];
      if (relu) v = fmaxf(v, 0.f);
      if (Cin) {
        const int64_t ci = z * sc + m * ldc + n;
        const float c = c_f32 ? static_cast<const float*>(Cin)[ci] : to_f(static_cast<const __nv_bfloat16*>(Cin)[ci]);
        v = fmaf(beta, c, v);
      }
      D[m * ldd + n] = from_f<TD>(v);
    }
  }
}

template <typename TA, typename TD>
void launch_simt(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
                 int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch, float alpha, float beta,
                 const void* Cin, int c_f32, int64_t ldc, int64_t sc, const float* bias, int relu, float* part,
                 int splits, int64_t kchunk, cudaStream_t s) {
  dim3 grid((unsigned)((N + SM_T - 1) / SM_T), (unsigned)((M + SM_T - 1) / SM_T),
            (unsigned)(part ? splits : batch));
  gemm_simt_kernel<TA, TD><<<grid, 256, 0, s>>>(M, N, K, (const TA*)A, lda, ta, sa, (const TA*)B, ldb, tb, sb,
                                                 (TD*)D, ldd, sd, alpha, beta, Cin, c_f32, ldc, sc, bias, relu, part,
                                                 kchunk);
  EVO_LAUNCH_CHECK();
  count_launch(1);
}

}  // namespace

float* gemm_split_ws(cudaStream_t s, size_t* bytes);  // gemm_tc.cu
void splitk_reduce(const float* ws, int splits, int64_t M, int64_t N, void* D, int64_t ldd, const void* Cin,
                   int64_t ldc, float alpha, float beta, const float* bias, int relu, int d_dtype, cudaStream_t s);

void gemm_simt(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
               int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch, float alpha, float beta,
               const void* Cin, int c_dtype, int64_t ldc, int64_t sc, const float* bias, int relu, int ab_dtype,
               int d_dtype, cudaStream_t s) {
  EVO_REQUIRE((M + SM_T - 1) / SM_T <= 65535 && (N + SM_T - 1) / SM_T < (1ll << 31) && batch <= 65535,
              EVO_ERR_ARG, "gemm: extents out of range for the CUDA-core kernel");
  if (beta == 0.f) Cin = nullptr;
  const int c32 = c_dtype == EVO_F32;
  // few output tiles and a long K (the embedding's weight gradients: K =
  // tokens): split K over blockIdx.z into the split-K workspace
  float* part = nullptr;
  int splits = 1;
  int64_t kchunk = K;
  const int64_t tiles = ((M + SM_T - 1) / SM_T) * ((N + SM_T - 1) / SM_T);
  const int nsm = num_sms();
  if (batch == 1 && tiles < 2 * nsm && K >= 2048 && N % 4 == 0 && (Cin == nullptr || c_dtype == d_dtype)) {
    size_t bytes = 0;
    float* ws = gemm_split_ws(s, &bytes);
    splits = (int)((2 * nsm + tiles - 1) / tiles);
    if (splits > K / 512) splits = (int)(K / 512);
    if (splits > 256) splits = 256;
    while (splits > 1 && (size_t)splits * M * N * 4 > bytes) --splits;
    if (ws && splits > 1) {
      kchunk = ((K + splits - 1) / splits + SK_T - 1) / SK_T * SK_T;
      splits = (int)((K + kchunk - 1) / kchunk);
      part = ws;
    }
  }
  using bf = __nv_bfloat16;
  if (ab_dtype == EVO_F32) {
    if (d_dtype == EVO_F32)
      launch_simt<float, float>(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, c32,
                                ldc, sc, bias, relu, part, splits, kchunk, s);
    else
      launch_simt<float, bf>(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, c32, ldc,
                             sc, bias, relu, part, splits, kchunk, s);
  } else {
    if (d_dtype == EVO_F32)
      launch_simt<bf, float>(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, c32, ldc,
                             sc, bias, relu, part, splits, kchunk, s);
    else
      launch_simt<bf, bf>(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, c32, ldc, sc,
                          bias, relu, part, splits, kchunk, s);
  }
  if (part) splitk_reduce(part, splits, M, N, D, ldd, Cin, ldc, alpha, beta, bias, relu, d_dtype, s);
}

}  // namespace evo
