// Library plumbing, dense projections (GEMM routing: gemm_tc.cu / gemm_simt.cu) and
// elementwise glue.
#include <mutex>
#include <string>

#include "common.cuh"
#include "reduce.cuh"

namespace evo {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches += n; }

DeferState& defer_state() {
  static thread_local DeferState st;
  return st;
}

static __global__ void __launch_bounds__(256) finalize_batch_kernel(const __grid_constant__ FinBatch b) {
  __shared__ float sm[8][33];
  const FinDesc& d = b.d[blockIdx.y];
  if ((int64_t)blockIdx.x * 32 >= d.C) return;  // whole block
  finalize_cols(d.part, d.G, d.C, d.ld, d.out, d.accumulate, blockIdx.x, sm);
}

// ---------------------------------------------------------------------------
// Per-stream scratch (split-K partials, column-sum partials) lives in one of
// EVO_STREAM_SLOTS slots.  A stream keeps its slot while it is in use; when a
// new stream arrives and every slot is taken, the least recently used slot is
// handed over -- its previous stream has gone quiet (old trainers / finished
// tests), whereas hashing could give two live, concurrently running streams
// (a capture stream and a branch stream) the same scratch.  The workspaces of
// all slots are allocated on the first GEMM, before any CUDA-graph capture.
int stream_slot(cudaStream_t s) {
  static thread_local cudaStream_t seen[EVO_STREAM_SLOTS] = {};
  static thread_local uint64_t used[EVO_STREAM_SLOTS] = {};
  static thread_local uint64_t tick = 0;
  static thread_local int n = 0;
  ++tick;
  for (int i = 0; i < n; ++i)
    if (seen[i] == s) {
      used[i] = tick;
      return i;
    }
  int slot = n;
  if (n < EVO_STREAM_SLOTS) {
    ++n;
  } else {
    slot = 0;
    for (int i = 1; i < EVO_STREAM_SLOTS; ++i)
      if (used[i] < used[slot]) slot = i;
  }
  seen[slot] = s;
  used[slot] = tick;
  return slot;
}

// vectorised glue (glue.cu); return false -> scalar kernels below
int64_t colsum_vec_ws(int64_t C);
bool colsum_vec(void* x, int xdt, int64_t ldx, const void* h, void* y, int ydt, float* out,
                int accumulate, void* ws, int64_t rows, int64_t C, int mode, cudaStream_t s);
bool bias_residual_vec(const void* res, int rdt, const void* y, int ydt, const float* bias, void* out,
                       int odt, int64_t rows, int64_t C, cudaStream_t s);
bool bias_relu_vec(void* y, int dt, const float* bias, int64_t rows, int64_t C, cudaStream_t s);
void pack_cols(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N, int n,
               int sdt, int ddt, int unpack, cudaStream_t s, int ns);

// tcgen05 + TMA GEMM (gemm_tc.cu): false when TMA cannot address an operand.
bool gemm_tc(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
             int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch, float alpha,
             float beta, const void* Cin, int64_t ldc, const float* bias, int relu, int d_dtype, cudaStream_t s);
// CUDA-core GEMM (gemm_simt.cu): the fp32 parity path and odd layouts.
void gemm_simt(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
               int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch, float alpha, float beta,
               const void* Cin, int c_dtype, int64_t ldc, int64_t sc, const float* bias, int relu, int ab_dtype,
               int d_dtype, cudaStream_t s);

// One GEMM with an optional fused epilogue, routed to the tensor cores when the
// operands are bf16 and TMA-addressable, else to the CUDA-core kernel.
static void gemm_route(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa,
                       const void* B, int64_t ldb, int tb, int64_t sb, void* D, int64_t ldd, int64_t sd, int batch,
                       float alpha, float beta, const void* Cin, int c_dtype, int64_t ldc, int64_t sc,
                       const float* bias, int relu, int ab_dtype, int d_dtype, cudaStream_t s) {
  const bool res_ok = Cin == nullptr || beta == 0.f || (c_dtype == d_dtype && (batch == 1 || sc == sd));
  if (ab_dtype == EVO_BF16 && res_ok &&
      gemm_tc(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, ldc, bias, relu, d_dtype,
              s))
    return;
  gemm_simt(M, N, K, A, lda, ta, sa, B, ldb, tb, sb, D, ldd, sd, batch, alpha, beta, Cin, c_dtype, ldc, sc, bias,
            relu, ab_dtype, d_dtype, s);
}
bool gemm_tc_relu_mask(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, const void* B,
                       int64_t ldb, int tb, const void* h, void* D, int d_dtype, cudaStream_t s, float* colsum,
                       int accumulate, void* ws);  // gemm_tc.cu
int64_t gemm_tc_relu_mask_ws(int64_t M, int64_t N);
bool gemm_tc_try(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa,
                 const void* B, int64_t ldb, int tb, int64_t sb, void* C, int64_t ldc, int64_t sc,
                 int batch, float alpha, float beta, int ab, int cd, cudaStream_t s);

// ---------------------------------------------------------------------------
// elementwise kernels

template <typename TR, typename TY, typename TO>
__global__ void bias_residual_kernel(const TR* __restrict__ res, const TY* __restrict__ y,
                                     const float* __restrict__ bias, TO* __restrict__ out,
                                     int64_t n, int64_t C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = to_f(y[i]);
    if (bias) v = v + bias[i % C];
    float r = res ? to_f(res[i]) : 0.f;
    out[i] = from_f<TO>(res ? r + v : v);
  }
}

template <typename T>
__global__ void bias_relu_kernel(T* __restrict__ y, const float* __restrict__ bias, int64_t n, int64_t C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = to_f(y[i]) + (bias ? bias[i % C] : 0.f);
    y[i] = from_f<T>(fmaxf(v, 0.f));
  }
}

template <typename TX, typename TY>
__global__ void cast_kernel(const TX* __restrict__ x, TY* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = from_f<TY>(to_f(x[i]));
}

__global__ void scale_kernel(float* y, float s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] *= s;
}

// colsum partials with optional cast-copy: block b handles rows b, b+G, ...
template <typename TX, typename TY>
__global__ void colsum_cast_kernel(const TX* __restrict__ x, TY* __restrict__ y,
                                   float* __restrict__ partials, int64_t rows, int64_t C) {
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
      float v = to_f(x[r * C + c]);
      acc += v;
      if (y) y[r * C + c] = from_f<TY>(v);
    }
    partials[blockIdx.x * C + c] = acc;
  }
}

template <typename T>
__global__ void relu_bwd_colsum_kernel(T* __restrict__ dh, const T* __restrict__ h,
                                       float* __restrict__ partials, int64_t rows, int64_t C) {
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
      int64_t i = r * C + c;
      float v = to_f(h[i]) > 0.f ? to_f(dh[i]) : 0.f;
      dh[i] = from_f<T>(v);
      acc += v;
    }
    partials[blockIdx.x * C + c] = acc;
  }
}

static unsigned ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 16;
  return (unsigned)(g < cap ? (g > 0 ? g : 1) : cap);
}

unsigned partial_grid(int64_t rows) {
  int64_t g = rows < EVO_PARTIAL_BLOCKS ? rows : EVO_PARTIAL_BLOCKS;
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace evo

using namespace evo;

extern "C" {

const char* evo_last_error(void) { return g_last_error.c_str(); }
int evo_version(void) { return 1; }
int64_t evo_launch_count(void) { return g_launches; }

int evo_defer_begin(void* arena, size_t bytes) {
  EVO_API_BEGIN
  DeferState& d = defer_state();
  EVO_REQUIRE(!d.on, EVO_ERR_ARG, "evo_defer_begin: already deferring");
  EVO_REQUIRE(arena != nullptr && bytes > 0, EVO_ERR_ARG, "evo_defer_begin: empty arena");
  d.on = true;
  d.arena = (char*)arena;
  d.cap = bytes;
  d.used = 0;
  d.list.clear();
  EVO_API_END
}

int evo_defer_end(void* stream) {
  EVO_API_BEGIN
  DeferState& d = defer_state();
  EVO_REQUIRE(d.on, EVO_ERR_ARG, "evo_defer_end without evo_defer_begin");
  d.on = false;
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t i0 = 0; i0 < d.list.size(); i0 += FIN_BATCH) {
    FinBatch b{};
    b.n = (int)std::min<size_t>(FIN_BATCH, d.list.size() - i0);
    int maxc = 0;
    for (int k = 0; k < b.n; ++k) {
      b.d[k] = d.list[i0 + k];
      maxc = std::max(maxc, b.d[k].C);
    }
    dim3 grid(cdiv(maxc, 32), (unsigned)b.n);
    finalize_batch_kernel<<<grid, 256, 0, s>>>(b);
    EVO_LAUNCH_CHECK();
    count_launch(1);
  }
  d.list.clear();
  d.used = 0;
  EVO_API_END
}

size_t evo_defer_used(void) { return defer_state().used; }

int evo_pack_cols(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N,
                  int n, int src_dtype, int dst_dtype, int unpack, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(n >= 0 && src && dst && C && N, EVO_ERR_ARG, "pack_cols: bad arguments");
  if (n == 0) return EVO_OK;
  pack_cols(src, dst, C, N, n, src_dtype, dst_dtype, unpack, (cudaStream_t)stream, 4);
  EVO_API_END
}

int evo_pack_cols_ns(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N,
                     int n, int ns, int src_dtype, int dst_dtype, int unpack, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(n >= 0 && src && dst && C && N && (ns == 2 || ns == 4), EVO_ERR_ARG,
              "pack_cols: bad arguments (ns must be 2 or 4)");
  if (n == 0) return EVO_OK;
  pack_cols(src, dst, C, N, n, src_dtype, dst_dtype, unpack, (cudaStream_t)stream, ns);
  EVO_API_END
}

int evo_device_check(int* sm_major, int* sm_minor, int* nsm) {
  EVO_API_BEGIN
  int dev = 0, ma = 0, mi = 0, n = 0;
  EVO_CUDA(cudaGetDevice(&dev));
  EVO_CUDA(cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev));
  EVO_CUDA(cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev));
  EVO_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  if (sm_major) *sm_major = ma;
  if (sm_minor) *sm_minor = mi;
  if (nsm) *nsm = n;
  EVO_REQUIRE(ma == 10 && mi == 0, EVO_ERR_UNSUPPORTED,
              "libevoformer_sm100 is built for sm_100a (B200); device is sm_" +
                  std::to_string(ma) + std::to_string(mi));
  EVO_API_END
}

int evo_gemm(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int trans_a,
             int64_t stride_a, const void* B, int64_t ldb, int trans_b, int64_t stride_b,
             void* C, int64_t ldc, int64_t stride_c, int batch, float alpha, float beta,
             int ab_dtype, int c_dtype, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(M >= 0 && N >= 0 && K >= 0 && batch >= 1, EVO_ERR_ARG, "gemm: bad extents");
  EVO_REQUIRE((ab_dtype == EVO_F32 || ab_dtype == EVO_BF16) && (c_dtype == EVO_F32 || c_dtype == EVO_BF16),
              EVO_ERR_ARG, "gemm: bad dtype code");
  if (M == 0 || N == 0) return EVO_OK;
  gemm_route(M, N, K, A, lda, trans_a, stride_a, B, ldb, trans_b, stride_b, C, ldc, stride_c, batch, alpha, beta,
             beta != 0.f ? C : nullptr, c_dtype, ldc, stride_c, nullptr, 0, ab_dtype, c_dtype, (cudaStream_t)stream);
  EVO_API_END
}

int64_t evo_gemm_relu_mask_workspace(int64_t M, int64_t N) { return gemm_tc_relu_mask_ws(M, N); }

int evo_gemm_relu_mask(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int trans_a, const void* B,
                       int64_t ldb, int trans_b, const void* h, void* D, int dtype, float* colsum, int accumulate,
                       void* ws, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(M >= 0 && N >= 0 && K >= 0, EVO_ERR_ARG, "gemm_relu_mask: bad extents");
  if (M == 0 || N == 0) return EVO_OK;
  EVO_REQUIRE(colsum == nullptr || ws != nullptr, EVO_ERR_ARG, "gemm_relu_mask: column sums need a workspace");
  EVO_REQUIRE(dtype == EVO_BF16 && gemm_tc_relu_mask(M, N, K, A, lda, trans_a, B, ldb, trans_b, h, D, dtype,
                                                    (cudaStream_t)stream, colsum, accumulate, ws),
              EVO_ERR_UNSUPPORTED, "gemm_relu_mask: bf16, TMA-addressable operands only");
  EVO_API_END
}

int evo_gemm_bias(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int trans_a, const void* B,
                  int64_t ldb, int trans_b, const void* res, int res_dtype, const float* bias,
                  const void* bias_bf16, int relu, void* out, int64_t ldo, int ab_dtype, int c_dtype,
                  void* stream) {
  EVO_API_BEGIN
  (void)bias_bf16;  // the fused epilogues add the fp32 bias
  EVO_REQUIRE(M >= 0 && N >= 0 && K >= 0, EVO_ERR_ARG, "gemm_bias: bad extents");
  EVO_REQUIRE(!(relu && res), EVO_ERR_ARG, "gemm_bias: relu with a residual is not a module of the path");
  EVO_REQUIRE(bias != nullptr, EVO_ERR_ARG, "gemm_bias: null bias");
  if (M == 0 || N == 0) return EVO_OK;
  // residual rows are contiguous [M, N] (ld = N), the output may be strided
  gemm_route(M, N, K, A, lda, trans_a, 0, B, ldb, trans_b, 0, out, ldo, 0, 1, 1.0f, res ? 1.0f : 0.0f, res,
             res_dtype, N, 0, bias, relu, ab_dtype, c_dtype, (cudaStream_t)stream);
  EVO_API_END
}

int evo_bias_residual(const void* res, int res_dtype, const void* y, int y_dtype, const float* bias,
                      void* out, int out_dtype, int64_t rows, int64_t C, void* stream) {
  EVO_API_BEGIN
  int64_t n = rows * C;
  if (n == 0) return EVO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (bias_residual_vec(res, res_dtype, y, y_dtype, bias, out, out_dtype, rows, C, s)) return EVO_OK;
  unsigned g = ew_grid(n);
  EVO_DISPATCH_T(res_dtype, TR, EVO_DISPATCH_T(y_dtype, TY, EVO_DISPATCH_T(out_dtype, TO, {
    bias_residual_kernel<TR, TY, TO><<<g, 256, 0, s>>>((const TR*)res, (const TY*)y, bias, (TO*)out, n, C);
  })));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_bias_relu(void* y, int dtype, const float* bias, int64_t rows, int64_t C, void* stream) {
  EVO_API_BEGIN
  int64_t n = rows * C;
  if (n == 0) return EVO_OK;
  if (bias_relu_vec(y, dtype, bias, rows, C, (cudaStream_t)stream)) return EVO_OK;
  EVO_DISPATCH_T(dtype, T, {
    bias_relu_kernel<T><<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>((T*)y, bias, n, C);
  });
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int64_t evo_colsum_workspace(int64_t C) {
  const int64_t a = (int64_t)EVO_PARTIAL_BLOCKS * C * 4, b = colsum_vec_ws(C);
  return a > b ? a : b;
}

int evo_colsum_cast(const void* x, int x_dtype, float* out, int accumulate, void* y, int y_dtype,
                    void* ws, int64_t rows, int64_t C, void* stream) {
  EVO_API_BEGIN
  cudaStream_t s = (cudaStream_t)stream;
  if (colsum_vec(const_cast<void*>(x), x_dtype, C, nullptr, y, y_dtype, out, accumulate, ws, rows, C,
                 0, s))
    return EVO_OK;
  unsigned g = partial_grid(rows);
  int bs = C >= 256 ? 256 : (int)((C + 31) / 32 * 32);
  EVO_DISPATCH_T(x_dtype, TX, EVO_DISPATCH_T(y_dtype, TY, {
    colsum_cast_kernel<TX, TY><<<g, bs, 0, s>>>((const TX*)x, (TY*)y, (float*)ws, rows, C);
  }));
  EVO_LAUNCH_CHECK();
  finalize_partials((const float*)ws, g, C, out, accumulate, s);
  count_launch(1);
  EVO_API_END
}

int evo_colsum_strided(const void* x, int x_dtype, int64_t ld, float* out, int accumulate, void* ws,
                       int64_t rows, int64_t C, void* stream) {
  EVO_API_BEGIN
  cudaStream_t s = (cudaStream_t)stream;
  if (colsum_vec(const_cast<void*>(x), x_dtype, ld, nullptr, nullptr, x_dtype, out, accumulate, ws, rows, C,
                 0, s))
    return EVO_OK;
  EVO_REQUIRE(ld == C, EVO_ERR_UNSUPPORTED, "colsum_strided: strided rows need 16-B aligned power-of-two widths");
  return evo_colsum_cast(x, x_dtype, out, accumulate, nullptr, x_dtype, ws, rows, C, stream);
  EVO_API_END
}

int evo_relu_bwd_colsum(void* dh, const void* h, int dtype, float* db, int accumulate, void* ws,
                        int64_t rows, int64_t C, void* stream) {
  EVO_API_BEGIN
  cudaStream_t s = (cudaStream_t)stream;
  if (colsum_vec(dh, dtype, C, h, nullptr, dtype, db, accumulate, ws, rows, C, 1, s)) return EVO_OK;
  unsigned g = partial_grid(rows);
  int bs = C >= 256 ? 256 : (int)((C + 31) / 32 * 32);
  EVO_DISPATCH_T(dtype, T, {
    relu_bwd_colsum_kernel<T><<<g, bs, 0, s>>>((T*)dh, (const T*)h, (float*)ws, rows, C);
  });
  EVO_LAUNCH_CHECK();
  finalize_partials((const float*)ws, g, C, db, accumulate, s);
  count_launch(1);
  EVO_API_END
}

int evo_cast(const void* x, int x_dtype, void* y, int y_dtype, int64_t n, void* stream) {
  EVO_API_BEGIN
  if (n == 0) return EVO_OK;
  EVO_DISPATCH_T(x_dtype, TX, EVO_DISPATCH_T(y_dtype, TY, {
    cast_kernel<TX, TY><<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>((const TX*)x, (TY*)y, n);
  }));
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

int evo_scale_inplace(float* y, float s_, int64_t n, void* stream) {
  EVO_API_BEGIN
  if (n == 0) return EVO_OK;
  scale_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(y, s_, n);
  EVO_LAUNCH_CHECK();
  count_launch(1);
  EVO_API_END
}

}  // extern "C"
