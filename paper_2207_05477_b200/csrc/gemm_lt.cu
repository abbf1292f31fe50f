// Dense projections through cuBLASLt with per-shape algorithm autotuning.
//
// cublasGemmEx's default heuristic picks split-K / small-tile kernels for the
// Evoformer's tall-skinny projections (M = 32768..65536 tokens, N, K = 128..1024)
// that run 3-5x below the HBM bound.  Here every distinct problem (extents,
// leading dimensions, transposes, batch strides, dtypes, epilogue) asks the
// Lt heuristic for its candidates once, times each on the caller's operands
// (into a scratch D, so C is never modified), and caches the fastest.  Inside
// CUDA-graph capture an uncached problem uses the heuristic's first choice
// without timing (capture forbids the synchronising benchmark).
//
// Epilogues fold the glue that used to follow the projections:
//   EPI_BIAS        D = op(A) op(B) + bias[col]            (+ beta * C)
//   EPI_RELU_BIAS   D = relu(op(A) op(B) + bias[col])
// and C may differ from D (D = AB + bias + C: the residual add of a module).
#include <cublasLt.h>
#include <cstdio>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace evo {

namespace {

struct LtState {
  cublasLtHandle_t h = nullptr;
  __nv_bfloat16* bias16 = nullptr;  // bf16 copy of an epilogue bias (Lt wants Dtype biases)
  int64_t bias16_n = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

LtState& lt_state(cudaStream_t stream) {
  static thread_local LtState st[16][EVO_STREAM_SLOTS];
  int dev = 0;
  EVO_CUDA(cudaGetDevice(&dev));
  if (!st[dev & 15][0].h) {
    // every slot at once: a stream first seen inside CUDA-graph capture (the
    // capture stream) must not allocate
    for (int k = 0; k < EVO_STREAM_SLOTS; ++k) {
      LtState& s = st[dev & 15][k];
      if (cublasLtCreate(&s.h) != CUBLAS_STATUS_SUCCESS) throw Error(EVO_ERR_CUDA, "cublasLtCreate failed");
      s.ws_bytes = size_t(32) << 20;
      EVO_CUDA(cudaMalloc(&s.ws, s.ws_bytes));
      s.bias16_n = 1 << 16;
      EVO_CUDA(cudaMalloc(&s.bias16, s.bias16_n * sizeof(__nv_bfloat16)));
    }
  }
  return st[dev & 15][stream_slot(stream)];
}

__global__ void bias_to_bf16_kernel(const float* __restrict__ b, __nv_bfloat16* __restrict__ o, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __float2bfloat16_rn(b[i]);
}

cudaDataType_t lt_dt(int d) { return d == EVO_F32 ? CUDA_R_32F : CUDA_R_16BF; }

using Key = std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int64_t,
                       int64_t, int64_t, int, int, int, int, int, int>;

struct Choice {
  cublasLtMatmulAlgo_t algo;
  bool tuned;
};

std::map<Key, Choice>& cache() {
  static thread_local std::map<Key, Choice> c;
  return c;
}

bool env_off() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_GEMM_LT");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

// EVO_GEMM_TUNE=0: take cuBLASLt's top heuristic choice without timing, so the
// algorithm per shape (and every result bit) is the same in every process
bool tune_off() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_GEMM_TUNE");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

struct Descs {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr, d = nullptr;
  ~Descs() {
    if (op) cublasLtMatmulDescDestroy(op);
    if (a) cublasLtMatrixLayoutDestroy(a);
    if (b) cublasLtMatrixLayoutDestroy(b);
    if (c) cublasLtMatrixLayoutDestroy(c);
    if (d) cublasLtMatrixLayoutDestroy(d);
  }
};

}  // namespace

enum { EPI_NONE = 0, EPI_BIAS = 1, EPI_RELU_BIAS = 2, EPI_RELU_AUX_BIAS = 3, EPI_DRELU = 4, EPI_BGRADA = 5,
       EPI_BGRADB = 6 };

namespace {

#define LT_OK(x)                                   \
  do {                                             \
    if ((x) != CUBLAS_STATUS_SUCCESS) return false; \
  } while (0)

}  // namespace

// Row-major D[M,N] = alpha * op(A) op(B) (+ bias[n]) (relu) + beta * C.
// Returns false (caller falls back) when Lt rejects the problem.
bool gemm_lt(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, int64_t sa, const void* B,
             int64_t ldb, int tb, int64_t sb, const void* Cin, void* D, int64_t ldc, int64_t sc, int batch,
             float alpha, float beta, int ab_dtype, int c_dtype, int epi, const float* bias, cudaStream_t s,
             void* aux, int64_t aux_ld, const void* bias16) {
  if (env_off()) return false;
  // small problems are launch-bound: keep them on the default cuBLAS path
  // (no timing-dependent algorithm choice where it cannot pay)
  // (fused epilogues included: Lt wants a bf16 bias for bf16 outputs, a rounding
  // that is only worth paying where the fused kernel saves a pass over HBM)
  if ((double)M * N * K * batch < (double)(1 << 28)) return false;
  LtState& st = lt_state(s);
  // column-major view: D^T[N, M] = op(B)^T op(A)^T  ->  Lt A := B, Lt B := A
  const cublasOperation_t opA = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t opB = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
  Descs ds;
  LT_OK(cublasLtMatmulDescCreate(&ds.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof(opA)));
  LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof(opB)));
  cublasLtEpilogue_t e = CUBLASLT_EPILOGUE_DEFAULT;
  if (epi == EPI_BIAS) e = CUBLASLT_EPILOGUE_BIAS;
  if (epi == EPI_RELU_BIAS) e = CUBLASLT_EPILOGUE_RELU_BIAS;
  if (epi == EPI_RELU_AUX_BIAS) e = CUBLASLT_EPILOGUE_RELU_AUX_BIAS;
  if (epi == EPI_DRELU) e = CUBLASLT_EPILOGUE_DRELU;
  if (epi == EPI_BGRADA) e = CUBLASLT_EPILOGUE_BGRADA;
  if (epi == EPI_BGRADB) e = CUBLASLT_EPILOGUE_BGRADB;
  if (epi == EPI_RELU_AUX_BIAS || epi == EPI_DRELU) {
    if (!aux || (aux_ld % 128) != 0 || aux_ld < N) return false;
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux)));
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &aux_ld, sizeof(aux_ld)));
  }
  if (epi == EPI_DRELU) {
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e)));
  } else if (epi == EPI_BGRADA || epi == EPI_BGRADB) {
    // bias-gradient output has the output's dtype: only fp32 outputs keep fp32 sums
    if (c_dtype != EVO_F32) return false;
    void* gptr = const_cast<float*>(bias);
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e)));
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &gptr, sizeof(gptr)));
  } else if (epi) {
    // the bias must have the output's dtype: bf16 outputs get a bf16 copy
    const void* bptr = bias;
    if (c_dtype == EVO_BF16 && bias16) {
      bptr = bias16;  // the caller's bf16 copy (the parameter store's shadow)
    } else if (c_dtype == EVO_BF16) {
      if (N > st.bias16_n) return false;
      bias_to_bf16_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(bias, st.bias16, N);
      EVO_LAUNCH_CHECK();
      bptr = st.bias16;
    }
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e)));
    LT_OK(cublasLtMatmulDescSetAttribute(ds.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bptr, sizeof(bptr)));
  }
  const cudaDataType_t abt = lt_dt(ab_dtype), ct = lt_dt(c_dtype);
  // Lt A = our B: stored [K x N] row-major (op N) == col-major N x K with ld ldb
  LT_OK(cublasLtMatrixLayoutCreate(&ds.a, abt, tb ? K : N, tb ? N : K, ldb));
  LT_OK(cublasLtMatrixLayoutCreate(&ds.b, abt, ta ? M : K, ta ? K : M, lda));
  LT_OK(cublasLtMatrixLayoutCreate(&ds.c, ct, N, M, ldc));
  LT_OK(cublasLtMatrixLayoutCreate(&ds.d, ct, N, M, ldc));
  if (batch > 1) {
    const int32_t bc = batch;
    for (auto* l : {&ds.a, &ds.b, &ds.c, &ds.d})
      LT_OK(cublasLtMatrixLayoutSetAttribute(*l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)));
    LT_OK(cublasLtMatrixLayoutSetAttribute(ds.a, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof(sb)));
    LT_OK(cublasLtMatrixLayoutSetAttribute(ds.b, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa)));
    LT_OK(cublasLtMatrixLayoutSetAttribute(ds.c, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc)));
    LT_OK(cublasLtMatrixLayoutSetAttribute(ds.d, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc)));
  }
  const Key key{M, N, K, lda, ldb, ldc, batch, ta, tb, sa, sb, sc, ab_dtype, c_dtype, epi, beta != 0.f,
                Cin != D, (int)(((uintptr_t)A | (uintptr_t)B | (uintptr_t)D | (uintptr_t)Cin) & 15)};
  auto& cc = cache();
  auto it = cc.find(key);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  EVO_CUDA(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (it == cc.end() || (!it->second.tuned && !capturing)) {
    cublasLtMatmulPreference_t pref = nullptr;
    LT_OK(cublasLtMatmulPreferenceCreate(&pref));
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &st.ws_bytes,
                                         sizeof(st.ws_bytes));
    cublasLtMatmulHeuristicResult_t res[16];
    int nres = 0;
    const cublasStatus_t hs =
        cublasLtMatmulAlgoGetHeuristic(st.h, ds.op, ds.a, ds.b, ds.c, ds.d, pref, 16, res, &nres);
    cublasLtMatmulPreferenceDestroy(pref);
    if (hs != CUBLAS_STATUS_SUCCESS || nres == 0) {
      if (getenv("EVO_GEMM_DEBUG"))
        fprintf(stderr, "gemm_lt heuristic: M=%lld N=%lld K=%lld epi=%d status=%d nres=%d\n", (long long)M,
                (long long)N, (long long)K, epi, (int)hs, nres);
      return false;
    }
    Choice ch{res[0].algo, false};
    if (!capturing && nres > 1 && !tune_off()) {
      // time every candidate into a scratch D (C untouched)
      const size_t esz = c_dtype == EVO_F32 ? 4 : 2;
      const size_t need = (size_t)((batch - 1) * sc + (M - 1) * ldc + N) * esz + 256;
      if (st.scratch_bytes < need) {
        if (st.scratch) EVO_CUDA(cudaFree(st.scratch));
        EVO_CUDA(cudaMalloc(&st.scratch, need));
        st.scratch_bytes = need;
      }
      const void* cin = beta != 0.f ? Cin : st.scratch;
      cudaEvent_t e0, e1;
      EVO_CUDA(cudaEventCreate(&e0));
      EVO_CUDA(cudaEventCreate(&e1));
      float tms[16];
      for (int r = 0; r < nres; ++r) {
        tms[r] = 1e30f;
        bool ok = true;
        for (int w = 0; w < 2 && ok; ++w)
          ok = cublasLtMatmul(st.h, ds.op, &alpha, B, ds.a, A, ds.b, &beta, cin, ds.c, st.scratch, ds.d,
                              &res[r].algo, st.ws, st.ws_bytes, s) == CUBLAS_STATUS_SUCCESS;
        if (!ok) continue;
        EVO_CUDA(cudaEventRecord(e0, s));
        for (int w = 0; w < 5; ++w)
          cublasLtMatmul(st.h, ds.op, &alpha, B, ds.a, A, ds.b, &beta, cin, ds.c, st.scratch, ds.d, &res[r].algo,
                         st.ws, st.ws_bytes, s);
        EVO_CUDA(cudaEventRecord(e1, s));
        EVO_CUDA(cudaEventSynchronize(e1));
        EVO_CUDA(cudaEventElapsedTime(&tms[r], e0, e1));
      }
      // the first candidate (heuristic order) within EVO_GEMM_TUNE_MARGIN (default
      // 0: the fastest) of the fastest; a margin of a few percent makes near-ties
      // resolve the same way from run to run (the chosen algorithm, and the
      // rounding it implies, then rarely depends on timing noise) at ~1% step time
      float best = 1e30f;
      for (int r = 0; r < nres; ++r) best = fminf(best, tms[r]);
      static const float margin = [] {
        const char* e = getenv("EVO_GEMM_TUNE_MARGIN");
        return e ? (float)atof(e) : 0.0f;
      }();
      for (int r = 0; r < nres; ++r)
        if (tms[r] <= best * (1.0f + margin)) {
          ch.algo = res[r].algo;
          break;
        }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      ch.tuned = true;
    } else if (!capturing) {
      ch.tuned = true;
    }
    it = cc.insert_or_assign(key, ch).first;
  }
  const cublasStatus_t rs = cublasLtMatmul(st.h, ds.op, &alpha, B, ds.a, A, ds.b, &beta, Cin, ds.c, D, ds.d,
                                           &it->second.algo, st.ws, st.ws_bytes, s);
  if (rs != CUBLAS_STATUS_SUCCESS && getenv("EVO_GEMM_DEBUG"))
    fprintf(stderr, "gemm_lt: M=%lld N=%lld K=%lld epi=%d status=%d\n", (long long)M, (long long)N, (long long)K,
            epi, (int)rs);
  return rs == CUBLAS_STATUS_SUCCESS;
}

}  // namespace evo
