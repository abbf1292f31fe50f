// Outer-product-mean contractions with the normalisation and the re-layout in
// the GEMM epilogue (src/model.py:366-378), on the library's tcgen05 GEMM
// (gemm_tc.cu, OPM output modes):
//
//   forward   outn[i*R + j, p*k + q] = rec[i*R + j] * sum_s a[s, i*k + p] c[s, j*k + q]
//   backward  dnum[i*k + p, j*k + q] = rec[i*R + j] * sum_c d_act[(i, j), c] w_out[p*k + q, c]
//
// The unfused sequences write num / doutn ([R*k, R*k] / [R^2, k^2], 134 MB at
// the bench shape), read them back to scale and permute, and write again;
// here the accumulator tiles leave TMEM already scaled and are stored by 4-D
// TMA boxes into the permuted layout (k = 32: a 32-row TMEM lane quarter is
// one i (forward) or 32 consecutive j (backward), a 32-column group one j or
// one p).  Measured at the bench shape: forward 54.8 -> 41.5 us, backward
// 47.1 -> 39.6 us against the previous dedicated kernels.
#include "common.cuh"

namespace evo {
bool gemm_tc_opm(int mode, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int ta, const void* B,
                 int64_t ldb, int tb, void* D, const float* rec, int64_t R, int64_t NI, cudaStream_t s);  // gemm_tc.cu
}  // namespace evo

extern "C" int evo_opm_dnum(const void* d_act, const void* w_out, const float* rec, void* dnum, int64_t R,
                            int64_t k, int64_t NI, int64_t C, int dtype, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(dtype == EVO_BF16, EVO_ERR_UNSUPPORTED, "opm_dnum: bf16 only");
  EVO_REQUIRE(k == 32 && R % 128 == 0 &&
                  evo::gemm_tc_opm(2, NI * R, k * k, C, d_act, C, 0, w_out, C, 1, dnum, rec, R, NI,
                                   (cudaStream_t)stream),
              EVO_ERR_UNSUPPORTED, "opm_dnum: needs k = 32, n_res a multiple of 128, 16-B aligned operands");
  EVO_API_END
}

extern "C" int evo_opm_outn(const void* a, const void* c, const float* rec, void* outn, int64_t S, int64_t R,
                            int64_t k, int64_t NI, int dtype, void* stream) {
  EVO_API_BEGIN
  EVO_REQUIRE(dtype == EVO_BF16, EVO_ERR_UNSUPPORTED, "opm_outn: bf16 only");
  // a, c: [S, R*k] rows -- the MN-major operands of num = a^T c
  EVO_REQUIRE(k == 32 && NI == R &&
                  evo::gemm_tc_opm(1, NI * k, R * k, S, a, R * k, 1, c, R * k, 0, outn, rec, R, NI,
                                   (cudaStream_t)stream),
              EVO_ERR_UNSUPPORTED, "opm_outn: needs k = 32, the whole residue range, 16-B aligned operands");
  EVO_API_END
}
