/*
 * evoformer_sm100.h -- C ABI of libevoformer_sm100.so, the B200 (sm_100a)
 * kernels behind the Evoformer hot path of the reference package `evotrain`
 * (reference: /root/reference/pkg/src/evotrain, abbreviated src/).
 *
 * The reference boundary is a pure-Python operator API; each entry point
 * below names the reference interface it replaces (file:line).  The Python
 * host package `paper_2207_05477_b200` binds these through ctypes (see
 * INTEGRATION.md for the binding a maintainer of the reference would add).
 *
 * Conventions
 *  - Every function returns EVO_OK (0) or an EVO_ERR_* code; the message of
 *    the last failure on the calling thread is evo_last_error().
 *  - The caller allocates every buffer (device pointers).  Workspaces are
 *    sized with the matching *_workspace() query.  No host synchronisation;
 *    all work is enqueued on `stream` (a cudaStream_t passed as void*).
 *  - Storage dtype codes: EVO_F32 (fp32 parity mode) or EVO_BF16 (bf16
 *    storage, fp32 math).  Parameters and their gradients are always fp32
 *    (the fused-buffer regions of src/fusion.py:84-111); residual-stream
 *    gradients are fp32.
 *  - Row-major tensors.  "Tokens" are rows of [B, L] problems: the token
 *    of (batch b, position l) is row b*tok_sb + l*tok_sl, which lets the
 *    four attention variants (MSA row/column, triangle start/end) read one
 *    token-major buffer without any transpose (src/model.py:320-398).
 */
#ifndef EVOFORMER_SM100_H
#define EVOFORMER_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVO_OK 0
#define EVO_ERR_ARG 1         /* shape/argument contract (DimensionError / ContractError) */
#define EVO_ERR_CUDA 2        /* CUDA runtime / launch failure */
#define EVO_ERR_UNSUPPORTED 3 /* no kernel for this shape/dtype/device */
#define EVO_ERR_INTERNAL 4

#define EVO_F32 0
#define EVO_BF16 1

/* Partial-sum rows used by every deterministic column reduction. */
#define EVO_PARTIAL_BLOCKS 256

/* ---- library ------------------------------------------------------------ */
const char* evo_last_error(void);
int evo_version(void);
/* 0 if the current device is sm_100 (B200) and the kernels can run. */
int evo_device_check(int* sm_major, int* sm_minor, int* num_sms);
/* Kernel-launch counter (launches issued by this library on this thread). */
int64_t evo_launch_count(void);
/* Deferred reductions: between begin and end, the per-block partial rows of
 * every column reduction (bias / LayerNorm-affine / pair-bias weight grads)
 * go into `arena` and their finalisation is batched into one launch at
 * evo_defer_end (fixed summation order, identical results).  The arena must
 * stay alive until evo_defer_end's work has run on `stream`. */
int evo_defer_begin(void* arena, size_t bytes);
int evo_defer_end(void* stream);
size_t evo_defer_used(void);

/* ---- dense projections ----------------------------------------------------
 * Replaces the np.matmul projections of src/attention.py:141,167,173,
 * src/model.py:314,346-347,363-364,378.  Row-major, batched-strided:
 *   C_b[M,N] = alpha * op(A_b)[M,K] . op(B_b)[K,N] + beta * C_b
 * ab_dtype: EVO_F32 (true fp32, no TF32) or EVO_BF16; c_dtype: F32 or BF16.
 * bf16 operands run on the library's tcgen05 + TMA GEMM (gemm_tc.cu:
 * persistent, warp-specialised, split-K with a deterministic reduction for
 * long K); fp32 operands (the parity mode: true fp32, no TF32) and operands
 * TMA cannot address (16-B alignment of base and row pitch) run on the
 * library's CUDA-core GEMM (gemm_simt.cu).  No CUDA math library is used. */
int evo_gemm(int64_t M, int64_t N, int64_t K,
             const void* A, int64_t lda, int trans_a, int64_t stride_a,
             const void* B, int64_t ldb, int trans_b, int64_t stride_b,
             void* C, int64_t ldc, int64_t stride_c, int batch,
             float alpha, float beta, int ab_dtype, int c_dtype, void* stream);

/* Number of evo_gemm / evo_gemm_bias calls that ran on the tensor cores
 * (process-wide; instrumentation for tests and the bench). */
int64_t evo_gemm_tc_launches(void);

/* Projection with its module epilogue fused (replaces the np.matmul + bias +
 * residual of src/attention.py:173 / src/model.py:346-348, 378 and the
 * matmul + bias + relu of src/model.py:346):
 *   out[M,N] = op(A) . op(B) + bias[N] (+ res[M,N])      relu == 0
 *   out[M,N] = relu(op(A) . op(B) + bias[N])              relu == 1, res == NULL
 * res: contiguous [M, N] (ld = N), alias of nothing else; res_dtype its storage
 * dtype.  The epilogue runs in fp32 on the accumulator (fp32 bias) before the
 * single rounding to c_dtype.  bias_bf16 is accepted for ABI compatibility and
 * ignored. */
int evo_gemm_bias(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int trans_a,
                  const void* B, int64_t ldb, int trans_b, const void* res, int res_dtype,
                  const float* bias, const void* bias_bf16, int relu, void* out, int64_t ldo,
                  int ab_dtype, int c_dtype, void* stream);

/* D[M, N] = (h > 0) ? op(A) op(B) : 0 -- the transition's ReLU backward in the
 * epilogue of the d(hidden) projection (src/model.py:344-348 differentiated);
 * h is the saved ReLU output, [M, N] contiguous like D.  With colsum != NULL
 * the epilogue also forms the column sums of the stored D (the hidden bias
 * gradient, b1), written (or added, accumulate = 1) to colsum[N] in a fixed
 * order; ws >= evo_gemm_relu_mask_workspace(M, N) bytes.  bf16 on the tensor
 * cores; EVO_ERR_UNSUPPORTED otherwise (the caller masks separately). */
int64_t evo_gemm_relu_mask_workspace(int64_t M, int64_t N);
int evo_gemm_relu_mask(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int trans_a, const void* B,
                       int64_t ldb, int trans_b, const void* h, void* D, int dtype, float* colsum, int accumulate,
                       void* ws, void* stream);

/* ---- LayerNorm (src/tensor.py:173-208) -----------------------------------
 * y = (x - mean) * rstd * gamma + beta over the last dim C; saves mean/rstd. */
int evo_layernorm_fwd(const void* x, int x_dtype, const float* gamma, const float* beta,
                      void* y, int y_dtype, float* mean, float* rstd,
                      int64_t rows, int64_t C, float eps, void* stream);
/* dx = dres + LN'(dy) (dres nullable; dx may alias dres), dgamma/dbeta
 * written (accumulate=0) or added (accumulate=1).  ws: workspace bytes from
 * evo_layernorm_bwd_workspace. */
int64_t evo_layernorm_bwd_workspace(int64_t rows, int64_t C);
int evo_layernorm_bwd(const void* x, int x_dtype, const void* dy, int dy_dtype,
                      const float* mean, const float* rstd, const float* gamma,
                      const float* dres, float* dx, float* dgamma, float* dbeta,
                      int accumulate, void* ws, int64_t rows, int64_t C, void* stream);
/* As evo_layernorm_bwd, also emitting a bf16 copy of dx (nullable) and the
 * column sums of dx (nullable) -- the next module's output-bias gradient and
 * GEMM operand come out of the same pass.  Power-of-two C in [32, 1024]. */
int evo_layernorm_bwd_ex(const void* x, int x_dtype, const void* dy, int dy_dtype,
                         const float* mean, const float* rstd, const float* gamma,
                         const float* dres, float* dx, void* dx_bf16, float* dxsum,
                         float* dgamma, float* dbeta, int accumulate, void* ws,
                         int64_t rows, int64_t C, void* stream);

/* ---- elementwise glue (src/tensor.py:244-331) ---------------------------- */
/* out = res + y + bias (res nullable, bias nullable). */
int evo_bias_residual(const void* res, int res_dtype, const void* y, int y_dtype,
                      const float* bias, void* out, int out_dtype,
                      int64_t rows, int64_t C, void* stream);
/* y = relu(y + bias), in place. */
int evo_bias_relu(void* y, int dtype, const float* bias, int64_t rows, int64_t C, void* stream);
/* dh *= (h > 0) in place; db (+)= colsum(dh). */
int evo_relu_bwd_colsum(void* dh, const void* h, int dtype, float* db, int accumulate,
                        void* ws, int64_t rows, int64_t C, void* stream);
/* out (+)= colsum(x) (x fp32 or bf16); optionally y = cast(x) to y_dtype. */
int64_t evo_colsum_workspace(int64_t C);
int evo_colsum_cast(const void* x, int x_dtype, float* out, int accumulate,
                    void* y, int y_dtype, void* ws, int64_t rows, int64_t C, void* stream);
/* Column sums of a row-strided [rows, C] view (leading dimension ld >= C):
 * bias gradients of column slices of a merged projection (the
 * `reduce_sum(dy, axis=0)` of src/attention.py:187 applied per slice). */
int evo_colsum_strided(const void* x, int x_dtype, int64_t ld, float* out, int accumulate, void* ws,
                       int64_t rows, int64_t C, void* stream);
int evo_cast(const void* x, int x_dtype, void* y, int y_dtype, int64_t n, void* stream);
/* Column-block packing for the merged Q|K|V|G projection (src/attention.py:
 * 133-141 concatenates Wq|Wk|Wv the same way): unpack=0 packs, for each of the
 * n groups, four [C, N] matrices src[4*i + s] into dst[i] = [C, 4N]; unpack=1
 * splits src[i] = [C, 4N] into dst[4*i + s].  Pointer/size arrays are host
 * memory; one launch per 64 groups. */
int evo_pack_cols(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N,
                  int n, int src_dtype, int dst_dtype, int unpack, void* stream);
/* The same with ns (2 or 4) matrices per group: dst[i] = [C, ns*N] (the OPM's
 * merged [w_left | w_right] projection, src/model.py:360-361). */
int evo_pack_cols_ns(const void* const* src, void* const* dst, const int64_t* C, const int64_t* N,
                     int n, int ns, int src_dtype, int dst_dtype, int unpack, void* stream);
/* in-place y *= s (fp32) */
int evo_scale_inplace(float* y, float s, int64_t n, void* stream);

/* ---- gated attention core (src/attention.py:118-233) ---------------------
 * qkvg: [tokens, 4*H*D] = x.[Wq|Wk|Wv|Wg] (row stride ld_qkvg).  Computes
 *   logits = (q.k^T)/sqrt(D) + (mask-1)*1e9 + nb,  w = softmax(logits),
 *   ctx = w.v,  gate = sigmoid(g + bg),  gated = ctx*gate
 * in the reference's accumulation order (:151-161).  mask is fp32 {0,1}
 * indexed b*mask_sb + l*mask_sl.  nb: [H, L, L] (query, key) in the storage
 * dtype -- bf16 in bf16 mode, as the reference rounds op outputs
 * (src/tensor.py:102-108); nullable.  lse: [B, H, L, 2] fp32 = (row max of
 * logits*log2(e), 1/row sum) -- kept apart because at a fully-masked row the
 * logits sit at -1e9 where m + log(sum) is not representable.
 * ctx/gate/gated: [tokens, H*D] storage dtype. */
int evo_attn_fwd(const void* qkvg, int64_t ld_qkvg, const float* mask, int64_t mask_sb,
                 int64_t mask_sl, const void* nb, const float* bg,
                 void* ctx, void* gate, void* gated, float* lse,
                 int64_t B, int64_t L, int64_t H, int64_t D, int64_t tok_sb, int64_t tok_sl,
                 int dtype, void* stream);
/* Backward closure (src/attention.py:178-221) from d(gated):
 * writes all four slots of dqkvg [tokens, 4*H*D] (dq, dk, dv, d(g pre-act)),
 * dnb [H, L, L] fp32 = sum over batches of dlogits (:219-220; nullable when
 * there is no bias), dbg (+)= colsum of d(g pre-act).  Deterministic. */
int64_t evo_attn_bwd_workspace(int64_t B, int64_t L, int64_t H, int64_t D, int dtype);
int evo_attn_bwd(const void* qkvg, int64_t ld_qkvg, const float* mask, int64_t mask_sb,
                 int64_t mask_sl, const void* nb, const void* ctx, const void* gate,
                 const void* dgated, const float* lse, void* dqkvg, float* dnb,
                 float* dbg, int accumulate, void* ws, size_t ws_bytes,
                 int64_t B, int64_t L, int64_t H, int64_t D, int64_t tok_sb, int64_t tok_sl,
                 int dtype, void* stream);

/* ---- pair bias (src/model.py:312-317) ------------------------------------
 * z: [R*R, C] pair tokens.  P[x,y,h] = LN(z[x,y]).w_bias[:,h]; written to
 * nb (storage dtype) as nb[h,x,y] (swap_xy=0: MSA row / triangle start) or
 * nb[h,y,x] (swap_xy=1: triangle end, whose rows are the pair's columns). */
/* The triangle attentions' input LayerNorm (ln_g, ln_b) and their pair-bias
 * projection (bias_ln_g, bias_ln_b, w_bias; src/model.py:312-317, 381-398)
 * read the same pair rows: one pass writes xl (bf16, z's layout), nb (as
 * evo_pair_bias_fwd_rect) and the shared row statistics.  bf16, c_z = 128,
 * H <= 8, >= 4096 tokens; EVO_ERR_UNSUPPORTED otherwise (the caller runs the
 * two ops separately). */
int evo_ln_pair_bias_fwd(const void* z, int dtype, const float* ln_g, const float* ln_b, const float* bias_ln_g,
                         const float* bias_ln_b, const float* w_bias, void* xl, void* nb, float* mean, float* rstd,
                         int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap_xy, void* stream);
int evo_pair_bias_fwd(const void* z, int dtype, const float* ln_g, const float* ln_b,
                      const float* w_bias, void* nb, float* mean, float* rstd,
                      int64_t R, int64_t C, int64_t H, int swap_xy, void* stream);
int64_t evo_pair_bias_bwd_workspace(int64_t C, int64_t H);
/* dz += LN_bwd(dP . w_bias^T) with dP read from dnb (fp32, same swap_xy);
 * dln_g, dln_b, dw_bias (+)= ... */
int evo_pair_bias_bwd(const void* z, int dtype, const float* mean, const float* rstd,
                      const float* ln_g, const float* ln_b, const float* w_bias, const float* dnb,
                      int swap_xy, float* dz, float* dln_g, float* dln_b,
                      float* dw_bias, int accumulate, void* ws,
                      int64_t R, int64_t C, int64_t H, void* stream);
/* Rectangular forms for one DAP shard: z holds NI x NJ tokens (x, y) at row
 * x*NJ + y; nb is [H, NI, NJ] (swap_xy=0) or [H, NJ, NI] (swap_xy=1).  The
 * square entry points above are these with NI = NJ = R. */
int evo_pair_bias_fwd_rect(const void* z, int dtype, const float* ln_g, const float* ln_b,
                           const float* w_bias, void* nb, float* mean, float* rstd,
                           int64_t NI, int64_t NJ, int64_t C, int64_t H, int swap_xy, void* stream);
/* evo_pair_bias_bwd_rect that also emits the updated dz as bf16 (dz16, may be
 * NULL) and its column sums (dzsum[C], written; may be NULL) in the same pass:
 * the next module's GEMM operand and output-bias gradient when this bias
 * gradient is the last write to dz.  bf16 z, c_z = 128, H <= 8, >= 4096
 * tokens (a multiple of 4); EVO_ERR_UNSUPPORTED (nothing written) otherwise. */
int evo_pair_bias_bwd_ex(const void* z, int dtype, const float* mean, const float* rstd, const float* ln_g,
                         const float* ln_b, const float* w_bias, const float* dnb, int swap_xy, float* dz,
                         float* dln_g, float* dln_b, float* dw_bias, int accumulate, void* ws, int64_t NI, int64_t NJ,
                         int64_t C, int64_t H, void* dz16, float* dzsum, void* stream);
int evo_pair_bias_bwd_rect(const void* z, int dtype, const float* mean, const float* rstd,
                           const float* ln_g, const float* ln_b, const float* w_bias, const float* dnb,
                           int swap_xy, float* dz, float* dln_g, float* dln_b,
                           float* dw_bias, int accumulate, void* ws,
                           int64_t NI, int64_t NJ, int64_t C, int64_t H, void* stream);

/* ---- outer product mean (src/model.py:351-378) ---------------------------
 * ab: [S*R, 2k] = LN(m).[Wl|Wr]; a = (ab[:, :k]+bl)*mask, c = (ab[:, k:]+br)*mask
 * written as [S, R*k] each. */
int evo_opm_proj(const void* ab, const float* bl, const float* br, const float* mask,
                 void* a, void* c, int64_t SR, int64_t k, int dtype, void* stream);
/* da, dc [S, R*k] -> d_ab [S*R, 2k] (masked), dbl/dbr (+)= colsums. */
int evo_opm_proj_bwd(const void* da, const void* dc, const float* mask, void* d_ab,
                     float* dbl, float* dbr, int accumulate, void* ws,
                     int64_t SR, int64_t k, int dtype, void* stream);
/* rec[i,j] = 1/(sum_s m[s,i] m[s,j] + 1e-3);  outn[i,j,p*k+q] = num[i*k+p, j*k+q]*rec[i,j] */
int evo_opm_norm_fwd(const void* num, int num_dtype, const float* mask, float* rec,
                     void* outn, int out_dtype, int64_t S, int64_t R, int64_t k, void* stream);
/* dnum[i*k+p, j*k+q] = doutn[i,j,p*k+q] * rec[i,j] */
int evo_opm_norm_bwd(const void* doutn, int in_dtype, const float* rec, void* dnum,
                     int out_dtype, int64_t R, int64_t k, void* stream);
/* Row-shard forms (DAP, src/model.py:375 reduce-scatter): num / dnum hold the
 * NI rows i0..i0+NI-1 ([NI*k, R*k]); rec and outn / doutn are [NI*R, ...];
 * the mask is the full [S, R] one. */
int evo_opm_norm_fwd_rows(const void* num, int num_dtype, const float* mask, float* rec,
                          void* outn, int out_dtype, int64_t S, int64_t R, int64_t k,
                          int64_t i0, int64_t NI, void* stream);
int evo_opm_norm_bwd_rows(const void* doutn, int in_dtype, const float* rec, void* dnum,
                          int out_dtype, int64_t R, int64_t k, int64_t NI, void* stream);
/* rec rows i0..i0+NI-1 alone (they depend only on the mask: computed once per
 * forward pass and shared by every block), and the normalisation with a given rec. */
int evo_opm_rec(const float* mask, float* rec, int64_t S, int64_t R, int64_t i0, int64_t NI, void* stream);
int evo_opm_norm_apply_rows(const void* num, int num_dtype, const float* rec, void* outn, int out_dtype,
                            int64_t R, int64_t k, int64_t NI, void* stream);

/* OPM backward d(pair) -> d(num) as one tcgen05 GEMM with the normalisation
 * and the [i*k+p, j*k+q] re-layout in its epilogue:
 *   dnum[i*k+p, j*k+q] = rec[i*R+j] * sum_c d_act[i*R+j, c] * w_out[p*k+q, c]
 * d_act [NI*R, C], w_out [k*k, C] bf16; dnum [NI*k, R*k] bf16.  Needs C = 128,
 * k = 32, R % 128 == 0 (EVO_ERR_UNSUPPORTED otherwise). */
int evo_opm_dnum(const void* d_act, const void* w_out, const float* rec, void* dnum, int64_t R, int64_t k,
                 int64_t NI, int64_t C, int dtype, void* stream);
/* OPM forward a, c -> outn: the sum over sequences as one tcgen05 GEMM with the
 * normalisation and the [(i, j), p*k+q] re-layout in its epilogue:
 *   outn[i*R+j, p*k+q] = rec[i*R+j] * sum_s a[s, i*k+p] * c[s, j*k+q]
 * a [S, NI*k], c [S, R*k], outn [NI*R, k*k] bf16.  Needs S = 128, k = 32,
 * R*k % 256 == 0 (EVO_ERR_UNSUPPORTED otherwise). */
int evo_opm_outn(const void* a, const void* c, const float* rec, void* outn, int64_t S, int64_t R, int64_t k,
                 int64_t NI, int dtype, void* stream);

/* ---- DAP re-layout (src/harness.py:262-293) ------------------------------
 * dst[b, a, :] = src[a, b, :] for src [A, B, elem_bytes]: the outer-axis swap
 * that brackets every DAP all-to-all / all-gather / reduce-scatter. */
int evo_swap01(const void* src, void* dst, int64_t A, int64_t B, int64_t elem_bytes, void* stream);

/* ---- loss (src/harness.py:313-320) ---------------------------------------
 * loss = km*sum(msa^2) + kz*sum(pair^2);  dmsa = 2*km*msa, dpair = 2*kz*pair (fp32). */
int64_t evo_sq_loss_workspace(void);
int evo_sq_loss(const void* msa, int64_t n_m, const void* pair, int64_t n_z, int dtype,
                float km, float kz, float* loss, float* dmsa, float* dpair, void* ws,
                void* stream);

/* ---- fused-buffer optimizer (src/fusion.py:150-233) ----------------------
 * One fp64 sum-of-squares pass over the pooled grad region, then one pass of
 * clip (scale = clip/norm if norm > clip) + Adam (bias-corrected) + EMA over
 * all five regions, optionally writing a bf16 shadow of the params.
 * Elementwise arithmetic is IEEE round-to-nearest in the reference's order,
 * so the trajectory is bitwise the reference's. */
int64_t evo_sumsq_workspace(void);
int evo_sumsq_f64(const float* g, int64_t n, double* out, void* ws, void* stream);
int evo_adam_clip_ema(float* p, const float* g, float* m, float* v, float* ema,
                      void* p_bf16, int64_t n, const double* sumsq, double clip,
                      float lr, float b1, float omb1, float b2, float omb2, float eps,
                      float bc1, float bc2, float decay, float omdecay, void* stream);
/* CUDA-graph-safe form of the same step: the step counter t lives on the
 * device.  evo_sumsq_f64_step also increments *step and writes this step's
 * bias corrections bc_out = (bc_table[t-1], bc_table[table_len + t-1]) (t
 * clamped to table_len: the host tabulates np.float32(1 - beta**t) for
 * t = 1..table_len, src/fusion.py:189-192, until both have rounded to 1.0f);
 * evo_adam_clip_ema_dev reads them from `bc`.  Replaying a captured step then
 * advances t exactly as an eager step does. */
int evo_sumsq_f64_step(const float* g, int64_t n, double* out, void* ws, int64_t* step,
                       const float* bc_table, int64_t table_len, float* bc_out, void* stream);
int evo_adam_clip_ema_dev(float* p, const float* g, float* m, float* v, float* ema,
                          void* p_bf16, int64_t n, const double* sumsq, double clip,
                          float lr, float b1, float omb1, float b2, float omb2, float eps,
                          const float* bc, float decay, float omdecay, void* stream);

/* ---- unfused gated-attention baseline (src/attention.py:78-115) -----------
 * gated_attention_reference: the reference's fine-grained composition with
 * materialised logits, the oracle of the fused operator
 * (tests/test_acceptance.py:46-71); fp32; its GEMMs are evo_gemm.
 * x [BS, H, R, R] logits -> softmax_j(x + (mask[bs*mask_sb + j*mask_sl] - 1)*1e9
 * + nb[h, i, j]) in place (:99-106; nb nullable). */
int evo_softmax_masked_rows(float* x, const float* mask, int64_t mask_sb, int64_t mask_sl, const float* nb,
                            int64_t BS, int64_t H, int64_t R, void* stream);
/* g <- w * (g - sum_j g * w) per row of R (softmax backward, in place) */
int evo_softmax_rows_bwd(const float* w, float* g, int64_t rows, int64_t R, void* stream);
/* gate = sigmoid(gp), gated = ctx * gate (:111-113), elementwise over n */
int evo_gate_fwd(const float* gp, const float* ctx, float* gate, float* gated, int64_t n, void* stream);
/* dctx = dgated * gate, dgp = dgated * ctx * gate * (1 - gate) */
int evo_gate_bwd(const float* dgated, const float* gate, const float* ctx, float* dctx, float* dgp, int64_t n,
                 void* stream);
/* out[c] (+)= sum_r x[r, c] over [rows, cols] fp32, rows in order (deterministic) */
int evo_sum_rows(const float* x, int64_t rows, int64_t cols, float* out, int accumulate, void* stream);

/* ---- triangle multiplication (extension; AF2 Supplementary Alg. 11/12) -----
 * Absent from the reference (planner inventory only, src/planner.py:37-45).
 * proj: [R*R, ld] token-major with column blocks [ap | ag | bp | bg] (width ch);
 * a = sigmoid(ag + b_ag) * (ap + b_ap) * mask (b likewise) written
 * channel-major [ch, R*R] for the channel-batched contractions (evo_gemm). */
int evo_trimul_gate_fwd(const void* proj, int64_t ld, const float* b_ap, const float* b_ag,
                        const float* b_bp, const float* b_bg, const float* mask, void* a_cm,
                        void* b_cm, int64_t RR, int64_t ch, int dtype, void* stream);
/* channel-major da, db -> token-major d(proj) [R*R, 4*ch] */
int evo_trimul_gate_bwd(const void* proj, int64_t ld, const float* b_ap, const float* b_ag,
                        const float* b_bp, const float* b_bg, const float* mask, const void* da_cm,
                        const void* db_cm, void* dproj, int64_t RR, int64_t ch, int dtype,
                        void* stream);
/* y[c, r] = x[r, c] (tiled; dtype conversion allowed) */
int evo_transpose2d(const void* x, int x_dtype, void* y, int y_dtype, int64_t rows, int64_t cols,
                    void* stream);
/* out = res + sigmoid(gp + bg) * (y + by), g_out = sigmoid(gp + bg); gp row stride ld_gp */
int evo_gated_residual(const void* res, const void* gp, int64_t ld_gp, const float* bg, const void* y,
                       const float* by, void* g_out, void* out, int64_t rows, int64_t C, int dtype,
                       void* stream);
/* dyb = dout*g, dgp = dout*(y+by)*g*(1-g) */
int evo_gated_residual_bwd(const float* dout, const void* g, const void* y, const float* by, void* dyb,
                           void* dgp, int64_t rows, int64_t C, int dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVOFORMER_SM100_H */
