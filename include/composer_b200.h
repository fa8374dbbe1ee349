/*
 * composer_b200 — C ABI of the B200-native decoder training-step kernels.
 *
 * Every function takes plain device pointers, extents, leading dimensions (in
 * elements) and a cudaStream_t passed as void*.  Kernels never allocate or free:
 * the caller (the Python host, through PyTorch's allocator) owns every buffer,
 * including workspaces.  Every function returns 0 on success or one of the CB_ERR_*
 * codes below; cb_last_error() returns the message of the most recent failure on
 * the calling thread.  The host maps codes onto the reference's ComposerError
 * taxonomy (reference pkg/src/composer/errors.py:8-112): CB_ERR_SHAPE -> ShapeError,
 * CB_ERR_UNSUPPORTED -> TypeMismatchError, anything else -> ComposerError.
 *
 * Each entry point names the reference operation it replaces (file:line in
 * /root/reference/pkg/src/composer/).  The reference computes only the forward
 * pass in float64 numpy; the backward and optimizer entry points implement the
 * gradient/update of that same forward (parity pinned by the repo's oracle/).
 *
 * dtype codes: CB_DT_F32 = 0, CB_DT_BF16 = 1.
 */
#ifndef COMPOSER_B200_H
#define COMPOSER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CB_API __attribute__((visibility("default")))

/* status / diagnostics */
CB_API const char* cb_last_error(void);
CB_API int cb_abi_version(void);
/* Kernels launched by this library in this process so far (benchmark evidence). */
CB_API long long cb_launch_count(void);

/* ---------------------------------------------------------------------------------
 * GEMM:  D[M,N] = alpha * op(A) @ op(B)  (+ D if accumulate)  (+ R if R != NULL)
 *   op(A) is MxK: trans_a = 0 -> A stored [M][K] (row stride lda); 1 -> A stored [K][M].
 *   op(B) is KxN: trans_b = 0 -> B stored [K][N] (row stride ldb); 1 -> B stored [N][K].
 *   trans_b = 0 is the reference's `x @ W` with W laid out [in, out]
 *   (layers.py:131,167 Linear; :340-348 attention projections; :412-416 FFN;
 *   :516 MoE router); trans_b = 1 with B = the embedding table is the tied head
 *   `h @ table.T` (layers.py:597).
 *   in_dtype selects the arithmetic: CB_DT_BF16 -> tcgen05 (bf16 x bf16 -> f32 TMEM
 *   accumulation) when operands are 16-byte aligned, else an f32-accumulating SIMT
 *   kernel; CB_DT_F32 -> f32 SIMT (the fp32 parity mode).
 * ------------------------------------------------------------------------------- */
CB_API int cb_gemm(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                   int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, const void* R, int64_t ldr,
                   int r_dtype, float alpha, int accumulate, void* stream);
/* The AdamW update (fn:adamw, layers.py:657-663; cb_adamw below) fused into a weight-gradient
 * GEMM whose product alpha * op(A) @ op(B) is the whole gradient of the output elements this
 * step: the epilogue updates param / exp_avg / exp_avg_sq (f32) and writes param_bf16
 * (optional) at D's positions; D (the gradient buffer's view, row stride ldd) is an address
 * frame only, never read or written.  Same engines as cb_gemm; bit-identical to cb_gemm
 * accumulating into a zeroed D followed by cb_adamw on D. */
CB_API int cb_gemm_adamw(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                         int64_t ldb, int trans_b, void* D, int64_t ldd, float alpha, float* param, float* exp_avg,
                         float* exp_avg_sq, void* param_bf16, float lr, float beta1, float beta2, float eps,
                         float weight_decay, int step, void* stream);
/* 0 = automatic engine choice, 1 = force SIMT, 2 = force tcgen05 (tests only). */
CB_API int cb_gemm_set_path(int path);
/* Cluster mode of the tcgen05 engine: 1 (default) = CTA-pair MMA (cta_group::2, 256x256
   tiles); 2 = cluster pairs sharing the B tile via TMA multicast; 3 = CTA pair; 0 = one CTA
   per 128-row tile. */
CB_API int cb_gemm_set_multicast(int mode);
/* Raster group height of the persistent GEMMs' tile order (tile rows that share each N step;
 * default 16; A/B of the L2 reuse pattern, no effect on results). */
CB_API int cb_gemm_set_raster(int group_m);
/* The CTA-pair GEMM's epilogues move their rows through a per-warp shared-memory stage so
 * global accesses are coalesced.  Bit mask: 1 bf16 outputs, 2 gated-activation backward;
 * 1 = both (default); 0 = per-lane row stores everywhere (A/B and tests). */
CB_API int cb_gemm_set_staged_epilogue(int enable);
/* Registers a caller-owned device buffer (16-byte aligned) the CTA-pair engine may use for
   split-K partials (f32 [S][M][N]) on GEMMs whose tile count leaves the last wave mostly
   idle; slices are summed in a fixed order by a second kernel (deterministic).  bytes = 0
   disables split-K.  The library never allocates. */
CB_API int cb_gemm_set_workspace(void* ptr, int64_t bytes);
/* D = op(A) @ op(B) with RoPE (layers.py:235-257; positions = row % seq_len) applied to
 * output columns [0, rope_cols) — the q|k part of the fused QKV projection (layers.py:340-343).
 * Rotated in the tcgen05 epilogue (no extra HBM pass); other engines rotate afterwards. */
CB_API int cb_gemm_rope(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                        int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, int seq_len, int head_dim,
                        int rope_cols, const float* cos_t, const float* sin_t, void* stream);
/* Gated-activation FFN GEMMs with the activation in the epilogue (replace reference
 * layers.py:405-416, act0(x @ w1) * act1(x @ w1_gate), and its backward); bf16, CTA-pair
 * tcgen05 engine.  act ids as cb_act_fwd.
 *   fwd: pre[M, 2H] = A @ B with B = [w1 | w1_gate] ([K, 2H] or its transpose),
 *        hidden[M, H] = act0(pre[:, :H]) * act1(pre[:, H:]) (from the bf16-rounded pre). H % 128 == 0.
 *   bwd: dhidden = A @ B (A = d(ffn output), B = w2^T); dpre[:, :H] = dhidden act0'(a) act1(g),
 *        dpre[:, H:] = dhidden act0(a) act1'(g) with [a | g] = pre; dhidden is never stored.
 * Both return CB_ERR_UNSUPPORTED without launching anything when the fused form does not
 * apply (M < 256, H % 32, alignment, engine disabled): the caller runs cb_gemm + cb_act_*. */
CB_API int cb_gemm_gated_fwd(int M, int H, int K, const void* A, int64_t lda, int trans_a, const void* B,
                             int64_t ldb, int trans_b, void* pre, int64_t ldpre, void* hidden, int64_t ldh, int act0,
                             int act1, void* stream);
CB_API int cb_gemm_gated_bwd(int M, int H, int K, const void* A, int64_t lda, int trans_a, const void* B,
                             int64_t ldb, int trans_b, const void* pre, int64_t ldpre, void* dpre, int64_t lddpre,
                             int act0, int act1, void* stream);

/* Grouped GEMMs: every MoE expert in ONE persistent launch (layers.py:513-533, the expert
 * einsums; replaces the per-expert loop and its host round trip for the expert offsets).
 * grp_off: DEVICE int[groups+1] row offsets, each a multiple of 256 (cb_moe_dispatch_padded).
 * mode 1 (groups split the rows): D[rows of g] = op(A)[rows of g] @ op(B_g); B_g is block g of
 *   B stacked along K ([groups*K][N], trans_b = 0) or along N ([groups*N][K], trans_b = 1);
 *   M = the row capacity (multiple of 256); only rows < grp_off[groups] are computed.
 * mode 2 (groups split K): D_g (+)= A[rows of g]^T @ B[rows of g] (trans_a = 1, trans_b = 0,
 *   K = the row capacity); D_g = rows [g*M, (g+1)*M) of D; an empty group writes nothing.
 * The gated forms are cb_gemm_gated_fwd/bwd (mode 1) with B = every expert's [W1|Wg]
 * stacked [groups*K][2H] (fwd) or W2 stacked [groups*H][K] read transposed (bwd). */
CB_API int cb_gemm_grouped(int mode, int groups, const int* grp_off, int M, int N, int K, const void* A, int64_t lda,
                           int trans_a, const void* B, int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype,
                           float alpha, int accumulate, void* stream);
CB_API int cb_gemm_gated_fwd_grouped(int groups, const int* grp_off, int M, int H, int K, const void* A, int64_t lda,
                                     const void* B, int64_t ldb, void* pre, int64_t ldpre, void* hidden, int64_t ldh,
                                     int act0, int act1, void* stream);
CB_API int cb_gemm_gated_bwd_grouped(int groups, const int* grp_off, int M, int H, int K, const void* A, int64_t lda,
                                     const void* B, int64_t ldb, const void* pre, int64_t ldpre, void* dpre,
                                     int64_t lddpre, int act0, int act1, void* stream);

/* ---------------------------------------------------------------------------------
 * RMSNorm (layers.py:176-193): y = x / sqrt(mean(x^2) + eps) * scale, rstd[row] saved.
 * Backward: dx = dres + d(norm)/dx . dy  (dres: the residual branch gradient, may be
 * NULL); dscale += sum_rows dy * x * rstd (needs `workspace` of
 * cb_rmsnorm_bwd_workspace bytes when dscale != NULL).  scale/rstd/dx/dscale are f32.
 * ------------------------------------------------------------------------------- */
CB_API int cb_rmsnorm_fwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale, float eps,
                          void* y, int64_t ldy, int y_dtype, float* rstd, void* stream);
CB_API int cb_rmsnorm_bwd_workspace(int rows, int dim, int64_t* bytes);
CB_API int cb_rmsnorm_bwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale,
                          const float* rstd, const void* dy, int64_t lddy, int dy_dtype, const float* dres,
                          int64_t lddres, float* dx, int64_t lddx, void* dx_bf16, int64_t lddxb, float* dscale,
                          float* workspace, void* stream);
/* out[d] (+)= sum_p partial[p][d] in fixed order (deterministic). */
CB_API int cb_col_reduce(int nparts, int dim, const float* partial, float* out, int accumulate, void* stream);

/* ---------------------------------------------------------------------------------
 * Embedding (layers.py:199-229): out[i] = table[ids[i]].  The backward is
 * deterministic: cb_sort_ids groups positions by id (stable counting sort: one CTA, or
 * per-1024-position chunks for vocab <= 64 such as the MoE expert ids; offsets
 * int32[vocab+1], cursor int32[cb_sort_ids_scratch(n, vocab)] scratch, perm int32[n]), then
 * cb_embedding_bwd adds each id's rows, in position order, into dtable (f32).
 * ------------------------------------------------------------------------------- */
CB_API int cb_embedding_fwd(int64_t n, int dim, const int64_t* ids, const void* table, int64_t ldt, int t_dtype,
                            void* out, int64_t ldo, int o_dtype, void* stream);
CB_API int64_t cb_sort_ids_scratch(int n, int vocab);
CB_API int cb_sort_ids(int n, int vocab, const int64_t* ids, int* offsets, int* cursor, int* perm, void* stream);
CB_API int cb_embedding_bwd(int vocab, int dim, const int* offsets, const int* perm, const void* dout, int64_t ldo,
                            int g_dtype, float* dtable, int64_t ldt, void* stream);

/* ---------------------------------------------------------------------------------
 * RoPE (layers.py:235-257, RoPEBehavior :267-276), in place on [rows = B*T] x heads x
 * head_dim with row stride ld: interleaved pairs rotated by cos/sin tables f32
 * [seq_len][head_dim/2]; inverse = 1 applies the transpose rotation (the backward).
 * ------------------------------------------------------------------------------- */
CB_API int cb_rope(int64_t rows, int seq_len, int heads, int head_dim, void* x, int64_t ld, int dtype,
                   const float* cos_t, const float* sin_t, int inverse, void* stream);

/* ---------------------------------------------------------------------------------
 * Activations (layers.py:55-77, FFN :405-416).  ids: 0 linear, 1 relu, 2 silu,
 * 3 sigmoid, 4 tanh.  out = act0(a) * act1(g) (g == NULL: out = act0(a)).
 * ------------------------------------------------------------------------------- */
CB_API int cb_act_fwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                      int64_t ldg, void* out, int64_t ldo, int dtype, void* stream);
CB_API int cb_act_bwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                      int64_t ldg, const void* dout, int64_t lddo, void* da, int64_t ldda, void* dg, int64_t lddg,
                      int dtype, void* stream);
/* out (+)= alpha * in, 2-D strided, with dtype conversion. */
CB_API int cb_copy2d(int64_t rows, int cols, const void* in, int64_t ldi, int in_dtype, void* out, int64_t ldo,
                     int out_dtype, float alpha, int accumulate, void* stream);
CB_API int cb_memset_zero(void* ptr, int64_t bytes, void* stream);
/* out[i] = scale * sum_q parts[q][i] for q = 0..nparts-1 in order (1 <= nparts <= 8; f32;
 * n % 4 == 0; 16-byte aligned).  `parts` is a HOST array of nparts device pointers.  The
 * local half of the FSDP gradient reduce-scatter (replaces the reduce in NCCL's
 * reduce_scatter_tensor(AVG); the reference has no distributed step). */
CB_API int cb_sum_parts(int nparts, int64_t n, const void* parts, void* out, float scale, void* stream);
/* f32 -> x1 + x2 + x3, three bf16 terms (relative remainder ~2^-24): the operand split of the f32
 * parity mode's GEMMs on the tcgen05 engine (ops.gemm: six bf16 products accumulated in f32, the
 * BF16x6 FP32 emulation).  src: [rows][cols] with row stride ld; outputs contiguous. */
CB_API int cb_split_bf16x3(int64_t rows, int cols, const float* src, int64_t ld, void* d1, void* d2, void* d3,
                           void* stream);

/* Stream memory operations for cross-GPU ordering without a kernel (FSDP barriers,
 * CB_FSDP_MEMOP_BARRIER): cb_stream_signal writes `epoch` to each of n 32-bit slots (peers'
 * signal slots through the symmetric-memory mapping; a memory barrier first orders the stream's
 * earlier writes); cb_stream_wait blocks the stream until each slot is >= epoch. */
CB_API int cb_stream_signal(void* const* slots, int n, uint32_t epoch, void* stream);
CB_API int cb_stream_wait(void* const* slots, int n, uint32_t epoch, void* stream);

/* ---------------------------------------------------------------------------------
 * Attention (layers.py:282-348), unmasked, flash-style (P never stored).  q/k/v/o
 * rows are tokens (b*T + t), head h at columns [h*hd, (h+1)*hd).  lse/delta are f32
 * [B][H][T].  kv_heads < heads is grouped-query attention (query head h reads kv head
 * h / (heads/kv_heads)); kv_heads == heads is the reference's attention.
 * o_lo (bf16 only, nullable, o's layout): the forward writes o - bf16(o), and the backward
 * forms delta = rowsum(dO * (o + o_lo)) — the flash backward's delta at ~16 significant bits
 * instead of bf16 o's 8 (it multiplies every dS = P (dP - delta) entry).
 * ds_ws (nullable, >= B*H*T*T bf16): with it and T % 128 == 0 the tcgen05 backward stores dS^T
 * from the dK/dV sweep and forms dQ as a GEMM over it (dq_gemm_k) instead of the dQ sweep that
 * recomputes S and dP (7 -> 5 MMA units per tile pair); without it, the two-sweep backward.
 * ------------------------------------------------------------------------------- */
CB_API int cb_attention_fwd(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype, const void* q,
                            int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* o, int64_t ldo,
                            void* o_lo, float* lse, float scale, void* stream);
CB_API int cb_attention_bwd(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype, const void* q,
                            int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, const void* o,
                            int64_t ldo, const void* o_lo, const float* lse, const void* dout, int64_t lddo,
                            float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                            float scale, void* ds_ws, int64_t ds_bytes, void* stream);
/* Backward for q/k rotated by cb_gemm_rope: dq/dk are returned un-rotated (the RoPE backward). */
CB_API int cb_attention_bwd_rope(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype,
                                 const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                 const void* o, int64_t ldo, const void* o_lo, const float* lse, const void* dout,
                                 int64_t lddo, float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                                 int64_t lddv, float scale, const float* cos_t, const float* sin_t, void* ds_ws,
                                 int64_t ds_bytes, void* stream);
/* 0 = automatic (tensor-core flash kernels when eligible), 1 = force SIMT (tests). */
CB_API int cb_attention_set_path(int path);
/* 1 (default) = the tcgen05/TMEM kernels for bf16 head_dim 128 (the Python layer zero-pads
 * head_dim 16/32/64 to 128 for them); 0 = the SIMT engine (tests). */
CB_API int cb_attention_set_tc(int enable);
/* 1 (default) = the backward's dQ sweep on CTA pairs (cta_group::2 MMAs over 256 query rows;
 * needs seq_len % 256 == 0, else the single-CTA sweep runs); 0 = single-CTA sweep.  Same bits. */
CB_API int cb_attention_set_dq_pair(int enable);
/* 1 = the backward's dK/dV sweep on CTA pairs (cta_group::2 MMAs over 256 keys; needs
 * seq_len % 256 == 0, else the single-CTA sweep runs); 0 (default) = single-CTA sweep. */
CB_API int cb_attention_set_dkdv_pair(int enable);

/* ---------------------------------------------------------------------------------
 * Next-token cross-entropy (TrainerBehavior.forward, layers.py:638-651) fused with its
 * gradient: row b*T+t of logits [B*T, V] predicts tokens[b, t+1]; rows t = T-1 get a
 * zero gradient.  dlogits = (softmax - onehot) * grad_scale (may alias logits, or be
 * NULL for forward-only).  row_loss f32[B*T] scratch; the mean over B*(T-1) rows goes
 * to *loss64 / *loss32 (either may be NULL).
 * ------------------------------------------------------------------------------- */
CB_API int cb_xent_fwd_bwd(int batch, int seq_len, int vocab, const void* logits, int64_t ld, int l_dtype,
                           const int64_t* tokens, float* row_loss, void* dlogits, int64_t ldg, int g_dtype,
                           float grad_scale, double* loss64, float* loss32, void* stream);

/* ---------------------------------------------------------------------------------
 * AdamW (the update the fn:adamw factory at layers.py:657-663,778-782 describes) over a
 * flat f32 shard; optionally refreshes the bf16 working copy in the same pass.
 * ------------------------------------------------------------------------------- */
CB_API int cb_adamw(int64_t n, float* param, const float* grad, float* exp_avg, float* exp_avg_sq, void* param_bf16,
                    float lr, float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale,
                    void* stream);
/* AdamW on the FSDP reduce-scatter's parts: grad = scale * (parts[0] + parts[1] + ...) summed in
 * list order (cb_sum_parts' arithmetic, so bit-identical to cb_sum_parts + cb_adamw) without the
 * summed gradient's HBM round trip; grad_out (nullable) still receives it.  n % 4 == 0. */
CB_API int cb_adamw_parts(int64_t n, int nparts, const void* parts, float scale, float* grad_out, float* param,
                          float* exp_avg, float* exp_avg_sq, void* param_bf16, float lr, float beta1, float beta2,
                          float eps, float weight_decay, int step, void* stream);

/* ---------------------------------------------------------------------------------
 * MoE (layers.py:422-533).  cb_moe_route: probs = softmax(x @ router) in f64 per token,
 * stable top-k (ties -> lowest expert id, layers.py:437), weights renormalized over the
 * k picks (layers.py:440); idx int32[n][k], weights f32[n][k], probs f32[n][E].
 * cb_moe_stats: out f64[1+2E] = [load_balance_loss, counts..., mean_probs...]
 * (layers.py:441-449).  Dispatch/combine use cb_sort_ids on the expert ids.
 * ------------------------------------------------------------------------------- */
CB_API int cb_moe_route(int64_t n, int dim, int experts, int top_k, const void* x, int64_t ldx, int x_dtype,
                        const float* router, int32_t* idx, float* weights, float* probs, void* stream);
CB_API int cb_moe_stats(int64_t n, int experts, int top_k, const int32_t* idx, const float* probs, double* out,
                        void* stream);
CB_API int cb_gather_rows(int64_t n, int dim, const int32_t* perm, int div, const void* x, int64_t ldx, void* out,
                          int64_t ldo, int dtype, void* stream);
/* out[t] (+)= sum_j w[t,j] * y[inv[t*k+j]]  (weights == NULL -> 1), slot order (layers.py:529-531). */
CB_API int cb_moe_combine(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights, const void* y,
                          int64_t ldy, int y_dtype, float* out, int64_t ldo, int accumulate, void* stream);
/* out[t] = res[t] + sum_j w[t,j] * y[inv[t*k+j]]: the MoE block output with the pre-norm residual
 * add of TransformerLayer (layers.py:539-551) fused; f32 y/res/out, 16-byte aligned rows,
 * dim % 4 == 0 (else CB_ERR_UNSUPPORTED, nothing launched). */
CB_API int cb_moe_combine_residual(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights,
                                   const float* y, int64_t ldy, const float* res, int64_t ldr, float* out,
                                   int64_t ldo, void* stream);
CB_API int cb_moe_combine_bwd(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights, const float* y,
                              int64_t ldy, const float* dout, int64_t lddo, void* dy, int64_t lddy, int dy_dtype,
                              float* dweights, void* stream);
CB_API int cb_moe_router_bwd(int64_t n, int experts, int top_k, const float* probs, const int32_t* idx,
                             const float* weights, const float* dweights, float* dlogits, void* stream);
/* Router backward products (x @ router, layers.py:516): drouter (+)= x^T dlogits (fixed token
 * blocks + ordered reduction; workspace ceil(n/128)*dim*experts floats) and
 * dx += dlogits router^T. */
CB_API int cb_moe_router_bwd_gemms(int64_t n, int dim, int experts, const void* x, int64_t ldx, int x_dtype,
                                   const float* dlogits, const float* router, float* drouter, float* dx,
                                   int64_t lddx, float* workspace, void* stream);
CB_API int cb_invert_perm(int64_t n, const int32_t* perm, int32_t* inv, void* stream);
CB_API int cb_widen_i32(int64_t n, const int32_t* a, int64_t* b, void* stream);
/* Padded expert layout for the grouped GEMMs, on the device: from the stable sort's expert
 * offsets, poff[e] (each expert's rows rounded up to 256), xe[poff[e] + j] = x[perm[off[e]+j] / top_k]
 * with the pad rows zeroed, and pinv[assignment] = its padded row (for cb_moe_combine{,_bwd}).
 * cap (rows of xe) >= nk + 255 * experts. */
CB_API int cb_moe_dispatch_padded(int64_t nk, int dim, int experts, int top_k, const int* offsets, const int32_t* perm,
                                  const void* x, int64_t ldx, int dtype, int* poff, int32_t* pinv, void* xe,
                                  int64_t ldxe, int cap, void* stream);
/* Zeroes the pad rows of a padded-layout buffer (e.g. the combine backward's dY). */
CB_API int cb_moe_zero_pad_rows(int cap, int dim, int experts, const int* offsets, const int* poff, void* buf,
                                int64_t ld, int dtype, void* stream);

/* ---------------------------------------------------------------------------------
 * Parameter init on the device, bit-identical to init_state (prng.py:61-69,
 * layers.py:114-116): numpy PCG64 stream from (state, inc) (the host derives them from
 * the key with SeedSequence), uniform(low, high) in C order.  Element i of a tensor with
 * `cols` columns lands at bucket position offset + (i/cols)*ld + col0 + i%cols (ld = 0:
 * offset + i).  master (f32) receives positions [master_begin, master_end) (this rank's
 * shard, indexed from master_begin); work (the full working copy) receives all.
 * ------------------------------------------------------------------------------- */
CB_API int cb_init_uniform(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int64_t n,
                           double low, double high, int64_t cols, int64_t ld, int64_t col0, int64_t offset,
                           float* master, int64_t master_begin, int64_t master_end, void* work, int work_dtype,
                           void* stream);
CB_API int cb_init_const(int64_t n, float value, int64_t cols, int64_t ld, int64_t col0, int64_t offset, float* master,
                         int64_t master_begin, int64_t master_end, void* work, int work_dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COMPOSER_B200_H */
