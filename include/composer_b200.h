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
/* 0 = automatic engine choice, 1 = force SIMT, 2 = force tcgen05 (tests only). */
CB_API int cb_gemm_set_path(int path);

#ifdef __cplusplus
}
#endif
#endif /* COMPOSER_B200_H */
