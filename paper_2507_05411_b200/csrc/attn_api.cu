// C-ABI entry points of the attention engines (dispatch: tensor-core flash kernels for
// bf16 with a supported head_dim, SIMT engine otherwise).
#include "attn.cuh"
#include "composer_b200.h"

namespace cb {
static int g_attn_path = 0;  // 0 auto, 1 force SIMT
}  // namespace cb

using namespace cb;

// tcgen05 backward: bf16 hd 128, 16-byte strides, and lse / delta rows the producer warp can
// bulk-copy (16-byte aligned rows: T % 4 == 0)
static bool tc_bwd_ok(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v, const float* lse,
                      const float* delta, int64_t lddo, int64_t lddq, int64_t lddk, int64_t lddv) {
  if (g_attn_path != 0 || !attn_tc_supported(g, dtype, q, k, v)) return false;
  if ((lddo | lddq | lddk | lddv) & 7) return false;
  return g.T % 4 == 0 && ((reinterpret_cast<uintptr_t>(lse) | reinterpret_cast<uintptr_t>(delta)) & 15) == 0;
}

// the optional dS^T workspace of the tcgen05 backward: B*H*T*T bf16, 16-byte aligned
static int ds_check(const AttnGeom& g, const void* ds_ws, int64_t ds_bytes) {
  if (!ds_ws) return CB_OK;
  const int64_t need = (int64_t)g.B * g.H * g.T * g.T * 2;
  if (ds_bytes < need || (reinterpret_cast<uintptr_t>(ds_ws) & 15))
    return fail(CB_ERR_ARG, "attention bwd: dS workspace needs %lld aligned bytes", (long long)need);
  return CB_OK;
}

namespace cb {
namespace tcb {
extern int g_dq_pair;
extern int g_dkdv_pair;
}
}  // namespace cb
extern "C" int cb_attention_set_dq_pair(int enable) {
  cb::tcb::g_dq_pair = enable ? 1 : 0;
  return CB_OK;
}
extern "C" int cb_attention_set_dkdv_pair(int enable) {
  cb::tcb::g_dkdv_pair = enable ? 1 : 0;
  return CB_OK;
}

extern "C" int cb_attention_set_path(int path) {
  if (path < 0 || path > 1) return fail(CB_ERR_ARG, "attention path must be 0 (auto) or 1 (simt)");
  g_attn_path = path;
  return CB_OK;
}

extern "C" int cb_attention_fwd(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype,
                                const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                void* o, int64_t ldo, void* o_lo, float* lse, float scale, void* stream) {
  AttnGeom g{batch, seq_len, heads, kv_heads, head_dim, ldq, ldk, ldv, ldo, scale};
  if (int s = check_geom(g)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (o_lo && dtype != CB_DT_BF16) return fail(CB_ERR_ARG, "attention: o_lo is the bf16 rounding residual of o");
  if (g_attn_path == 0 && attn_tc_supported(g, dtype, q, k, v)) return attn_fwd_tc(g, q, k, v, o, o_lo, lse, st);
  if (o_lo) {  // the other engines do not produce the residual: zero (delta then uses bf16 o)
    cudaError_t e = cudaMemset2DAsync(o_lo, (size_t)ldo * 2, 0, (size_t)heads * head_dim * 2,
                                      (size_t)batch * seq_len, st);
    if (e != cudaSuccess) return fail(CB_ERR_CUDA, "attention: o_lo memset: %s", cudaGetErrorString(e));
  }
  return attn_fwd_simt(g, dtype, q, k, v, o, lse, st);
}

extern "C" int cb_attention_bwd(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype,
                                const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                                const void* o, int64_t ldo, const void* o_lo, const float* lse, const void* dout,
                                int64_t lddo, float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                                int64_t lddv, float scale, void* ds_ws, int64_t ds_bytes, void* stream) {
  AttnGeom g{batch, seq_len, heads, kv_heads, head_dim, ldq, ldk, ldv, ldo, scale};
  if (int s = check_geom(g)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (int s = ds_check(g, ds_ws, ds_bytes)) return s;
  if (int s = attn_delta(g, dtype, o, o_lo, dout, lddo, delta, st)) return s;
  if (tc_bwd_ok(g, dtype, q, k, v, lse, delta, lddo, lddq, lddk, lddv))
    return attn_bwd_tc(g, q, k, v, dout, lddo, lse, delta, dq, lddq, dk, lddk, dv, lddv, st, nullptr, nullptr, ds_ws);
  return attn_bwd_simt(g, dtype, q, k, v, dout, lddo, lse, delta, dq, lddq, dk, lddk, dv, lddv, st);
}

// Backward of attention whose q/k were rotated by RoPE in the projection epilogue
// (cb_gemm_rope): dq / dk come back un-rotated (inverse rotation, reference
// layers.py:235-257).  The tcgen05 kernels fuse the rotation into their dQ / dK stores;
// other engines run cb_rope(inverse) afterwards.
extern "C" int cb_attention_bwd_rope(int batch, int seq_len, int heads, int kv_heads, int head_dim, int dtype,
                                     const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                                     int64_t ldv, const void* o, int64_t ldo, const void* o_lo, const float* lse,
                                     const void* dout, int64_t lddo, float* delta, void* dq, int64_t lddq, void* dk,
                                     int64_t lddk, void* dv, int64_t lddv, float scale, const float* cos_t,
                                     const float* sin_t, void* ds_ws, int64_t ds_bytes, void* stream) {
  AttnGeom g{batch, seq_len, heads, kv_heads, head_dim, ldq, ldk, ldv, ldo, scale};
  if (int s = check_geom(g)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (int s = ds_check(g, ds_ws, ds_bytes)) return s;
  if (tc_bwd_ok(g, dtype, q, k, v, lse, delta, lddo, lddq, lddk, lddv)) {
    if (int s = attn_delta(g, dtype, o, o_lo, dout, lddo, delta, st)) return s;
    return attn_bwd_tc(g, q, k, v, dout, lddo, lse, delta, dq, lddq, dk, lddk, dv, lddv, st, cos_t, sin_t, ds_ws);
  }
  if (int s = cb_attention_bwd(batch, seq_len, heads, kv_heads, head_dim, dtype, q, ldq, k, ldk, v, ldv, o, ldo, o_lo,
                               lse, dout, lddo, delta, dq, lddq, dk, lddk, dv, lddv, scale, nullptr, 0, stream))
    return s;
  const int64_t rows = (int64_t)batch * seq_len;
  if (int s = cb_rope(rows, seq_len, heads, head_dim, dq, lddq, dtype, cos_t, sin_t, 1, stream)) return s;
  return cb_rope(rows, seq_len, kv_heads, head_dim, dk, lddk, dtype, cos_t, sin_t, 1, stream);
}
