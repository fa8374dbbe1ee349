// Shared declarations of the attention engines (attn_tc.cu, attn_tc_bwd.cu, attn_simt.cu,
// attn_api.cu).
#pragma once
#include "common.cuh"

namespace cb {
struct AttnGeom {
  int B, T, H, KVH, hd;
  int64_t ldq, ldk, ldv, ldo;
  float scale;
};
int check_geom(const AttnGeom& g);
int attn_fwd_simt(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v, void* o, float* lse,
                  cudaStream_t st);
// delta = rowsum(dout * (o + o_lo)); o_lo (nullable, bf16) is the bf16 rounding residual of o
// written by the tcgen05 forward, so delta sees o at ~16 significant bits
int attn_delta(const AttnGeom& g, int dtype, const void* o, const void* o_lo, const void* dout, int64_t lddo,
               float* delta, cudaStream_t st);
int attn_bwd_simt(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v, const void* dout,
                  int64_t lddo, const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk,
                  void* dv, int64_t lddv, cudaStream_t st);
bool attn_tc_supported(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v);
int attn_fwd_tc(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, void* o_lo, float* lse,
                cudaStream_t st);
int attn_bwd_tc(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, int64_t lddo,
                const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                int64_t lddv, cudaStream_t st, const float* rope_cos = nullptr, const float* rope_sin = nullptr,
                void* ds_ws = nullptr);
}  // namespace cb
