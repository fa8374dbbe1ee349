// Fused AdamW update over a flat parameter shard.
//
// The reference carries only the optimizer's configuration (reference layers.py:657-663,
// 778-782: fn:adamw with lr, beta1=0.9, beta2=0.999) and never applies it.  This kernel
// is the update those fields describe, with the documented extra hyper-parameters
// (eps=1e-8, decoupled weight decay wd=0 by default, bias correction at step t):
//   g   = grad * grad_scale
//   m   = b1*m + (1-b1)*g ;  v = b2*v + (1-b2)*g^2
//   p  -= lr * ( (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps) + wd*p )
// One pass: reads p, g, m, v (f32), writes p, m, v and (optionally) the bf16 working
// copy the GEMMs read — 30 bytes per parameter of HBM traffic.
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

__global__ void __launch_bounds__(256) adamw_k(int64_t n, float* __restrict__ p, const float* __restrict__ g,
                                               float* __restrict__ m, float* __restrict__ v,
                                               __nv_bfloat16* __restrict__ pbf, float lr, float b1, float b2,
                                               float eps, float wd, float bc1, float bc2, float gs) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 P = reinterpret_cast<float4*>(p)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float4 M = reinterpret_cast<float4*>(m)[i];
    float4 V = reinterpret_cast<float4*>(v)[i];
    float* pp = &P.x;
    const float* gg = &G.x;
    float* mm = &M.x;
    float* vv = &V.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) adam_elem(pp[j], __fmul_rn(gg[j], gs), mm[j], vv[j], lr, b1, b2, eps, wd, bc1, bc2);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = M;
    reinterpret_cast<float4*>(v)[i] = V;
    if (pbf) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pbf)[i] = pk;
    }
  }
  // tail
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float pi = p[i], mi = m[i], vi = v[i];
    adam_elem(pi, __fmul_rn(g[i], gs), mi, vi, lr, b1, b2, eps, wd, bc1, bc2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (pbf) pbf[i] = __float2bfloat16_rn(pi);
  }
}

// AdamW whose gradient is the in-order sum of the FSDP reduce-scatter's parts (this rank's
// slice of every rank's gradient, cb_sum_parts' operands): g = scale * (p0 + p1 + ...),
// exactly cb_sum_parts' arithmetic, so the result is bit-identical to sum_parts + adamw while
// the summed gradient never round-trips through HBM (optionally still stored to g_out).
struct Parts {
  const float* p[8];
};

__global__ void __launch_bounds__(256) adamw_parts_k(int64_t n4, Parts s, int nparts, float scale,
                                                     float* __restrict__ g_out, float* __restrict__ p,
                                                     float* __restrict__ m, float* __restrict__ v,
                                                     __nv_bfloat16* __restrict__ pbf, float lr, float b1, float b2,
                                                     float eps, float wd, float bc1, float bc2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 G = __ldcs(reinterpret_cast<const float4*>(s.p[0]) + i);
    for (int q = 1; q < nparts; ++q) {
      const float4 b = __ldcs(reinterpret_cast<const float4*>(s.p[q]) + i);
      G.x += b.x;
      G.y += b.y;
      G.z += b.z;
      G.w += b.w;
    }
    G.x *= scale;
    G.y *= scale;
    G.z *= scale;
    G.w *= scale;
    if (g_out) reinterpret_cast<float4*>(g_out)[i] = G;
    float4 P = reinterpret_cast<float4*>(p)[i];
    float4 M = reinterpret_cast<float4*>(m)[i];
    float4 V = reinterpret_cast<float4*>(v)[i];
    float* pp = &P.x;
    const float* gg = &G.x;
    float* mm = &M.x;
    float* vv = &V.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) adam_elem(pp[j], __fmul_rn(gg[j], 1.f), mm[j], vv[j], lr, b1, b2, eps, wd, bc1, bc2);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = M;
    reinterpret_cast<float4*>(v)[i] = V;
    if (pbf) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(pbf)[i] = pk;
    }
  }
}

}  // namespace cb

using namespace cb;

extern "C" int cb_adamw_parts(int64_t n, int nparts, const void* parts, float scale, float* grad_out, float* param,
                              float* exp_avg, float* exp_avg_sq, void* param_bf16, float lr, float beta1, float beta2,
                              float eps, float weight_decay, int step, void* stream) {
  if (n <= 0) return CB_OK;
  if (step < 1) return fail(CB_ERR_ARG, "adamw_parts: step must be >= 1");
  if (nparts < 1 || nparts > 8) return fail(CB_ERR_SHAPE, "adamw_parts: nparts %d not in [1, 8]", nparts);
  if (n % 4) return fail(CB_ERR_SHAPE, "adamw_parts: n %lld not a multiple of 4", (long long)n);
  Parts s{};
  const float* const* hp = reinterpret_cast<const float* const*>(parts);
  uintptr_t al = reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(exp_avg) |
                 reinterpret_cast<uintptr_t>(exp_avg_sq) | reinterpret_cast<uintptr_t>(grad_out);
  for (int q = 0; q < nparts; ++q) {
    s.p[q] = hp[q];
    al |= reinterpret_cast<uintptr_t>(hp[q]);
  }
  if (al & 15) return fail(CB_ERR_ARG, "adamw_parts: buffers must be 16-byte aligned");
  if (param_bf16 && (reinterpret_cast<uintptr_t>(param_bf16) & 7))
    return fail(CB_ERR_ARG, "adamw_parts: bf16 copy must be 8-byte aligned");
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  const int64_t n4 = n / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  adamw_parts_k<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(n4, s, nparts, scale, grad_out, param, exp_avg,
                                                               exp_avg_sq, (__nv_bfloat16*)param_bf16, lr, beta1,
                                                               beta2, eps, weight_decay, (float)bc1, (float)bc2);
  return check_launch("adamw_parts");
}

extern "C" int cb_adamw(int64_t n, float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                        void* param_bf16, float lr, float beta1, float beta2, float eps, float weight_decay,
                        int step, float grad_scale, void* stream) {
  if (n <= 0) return CB_OK;
  if (step < 1) return fail(CB_ERR_ARG, "adamw: step must be >= 1");
  if ((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(exp_avg) |
       reinterpret_cast<uintptr_t>(exp_avg_sq)) & 15)
    return fail(CB_ERR_ARG, "adamw: buffers must be 16-byte aligned");
  if (param_bf16 && (reinterpret_cast<uintptr_t>(param_bf16) & 7)) return fail(CB_ERR_ARG, "adamw: bf16 copy must be 8-byte aligned");
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  adamw_k<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(n, param, grad, exp_avg, exp_avg_sq,
                                                         (__nv_bfloat16*)param_bf16, lr, beta1, beta2, eps,
                                                         weight_decay, (float)bc1, (float)bc2, grad_scale);
  return check_launch("adamw");
}
