// Unmasked multi-head attention, SIMT engine (any head_dim, f32 or bf16 I/O, f32 math).
//
// Reference: AttentionBehavior.forward, reference layers.py:331-348 — scores = q k^T/sqrt(hd),
// softmax over ALL keys (no causal mask, reference layers.py:285-286), context = probs @ v.
// Flash-style: the [B,H,T,T] probability tensor the reference materializes is never
// stored; the forward keeps the per-row log-sum-exp and the backward recomputes P.
// Layout: token-major rows (b*T + t), head h at columns [h*hd, (h+1)*hd) of a row with
// stride ld — exactly the projection GEMM's output, so no transposes are needed.
// Grouped-query attention: query head h reads kv head h / (H / KVH) (KVH == H is the
// reference's multi-head case).
//
// This engine serves the f32 parity mode and head dims the tensor-core kernel does not
// instantiate; the bf16 hot path is the tcgen05 engine (attn_tc*.cu).
#include "attn.cuh"
#include "composer_b200.h"

namespace cb {

constexpr int kMaxHd = 256;

// one warp per (b, h, t)
template <typename T>
__global__ void __launch_bounds__(128) attn_fwd_simt_k(AttnGeom g, const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, T* __restrict__ o,
                                                       float* __restrict__ lse) {
  __shared__ float sq[4][kMaxHd];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 4 + warp;
  if (gw >= (int64_t)g.B * g.H * g.T) return;
  const int t = (int)(gw % g.T);
  const int h = (int)((gw / g.T) % g.H);
  const int b = (int)(gw / ((int64_t)g.T * g.H));
  const int kvh = h / (g.H / g.KVH);
  const T* qr = q + ((int64_t)b * g.T + t) * g.ldq + (int64_t)h * g.hd;
  for (int d = lane; d < g.hd; d += 32) sq[warp][d] = to_f32(qr[d]) * g.scale;
  __syncwarp();
  const int nd = (g.hd + 31) / 32;
  float acc[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) acc[i] = 0.f;
  float m = -INFINITY, l = 0.f;
  const T* kb = k + (int64_t)b * g.T * g.ldk + (int64_t)kvh * g.hd;
  const T* vb = v + (int64_t)b * g.T * g.ldv + (int64_t)kvh * g.hd;
  for (int j0 = 0; j0 < g.T; j0 += 32) {
    const int j = j0 + lane;
    float s = -INFINITY;
    if (j < g.T) {
      const T* kr = kb + (int64_t)j * g.ldk;
      s = 0.f;
      for (int d = 0; d < g.hd; ++d) s = fmaf(sq[warp][d], to_f32(kr[d]), s);
    }
    const float mn = fmaxf(m, warp_max(s));
    const float p = (j < g.T) ? __expf(s - mn) : 0.f;
    const float corr = __expf(m - mn);
    l = l * corr + warp_sum(p);
#pragma unroll
    for (int i = 0; i < kMaxHd / 32; ++i) acc[i] *= corr;
    const int cnt = min(32, g.T - j0);
    for (int jj = 0; jj < cnt; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
      const T* vr = vb + (int64_t)(j0 + jj) * g.ldv;
#pragma unroll
      for (int i = 0; i < kMaxHd / 32; ++i) {
        const int d = lane + 32 * i;
        if (i < nd && d < g.hd) acc[i] = fmaf(pj, to_f32(vr[d]), acc[i]);
      }
    }
    m = mn;
  }
  T* orow = o + ((int64_t)b * g.T + t) * g.ldo + (int64_t)h * g.hd;
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) {
    const int d = lane + 32 * i;
    if (i < nd && d < g.hd) orow[d] = from_f32<T>(acc[i] * inv);
  }
  if (lane == 0) lse[((int64_t)b * g.H + h) * g.T + t] = m + logf(l);
}

// delta[b,h,t] = sum_d dO * O
template <typename T>
__global__ void __launch_bounds__(128) attn_delta_k(AttnGeom g, const T* __restrict__ o, const T* __restrict__ dout,
                                                    int64_t lddo, float* __restrict__ delta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 4 + warp;
  if (gw >= (int64_t)g.B * g.H * g.T) return;
  const int t = (int)(gw % g.T);
  const int h = (int)((gw / g.T) % g.H);
  const int b = (int)(gw / ((int64_t)g.T * g.H));
  const T* orow = o + ((int64_t)b * g.T + t) * g.ldo + (int64_t)h * g.hd;
  const T* grow = dout + ((int64_t)b * g.T + t) * lddo + (int64_t)h * g.hd;
  float s = 0.f;
  for (int d = lane; d < g.hd; d += 32) s = fmaf(to_f32(orow[d]), to_f32(grow[d]), s);
  s = warp_sum(s);
  if (lane == 0) delta[((int64_t)b * g.H + h) * g.T + t] = s;
}

// dQ: one warp per (b, h, t)
template <typename T>
__global__ void __launch_bounds__(128) attn_dq_simt_k(AttnGeom g, const T* __restrict__ q, const T* __restrict__ k,
                                                      const T* __restrict__ v, const T* __restrict__ dout, int64_t lddo,
                                                      const float* __restrict__ lse, const float* __restrict__ delta,
                                                      T* __restrict__ dq, int64_t lddq) {
  __shared__ float sq[4][kMaxHd];
  __shared__ float sg[4][kMaxHd];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 4 + warp;
  if (gw >= (int64_t)g.B * g.H * g.T) return;
  const int t = (int)(gw % g.T);
  const int h = (int)((gw / g.T) % g.H);
  const int b = (int)(gw / ((int64_t)g.T * g.H));
  const int kvh = h / (g.H / g.KVH);
  const int64_t row = (int64_t)b * g.T + t;
  for (int d = lane; d < g.hd; d += 32) {
    sq[warp][d] = to_f32(q[row * g.ldq + (int64_t)h * g.hd + d]) * g.scale;
    sg[warp][d] = to_f32(dout[row * lddo + (int64_t)h * g.hd + d]);
  }
  __syncwarp();
  const float L = lse[((int64_t)b * g.H + h) * g.T + t];
  const float D = delta[((int64_t)b * g.H + h) * g.T + t];
  const int nd = (g.hd + 31) / 32;
  float acc[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) acc[i] = 0.f;
  const T* kb = k + (int64_t)b * g.T * g.ldk + (int64_t)kvh * g.hd;
  const T* vb = v + (int64_t)b * g.T * g.ldv + (int64_t)kvh * g.hd;
  for (int j0 = 0; j0 < g.T; j0 += 32) {
    const int j = j0 + lane;
    float ds = 0.f;
    if (j < g.T) {
      const T* kr = kb + (int64_t)j * g.ldk;
      const T* vr = vb + (int64_t)j * g.ldv;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < g.hd; ++d) {
        s = fmaf(sq[warp][d], to_f32(kr[d]), s);
        dp = fmaf(sg[warp][d], to_f32(vr[d]), dp);
      }
      const float p = __expf(s - L);
      ds = p * (dp - D);
    }
    const int cnt = min(32, g.T - j0);
    for (int jj = 0; jj < cnt; ++jj) {
      const float dsj = __shfl_sync(0xffffffffu, ds, jj);
      const T* kr = kb + (int64_t)(j0 + jj) * g.ldk;
#pragma unroll
      for (int i = 0; i < kMaxHd / 32; ++i) {
        const int d = lane + 32 * i;
        if (i < nd && d < g.hd) acc[i] = fmaf(dsj, to_f32(kr[d]), acc[i]);
      }
    }
  }
  T* out = dq + row * lddq + (int64_t)h * g.hd;
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) {
    const int d = lane + 32 * i;
    if (i < nd && d < g.hd) out[d] = from_f32<T>(acc[i] * g.scale);
  }
}

// dK, dV: one warp per (b, kvh, j); sums over every query head of the kv group.
template <typename T>
__global__ void __launch_bounds__(128) attn_dkv_simt_k(AttnGeom g, const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, const T* __restrict__ dout,
                                                       int64_t lddo, const float* __restrict__ lse,
                                                       const float* __restrict__ delta, T* __restrict__ dk,
                                                       int64_t lddk, T* __restrict__ dv, int64_t lddv) {
  __shared__ float sk[4][kMaxHd];
  __shared__ float sv[4][kMaxHd];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 4 + warp;
  if (gw >= (int64_t)g.B * g.KVH * g.T) return;
  const int j = (int)(gw % g.T);
  const int kvh = (int)((gw / g.T) % g.KVH);
  const int b = (int)(gw / ((int64_t)g.T * g.KVH));
  const int group = g.H / g.KVH;
  const int64_t krow = (int64_t)b * g.T + j;
  for (int d = lane; d < g.hd; d += 32) {
    sk[warp][d] = to_f32(k[krow * g.ldk + (int64_t)kvh * g.hd + d]);
    sv[warp][d] = to_f32(v[krow * g.ldv + (int64_t)kvh * g.hd + d]);
  }
  __syncwarp();
  const int nd = (g.hd + 31) / 32;
  float adk[kMaxHd / 32], adv[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) adk[i] = adv[i] = 0.f;
  for (int hh = 0; hh < group; ++hh) {
    const int h = kvh * group + hh;
    const float* lrow = lse + ((int64_t)b * g.H + h) * g.T;
    const float* drow = delta + ((int64_t)b * g.H + h) * g.T;
    for (int i0 = 0; i0 < g.T; i0 += 32) {
      const int i = i0 + lane;
      float p = 0.f, ds = 0.f;
      if (i < g.T) {
        const T* qr = q + ((int64_t)b * g.T + i) * g.ldq + (int64_t)h * g.hd;
        const T* gr = dout + ((int64_t)b * g.T + i) * lddo + (int64_t)h * g.hd;
        float s = 0.f, dp = 0.f;
        for (int d = 0; d < g.hd; ++d) {
          s = fmaf(to_f32(qr[d]), sk[warp][d], s);
          dp = fmaf(to_f32(gr[d]), sv[warp][d], dp);
        }
        p = __expf(s * g.scale - lrow[i]);
        ds = p * (dp - drow[i]);
      }
      const int cnt = min(32, g.T - i0);
      for (int ii = 0; ii < cnt; ++ii) {
        const float pi = __shfl_sync(0xffffffffu, p, ii);
        const float dsi = __shfl_sync(0xffffffffu, ds, ii);
        const T* qr = q + ((int64_t)b * g.T + i0 + ii) * g.ldq + (int64_t)h * g.hd;
        const T* gr = dout + ((int64_t)b * g.T + i0 + ii) * lddo + (int64_t)h * g.hd;
#pragma unroll
        for (int x = 0; x < kMaxHd / 32; ++x) {
          const int d = lane + 32 * x;
          if (x < nd && d < g.hd) {
            adv[x] = fmaf(pi, to_f32(gr[d]), adv[x]);
            adk[x] = fmaf(dsi, to_f32(qr[d]), adk[x]);
          }
        }
      }
    }
  }
  T* ok = dk + krow * lddk + (int64_t)kvh * g.hd;
  T* ov = dv + krow * lddv + (int64_t)kvh * g.hd;
#pragma unroll
  for (int x = 0; x < kMaxHd / 32; ++x) {
    const int d = lane + 32 * x;
    if (x < nd && d < g.hd) {
      ok[d] = from_f32<T>(adk[x] * g.scale);
      ov[d] = from_f32<T>(adv[x]);
    }
  }
}

int check_geom(const AttnGeom& g) {
  if (g.B <= 0 || g.T <= 0 || g.H <= 0 || g.KVH <= 0 || g.hd <= 0)
    return fail(CB_ERR_SHAPE, "attention: non-positive extent");
  if (g.H % g.KVH) return fail(CB_ERR_SHAPE, "attention: heads %d not divisible by kv heads %d", g.H, g.KVH);
  return CB_OK;
}

int attn_fwd_simt(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v, void* o, float* lse,
                  cudaStream_t st) {
  if (g.hd > kMaxHd) return fail(CB_ERR_UNSUPPORTED, "attention: head_dim %d > %d", g.hd, kMaxHd);
  const int64_t warps = (int64_t)g.B * g.H * g.T;
  const int blocks = (int)((warps + 3) / 4);
  if (dtype == CB_DT_F32)
    attn_fwd_simt_k<float><<<blocks, 128, 0, st>>>(g, (const float*)q, (const float*)k, (const float*)v, (float*)o, lse);
  else
    attn_fwd_simt_k<__nv_bfloat16><<<blocks, 128, 0, st>>>(g, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                           (const __nv_bfloat16*)v, (__nv_bfloat16*)o, lse);
  return check_launch("attn_fwd_simt");
}

// delta for bf16 with hd % 8 == 0 and 16-byte aligned rows: hd/8 lanes per row, uint4 loads
__global__ void __launch_bounds__(256) attn_delta_vec_k(AttnGeom g, const __nv_bfloat16* __restrict__ o,
                                                        const __nv_bfloat16* __restrict__ o_lo,
                                                        const __nv_bfloat16* __restrict__ dout, int64_t lddo,
                                                        float* __restrict__ delta, int lanes_per_row) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / lanes_per_row;  // (b*T + t)*H + h
  const int l = (int)(gid - row * lanes_per_row);
  const int64_t total = (int64_t)g.B * g.T * g.H;
  float s = 0.f;
  int h = 0;
  int64_t tok = 0;
  if (row < total) {
    h = (int)(row % g.H);
    tok = row / g.H;
    const uint4 a = *reinterpret_cast<const uint4*>(o + tok * g.ldo + (int64_t)h * g.hd + l * 8);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + tok * lddo + (int64_t)h * g.hd + l * 8);
    const uint4 c = o_lo ? *reinterpret_cast<const uint4*>(o_lo + tok * g.ldo + (int64_t)h * g.hd + l * 8)
                         : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
    const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fa = __bfloat1622float2(pa[i]), fb = __bfloat1622float2(pb[i]), fc = __bfloat1622float2(pc[i]);
      s = fmaf(fa.x + fc.x, fb.x, fmaf(fa.y + fc.y, fb.y, s));
    }
  }
  for (int off = lanes_per_row >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (row < total && l == 0) {
    const int64_t b = tok / g.T, t = tok % g.T;
    delta[(b * g.H + h) * g.T + t] = s;
  }
}

int attn_delta(const AttnGeom& g, int dtype, const void* o, const void* o_lo, const void* dout, int64_t lddo,
               float* delta, cudaStream_t st) {
  const int lpr = g.hd / 8;
  if (dtype == CB_DT_BF16 && g.hd % 8 == 0 && lpr <= 32 && (lpr & (lpr - 1)) == 0 && !((g.ldo | lddo) & 7) &&
      !((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(o_lo) | reinterpret_cast<uintptr_t>(dout)) &
        15)) {
    const int64_t threads = (int64_t)g.B * g.T * g.H * lpr;
    attn_delta_vec_k<<<(int)((threads + 255) / 256), 256, 0, st>>>(
        g, (const __nv_bfloat16*)o, (const __nv_bfloat16*)o_lo, (const __nv_bfloat16*)dout, lddo, delta, lpr);
    return check_launch("attn_delta");
  }
  if (o_lo) return fail(CB_ERR_ARG, "attention delta: o_lo needs bf16, head_dim %% 8 == 0 and 16-byte rows");
  const int64_t warps = (int64_t)g.B * g.H * g.T;
  const int blocks = (int)((warps + 3) / 4);
  if (dtype == CB_DT_F32)
    attn_delta_k<float><<<blocks, 128, 0, st>>>(g, (const float*)o, (const float*)dout, lddo, delta);
  else
    attn_delta_k<__nv_bfloat16><<<blocks, 128, 0, st>>>(g, (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, lddo,
                                                        delta);
  return check_launch("attn_delta");
}

int attn_bwd_simt(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v, const void* dout,
                  int64_t lddo, const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk,
                  void* dv, int64_t lddv, cudaStream_t st) {
  if (g.hd > kMaxHd) return fail(CB_ERR_UNSUPPORTED, "attention: head_dim %d > %d", g.hd, kMaxHd);
  const int64_t wq = (int64_t)g.B * g.H * g.T, wk = (int64_t)g.B * g.KVH * g.T;
  if (dtype == CB_DT_F32) {
    attn_dq_simt_k<float><<<(int)((wq + 3) / 4), 128, 0, st>>>(g, (const float*)q, (const float*)k, (const float*)v,
                                                               (const float*)dout, lddo, lse, delta, (float*)dq, lddq);
    attn_dkv_simt_k<float><<<(int)((wk + 3) / 4), 128, 0, st>>>(g, (const float*)q, (const float*)k, (const float*)v,
                                                                (const float*)dout, lddo, lse, delta, (float*)dk, lddk,
                                                                (float*)dv, lddv);
  } else {
    using B = __nv_bfloat16;
    attn_dq_simt_k<B><<<(int)((wq + 3) / 4), 128, 0, st>>>(g, (const B*)q, (const B*)k, (const B*)v, (const B*)dout,
                                                           lddo, lse, delta, (B*)dq, lddq);
    attn_dkv_simt_k<B><<<(int)((wk + 3) / 4), 128, 0, st>>>(g, (const B*)q, (const B*)k, (const B*)v, (const B*)dout,
                                                            lddo, lse, delta, (B*)dk, lddk, (B*)dv, lddv);
  }
  return check_launch("attn_bwd_simt", 2);
}

}  // namespace cb
