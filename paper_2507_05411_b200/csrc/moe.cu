// Mixture-of-experts routing, dispatch and combine (reference layers.py:422-533).
//
//  cb_moe_route     probs = softmax(x @ router) computed in f64 per token (one warp per
//                   token: for E <= 8 every lane accumulates all experts over a column
//                   slice, lanes summed in a fixed order), stable top-k by (prob desc, id asc) —
//                   exactly argsort(-probs, kind="stable")[:k] (layers.py:437) — and the
//                   renormalized gate weights picked/sum(picked) (layers.py:440).  Router
//                   inputs that are bit-identical to the reference's give bit-identical
//                   expert assignments (f64 logits).
//  cb_moe_stats     load_balance_loss = E * sum_e f_e * mean_p_e (layers.py:441-449),
//                   deterministic single-CTA reduction (summary only, not in the loss).
//  cb_gather_rows   dispatch: rows of x into expert-sorted order (perm from cb_sort_ids).
//  cb_moe_combine   out[t] = sum_slot w[t,slot] * y[pos(t,slot)] in slot order (layers.py:529-531).
//  cb_moe_combine_bwd / cb_moe_router_bwd: the reverse of combine, renormalization and softmax.
#include <algorithm>

#include "common.cuh"
#include "composer_b200.h"

namespace cb {

constexpr int kMaxExperts = 32;

template <typename TX>
__global__ void __launch_bounds__(128) moe_route_k(int64_t n, int d, int E, int k, const TX* __restrict__ x, int64_t ldx,
                                                   const float* __restrict__ router, int32_t* __restrict__ idx,
                                                   float* __restrict__ w, float* __restrict__ probs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 4 + warp;
  if (t >= n) return;
  const TX* xr = x + t * ldx;
  double logit = -INFINITY;
  if (lane < E) {
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = fma((double)to_f32(xr[c]), (double)router[(int64_t)c * E + lane], acc);
    logit = acc;
  }
  double mx = logit;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double e = lane < E ? exp(logit - mx) : 0.0;
  double s = e;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double p = e / s;
  if (lane < E) probs[t * E + lane] = (float)p;
  // stable top-k: repeatedly take (max prob, lowest id)
  bool taken = lane >= E;
  double picked[kMaxExperts];
  int pid[kMaxExperts];
  double psum = 0.0;
  for (int j = 0; j < k; ++j) {
    double bv = taken ? -1.0 : p;
    int bi = taken ? 1 << 30 : lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == bi) taken = true;
    picked[j] = bv;
    pid[j] = bi;
    psum += bv;
  }
  if (lane == 0) {
    for (int j = 0; j < k; ++j) {
      idx[t * k + j] = pid[j];
      w[t * k + j] = (float)(picked[j] / psum);
    }
  }
}

// E <= 8 experts, bf16 x, d % 256 == 0: the router matrix widened to f64 once per CTA into
// shared memory (128 KB at d = 2048), one warp per group of kRouteTok tokens.  Lane l owns
// columns 256 i + 8 l + u (u < 8): a 16-byte load brings 8 of a token's bf16 values, and the
// router is stored as [i][u][expert pair][lane] (16 B per entry) so every shared-memory read of
// a warp is 512 contiguous bytes (conflict-free).  Each lane accumulates a fixed-order f64 fma
// chain over its columns, then a fixed-order f64 butterfly across lanes — the same logits on
// every run; top-k bit-exactness against the reference holds as for any f64 summation order
// (ties resolved on identical logits).  The one-token-per-warp f32-staged form spent 9 f32->f64
// conversions and a 2-byte load per 8 DFMA.  Softmax / stable top-k / renormalisation as
// moe_route_k.  Grid-stride over token groups, one CTA per SM.
constexpr int kRouteWarps = 8;
constexpr int kRouteTok = 4;

__device__ __forceinline__ void route_finish(double (&acc)[8], int64_t t, int E, int k, int lane,
                                             int32_t* __restrict__ idx, float* __restrict__ w,
                                             float* __restrict__ probs) {
  double logit = -INFINITY;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (lane == e && e < E) logit = acc[e];
  }
  double mx = logit;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double ex = lane < E ? exp(logit - mx) : 0.0;
  double sum = ex;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double pr = ex / sum;
  if (lane < E) probs[t * E + lane] = (float)pr;
  // stable top-k: repeatedly take (max prob, lowest id); k <= 8
  bool taken = lane >= E;
  double picked[8];
  int pid[8];
  double psum = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    double bv = taken ? -1.0 : pr;
    int bi = taken ? 1 << 30 : lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == bi) taken = true;
    picked[j] = bv;
    pid[j] = bi;
    psum += bv;
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= k) break;
      idx[t * k + j] = pid[j];
      w[t * k + j] = (float)(picked[j] / psum);
    }
  }
}

__global__ void __launch_bounds__(kRouteWarps * 32) moe_route8_k(int64_t n, int d, int E, int k,
                                                                  const __nv_bfloat16* __restrict__ x, int64_t ldx,
                                                                  const float* __restrict__ router,
                                                                  int32_t* __restrict__ idx, float* __restrict__ w,
                                                                  float* __restrict__ probs) {
  extern __shared__ double2 rsm2[];  // [d/256][8 u][4 expert pairs][32 lanes]
  for (int i = threadIdx.x; i < d * 4; i += blockDim.x) {
    const int c = i >> 2, ep = i & 3;  // column, expert pair
    const int blk = c >> 8, l = (c >> 3) & 31, u = c & 7;
    const int e0 = 2 * ep, e1 = e0 + 1;
    rsm2[((blk * 8 + u) * 4 + ep) * 32 + l] =
        make_double2(e0 < E ? (double)router[(int64_t)c * E + e0] : 0.0, e1 < E ? (double)router[(int64_t)c * E + e1] : 0.0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = d >> 8;
  const int64_t groups = (n + kRouteTok - 1) / kRouteTok;
  for (int64_t g = (int64_t)blockIdx.x * kRouteWarps + warp; g < groups; g += (int64_t)gridDim.x * kRouteWarps) {
    const int64_t t0 = g * kRouteTok;
    const int nt = (int)min((int64_t)kRouteTok, n - t0);
    const uint4* xr[kRouteTok];
#pragma unroll
    for (int q = 0; q < kRouteTok; ++q)  // tail: re-read token t0
      xr[q] = reinterpret_cast<const uint4*>(x + (t0 + (q < nt ? q : 0)) * ldx) + lane;
    double acc[kRouteTok][8];
#pragma unroll
    for (int q = 0; q < kRouteTok; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[q][e] = 0.0;
#pragma unroll 1
    for (int blk = 0; blk < nblk; ++blk) {
      uint4 xv[kRouteTok];
#pragma unroll
      for (int q = 0; q < kRouteTok; ++q) xv[q] = xr[q][blk * 32];
      const double2* rb = rsm2 + blk * 8 * 4 * 32 + lane;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 r01 = rb[(u * 4 + 0) * 32], r23 = rb[(u * 4 + 1) * 32];
        const double2 r45 = rb[(u * 4 + 2) * 32], r67 = rb[(u * 4 + 3) * 32];
#pragma unroll
        for (int q = 0; q < kRouteTok; ++q) {
          const uint32_t word = (&xv[q].x)[u >> 1];
          const double xd = (double)__uint_as_float((u & 1) ? (word & 0xffff0000u) : (word << 16));
          acc[q][0] = fma(xd, r01.x, acc[q][0]);
          acc[q][1] = fma(xd, r01.y, acc[q][1]);
          acc[q][2] = fma(xd, r23.x, acc[q][2]);
          acc[q][3] = fma(xd, r23.y, acc[q][3]);
          acc[q][4] = fma(xd, r45.x, acc[q][4]);
          acc[q][5] = fma(xd, r45.y, acc[q][5]);
          acc[q][6] = fma(xd, r67.x, acc[q][6]);
          acc[q][7] = fma(xd, r67.y, acc[q][7]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kRouteTok; ++q)
      if (q < nt) route_finish(acc[q], t0 + q, E, k, lane, idx, w, probs);
  }
}

// NE: compile-time expert bound (8 or kMaxExperts) so the per-thread sums and counts stay in
// registers (a runtime-indexed count array lived in local memory: 50 us per call at 16K tokens)
template <int NE>
__global__ void __launch_bounds__(1024) moe_stats_k(int64_t n, int E, int k, const int32_t* __restrict__ idx,
                                                    const float* __restrict__ probs, double* __restrict__ out) {
  __shared__ double psum[kMaxExperts][33];
  __shared__ int cnt[kMaxExperts][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // each warp accumulates a strided subset of tokens in fixed order -> deterministic
  double ps[NE];
  int cs[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    ps[e] = 0.0;
    cs[e] = 0;
  }
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e < E) ps[e] += (double)probs[t * E + e];
    for (int j = 0; j < k; ++j) {
      const int id = idx[t * k + j];
#pragma unroll
      for (int e = 0; e < NE; ++e) cs[e] += id == e;
    }
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    if (e >= E) break;
    double v = ps[e];
    int c = cs[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      psum[e][warp] = v;
      cnt[e][warp] = c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    double lbl = 0.0;
    for (int e = 0; e < E; ++e) {
      double p = 0.0;
      long long c = 0;
      for (int w2 = 0; w2 < nw; ++w2) {
        p += psum[e][w2];
        c += cnt[e][w2];
      }
      const double f = (double)c / (double)(n * k);
      lbl += f * (p / (double)n);
      out[1 + e] = (double)c;
      out[1 + E + e] = p / (double)n;
    }
    out[0] = (double)E * lbl;
  }
}

template <typename T>
__global__ void gather_rows_k(int64_t n, int d, const int32_t* __restrict__ perm, int div, const T* __restrict__ x,
                              int64_t ldx, T* __restrict__ out, int64_t ldo) {
  const int64_t r = blockIdx.x;
  if (r >= n) return;
  const int64_t src = perm[r] / div;
  for (int c = threadIdx.x; c < d; c += blockDim.x) out[r * ldo + c] = x[src * ldx + c];
}

// out[t] (+)= sum_j w[t,j] * y[inv[t*k+j]]  (w == NULL -> weights 1)
template <typename TY>
__global__ void combine_k(int64_t n, int d, int k, const int32_t* __restrict__ inv, const float* __restrict__ w,
                          const TY* __restrict__ y, int64_t ldy, float* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t t = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < k; ++j) {
      const float wj = w ? w[t * k + j] : 1.f;
      acc += wj * to_f32(y[(int64_t)inv[t * k + j] * ldy + c]);
    }
    out[t * ldo + c] = accumulate ? out[t * ldo + c] + acc : acc;
  }
}

// Vectorized forms (f32 y / dout, d % 4 == 0, 16-byte aligned rows): one warp per token,
// float4 loads — the scalar block-per-token kernels above moved ~1/10 of HBM bandwidth
__global__ void __launch_bounds__(256) combine_v4_k(int64_t n, int d4, int k, const int32_t* __restrict__ inv,
                                                    const float* __restrict__ w, const float* __restrict__ y,
                                                    int64_t ldy, float* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= n) return;
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < d4; c += 32) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float wj = w ? w[t * k + j] : 1.f;
      const float4 v = reinterpret_cast<const float4*>(y + (int64_t)inv[t * k + j] * ldy)[c];
      acc.x += wj * v.x;
      acc.y += wj * v.y;
      acc.z += wj * v.z;
      acc.w += wj * v.w;
    }
    float4* o = reinterpret_cast<float4*>(out + t * ldo) + c;
    if (accumulate) {
      const float4 p = *o;
      acc.x = p.x + acc.x;
      acc.y = p.y + acc.y;
      acc.z = p.z + acc.z;
      acc.w = p.w + acc.w;
    }
    *o = acc;
  }
}

// out[t] = res[t] + sum_j w[t,j] * y[inv[t*k+j]]: the MoE block's residual add fused into the
// combine (one pass over the residual instead of a combine pass plus an add pass); the same
// bits as combine then add (float addition commutes)
__global__ void __launch_bounds__(256) combine_res_v4_k(int64_t n, int d4, int k, const int32_t* __restrict__ inv,
                                                        const float* __restrict__ w, const float* __restrict__ y,
                                                        int64_t ldy, const float* __restrict__ res, int64_t ldr,
                                                        float* __restrict__ out, int64_t ldo) {
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= n) return;
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < d4; c += 32) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float wj = w[t * k + j];
      const float4 v = reinterpret_cast<const float4*>(y + (int64_t)inv[t * k + j] * ldy)[c];
      acc.x += wj * v.x;
      acc.y += wj * v.y;
      acc.z += wj * v.z;
      acc.w += wj * v.w;
    }
    const float4 p = reinterpret_cast<const float4*>(res + t * ldr)[c];
    reinterpret_cast<float4*>(out + t * ldo)[c] = make_float4(p.x + acc.x, p.y + acc.y, p.z + acc.z, p.w + acc.w);
  }
}

template <typename TG>
__device__ __forceinline__ void store4(TG* dst, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* dst, float4 v) {
  *reinterpret_cast<float4*>(dst) = v;
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* dst, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst) = u;
}

// One warp per token; the token's dout row is read once for all k slots (k <= 8), in chunks of
// kCbChunk float4 per lane whose loads are all issued before their use (the one-float4-at-a-
// time loop was load-latency bound at ~3.4 TB/s).  Each dw[t,j] still accumulates over the
// columns in ascending order, as in the scalar kernel.
constexpr int kCbChunk = 8;
template <typename TG>
__global__ void __launch_bounds__(256) combine_bwd_v4_k(int64_t n, int d4, int k, const int32_t* __restrict__ inv,
                                                        const float* __restrict__ w, const float* __restrict__ y,
                                                        int64_t ldy, const float* __restrict__ dout, int64_t lddo,
                                                        TG* __restrict__ dy, int64_t lddy, float* __restrict__ dw) {
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= n) return;
  const int lane = threadIdx.x & 31;
  const float4* g4 = reinterpret_cast<const float4*>(dout + t * lddo);
  float dot[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) dot[j] = 0.f;
  for (int c0 = 0; c0 < d4; c0 += 32 * kCbChunk) {
    float4 g[kCbChunk];
#pragma unroll
    for (int i = 0; i < kCbChunk; ++i) {
      const int c = c0 + i * 32 + lane;
      g[i] = c < d4 ? g4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= k) break;
      const int64_t r = inv[t * k + j];
      const float wj = w[t * k + j];
      const float4* y4 = reinterpret_cast<const float4*>(y + r * ldy);
      float4 v[kCbChunk];
#pragma unroll
      for (int i = 0; i < kCbChunk; ++i) {
        const int c = c0 + i * 32 + lane;
        v[i] = c < d4 ? y4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < kCbChunk; ++i) {
        const int c = c0 + i * 32 + lane;
        if (c < d4) {
          store4<TG>(dy + r * lddy + 4 * c, make_float4(wj * g[i].x, wj * g[i].y, wj * g[i].z, wj * g[i].w));
          dot[j] = fmaf(g[i].x, v[i].x, fmaf(g[i].y, v[i].y, fmaf(g[i].z, v[i].z, fmaf(g[i].w, v[i].w, dot[j]))));
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j < k) {
      const float s = warp_sum(dot[j]);
      if (lane == 0) dw[t * k + j] = s;
    }
  }
}

// dy[inv[t*k+j]] = w[t,j] * dout[t] ;  dw[t,j] = dout[t] . y[inv[t*k+j]]
template <typename TG>
__global__ void __launch_bounds__(256) combine_bwd_k(int64_t n, int d, int k, const int32_t* __restrict__ inv,
                                                     const float* __restrict__ w, const float* __restrict__ y,
                                                     int64_t ldy, const float* __restrict__ dout, int64_t lddo,
                                                     TG* __restrict__ dy, int64_t lddy, float* __restrict__ dw) {
  __shared__ float red[32];
  const int64_t t = blockIdx.x;
  for (int j = 0; j < k; ++j) {
    const int64_t r = inv[t * k + j];
    const float wj = w[t * k + j];
    float dot = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      const float g = dout[t * lddo + c];
      dy[r * lddy + c] = from_f32<TG>(wj * g);
      dot = fmaf(g, y[r * ldy + c], dot);
    }
    dot = block_sum(dot, red);
    if (threadIdx.x == 0) dw[t * k + j] = dot;
  }
}

// gradient of w = renorm(top-k(softmax(logits))) w.r.t. the logits
__global__ void moe_router_bwd_k(int64_t n, int E, int k, const float* __restrict__ probs,
                                 const int32_t* __restrict__ idx, const float* __restrict__ w,
                                 const float* __restrict__ dw, float* __restrict__ dlogits) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  float dp[kMaxExperts];
  for (int e = 0; e < E; ++e) dp[e] = 0.f;
  float S = 0.f, wdw = 0.f;
  for (int j = 0; j < k; ++j) {
    S += probs[t * E + idx[t * k + j]];
    wdw += w[t * k + j] * dw[t * k + j];
  }
  for (int j = 0; j < k; ++j) dp[idx[t * k + j]] += (dw[t * k + j] - wdw) / S;
  float pdp = 0.f;
  for (int e = 0; e < E; ++e) pdp += probs[t * E + e] * dp[e];
  for (int e = 0; e < E; ++e) dlogits[t * E + e] = probs[t * E + e] * (dp[e] - pdp);
}

}  // namespace cb

using namespace cb;

extern "C" int cb_moe_route(int64_t n, int dim, int experts, int top_k, const void* x, int64_t ldx, int x_dtype,
                            const float* router, int32_t* idx, float* weights, float* probs, void* stream) {
  if (experts < 1 || experts > kMaxExperts) return fail(CB_ERR_UNSUPPORTED, "moe: experts must be in [1, %d]", kMaxExperts);
  if (top_k < 1 || top_k > experts) return fail(CB_ERR_SHAPE, "top_k=%d must lie in [1, %d]", top_k, experts);
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t rsm_bytes = (size_t)dim * 8 * sizeof(double);
  if (x_dtype == CB_DT_BF16 && experts <= 8 && dim % 256 == 0 && ldx % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && rsm_bytes <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(moe_route8_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int64_t need = (n + kRouteWarps * kRouteTok - 1) / (kRouteWarps * kRouteTok);
    const int blocks8 = (int)std::min<int64_t>(need, kNumSMs);
    moe_route8_k<<<blocks8, kRouteWarps * 32, rsm_bytes, st>>>(n, dim, experts, top_k, (const __nv_bfloat16*)x, ldx,
                                                               router, idx, weights, probs);
    return check_launch("moe_route8");
  }
  const int blocks = (int)((n + 3) / 4);
  if (x_dtype == CB_DT_F32)
    moe_route_k<float><<<blocks, 128, 0, st>>>(n, dim, experts, top_k, (const float*)x, ldx, router, idx, weights, probs);
  else
    moe_route_k<__nv_bfloat16><<<blocks, 128, 0, st>>>(n, dim, experts, top_k, (const __nv_bfloat16*)x, ldx, router, idx,
                                                       weights, probs);
  return check_launch("moe_route");
}

// out f64[1 + 2E]: [load_balance_loss, counts_e..., mean_probs_e...]
extern "C" int cb_moe_stats(int64_t n, int experts, int top_k, const int32_t* idx, const float* probs, double* out,
                            void* stream) {
  if (n <= 0) return CB_OK;
  if (experts <= 8)
    moe_stats_k<8><<<1, 1024, 0, (cudaStream_t)stream>>>(n, experts, top_k, idx, probs, out);
  else
    moe_stats_k<kMaxExperts><<<1, 1024, 0, (cudaStream_t)stream>>>(n, experts, top_k, idx, probs, out);
  return check_launch("moe_stats");
}

extern "C" int cb_gather_rows(int64_t n, int dim, const int32_t* perm, int div, const void* x, int64_t ldx, void* out,
                              int64_t ldo, int dtype, void* stream) {
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32)
    gather_rows_k<float><<<n, 256, 0, st>>>(n, dim, perm, div, (const float*)x, ldx, (float*)out, ldo);
  else
    gather_rows_k<__nv_bfloat16><<<n, 256, 0, st>>>(n, dim, perm, div, (const __nv_bfloat16*)x, ldx,
                                                    (__nv_bfloat16*)out, ldo);
  return check_launch("gather_rows");
}

extern "C" int cb_moe_combine(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights, const void* y,
                              int64_t ldy, int y_dtype, float* out, int64_t ldo, int accumulate, void* stream) {
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool v4 = y_dtype == CB_DT_F32 && dim % 4 == 0 && ((ldy | ldo) & 3) == 0 &&
                  !((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(out)) & 15);
  if (v4) {
    combine_v4_k<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, dim / 4, top_k, inv, weights, (const float*)y, ldy, out,
                                                          ldo, accumulate);
    return check_launch("moe_combine");
  }
  if (y_dtype == CB_DT_F32)
    combine_k<float><<<n, 256, 0, st>>>(n, dim, top_k, inv, weights, (const float*)y, ldy, out, ldo, accumulate);
  else
    combine_k<__nv_bfloat16><<<n, 256, 0, st>>>(n, dim, top_k, inv, weights, (const __nv_bfloat16*)y, ldy, out, ldo,
                                                accumulate);
  return check_launch("moe_combine");
}

extern "C" int cb_moe_combine_residual(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights,
                                       const float* y, int64_t ldy, const float* res, int64_t ldr, float* out,
                                       int64_t ldo, void* stream) {
  if (n <= 0) return CB_OK;
  if (!weights || dim % 4 || ((ldy | ldr | ldo) & 3) ||
      ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(res) | reinterpret_cast<uintptr_t>(out)) & 15))
    return fail(CB_ERR_UNSUPPORTED, "moe_combine_residual: needs f32 16-byte aligned rows, dim %% 4 == 0");
  combine_res_v4_k<<<(unsigned)((n + 7) / 8), 256, 0, (cudaStream_t)stream>>>(n, dim / 4, top_k, inv, weights, y, ldy,
                                                                              res, ldr, out, ldo);
  return check_launch("moe_combine_residual");
}

extern "C" int cb_moe_combine_bwd(int64_t n, int dim, int top_k, const int32_t* inv, const float* weights,
                                  const float* y, int64_t ldy, const float* dout, int64_t lddo, void* dy, int64_t lddy,
                                  int dy_dtype, float* dweights, void* stream) {
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool v4 = top_k <= 8 && dim % 4 == 0 && ((ldy | lddo | lddy) & 3) == 0 &&
                  !((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(dout) |
                     reinterpret_cast<uintptr_t>(dy)) & (dy_dtype == CB_DT_F32 ? 15 : 7)) &&
                  !(reinterpret_cast<uintptr_t>(y) & 15) && !(reinterpret_cast<uintptr_t>(dout) & 15);
  if (v4) {
    const unsigned blocks = (unsigned)((n + 7) / 8);
    if (dy_dtype == CB_DT_F32)
      combine_bwd_v4_k<float><<<blocks, 256, 0, st>>>(n, dim / 4, top_k, inv, weights, y, ldy, dout, lddo, (float*)dy,
                                                      lddy, dweights);
    else
      combine_bwd_v4_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(n, dim / 4, top_k, inv, weights, y, ldy, dout, lddo,
                                                              (__nv_bfloat16*)dy, lddy, dweights);
    return check_launch("moe_combine_bwd");
  }
  if (dy_dtype == CB_DT_F32)
    combine_bwd_k<float><<<n, 256, 0, st>>>(n, dim, top_k, inv, weights, y, ldy, dout, lddo, (float*)dy, lddy, dweights);
  else
    combine_bwd_k<__nv_bfloat16><<<n, 256, 0, st>>>(n, dim, top_k, inv, weights, y, ldy, dout, lddo,
                                                    (__nv_bfloat16*)dy, lddy, dweights);
  return check_launch("moe_combine_bwd");
}

extern "C" int cb_moe_router_bwd(int64_t n, int experts, int top_k, const float* probs, const int32_t* idx,
                                 const float* weights, const float* dweights, float* dlogits, void* stream) {
  if (n <= 0) return CB_OK;
  moe_router_bwd_k<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, experts, top_k, probs, idx, weights,
                                                                            dweights, dlogits);
  return check_launch("moe_router_bwd");
}

// Router backward products, E <= 32 experts (tiny N/K that GEMM tiles waste):
//   partial[blk][c*E + e] = sum_{t in blk's tokens} x[t][c] * dlog[t][e]   (then col-reduce)
//   dx[t][c] += sum_e dlog[t][e] * router[c][e]
// NE: compile-time expert bound (8 or kMaxExperts) so the per-expert loops unroll to E.
template <typename TX, int NE>
__global__ void __launch_bounds__(256) router_wgrad_k(int64_t n, int d, int E, int tok_per_blk,
                                                      const TX* __restrict__ x, int64_t ldx,
                                                      const float* __restrict__ dlog, float* __restrict__ partial) {
  __shared__ __align__(16) float sg[64][NE];
  const int64_t t0 = (int64_t)blockIdx.x * tok_per_blk;
  const int64_t t1 = min(n, t0 + tok_per_blk);
  const int c0 = blockIdx.y * 256 + threadIdx.x;  // this thread's column
  float acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.f;
  for (int64_t tb = t0; tb < t1; tb += 64) {
    const int cnt = (int)(t1 - tb < 64 ? t1 - tb : 64);
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * NE; i += blockDim.x) {
      const int j = i / NE, e = i % NE;
      sg[j][e] = (j < cnt && e < E) ? dlog[(tb + j) * E + e] : 0.f;
    }
    __syncthreads();
    if (c0 < d) {
#pragma unroll 4
      for (int j = 0; j < cnt; ++j) {
        const float xv = to_f32(x[(tb + j) * ldx + c0]);
#pragma unroll
        for (int e = 0; e < NE; e += 4) {
          const float4 g = *reinterpret_cast<const float4*>(&sg[j][e]);
          acc[e] = fmaf(xv, g.x, acc[e]);
          acc[e + 1] = fmaf(xv, g.y, acc[e + 1]);
          acc[e + 2] = fmaf(xv, g.z, acc[e + 2]);
          acc[e + 3] = fmaf(xv, g.w, acc[e + 3]);
        }
      }
    }
  }
  if (c0 < d) {
    float* pr = partial + (int64_t)blockIdx.x * d * E + (int64_t)c0 * E;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (e < E) pr[e] = acc[e];
  }
}

template <int NE>
__global__ void __launch_bounds__(256) router_dx_k(int64_t n, int d, int E, const float* __restrict__ dlog,
                                                   const float* __restrict__ router, float* __restrict__ dx,
                                                   int64_t lddx) {
  const int64_t t = blockIdx.x;
  float g[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) g[e] = e < E ? dlog[t * E + e] : 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    if (NE == 8 && E == 8) {  // one 32-byte router row
      const float4 r0 = *reinterpret_cast<const float4*>(router + (int64_t)c * 8);
      const float4 r1 = *reinterpret_cast<const float4*>(router + (int64_t)c * 8 + 4);
      s = fmaf(g[0], r0.x, s);
      s = fmaf(g[1], r0.y, s);
      s = fmaf(g[2], r0.z, s);
      s = fmaf(g[3], r0.w, s);
      s = fmaf(g[4], r1.x, s);
      s = fmaf(g[5], r1.y, s);
      s = fmaf(g[6], r1.z, s);
      s = fmaf(g[7], r1.w, s);
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (e < E) s = fmaf(g[e], router[(int64_t)c * E + e], s);
    }
    dx[t * lddx + c] += s;
  }
}

// E == 8, d % 4 == 0, 16-byte aligned rows: a thread owns 4 columns (their 32 router values in
// registers) for a block of tokens, so the router is read once per block instead of once per
// token and column; each element's sum is the same e-ordered fma chain as router_dx_k.
constexpr int kRouterDxTok = 64;
__global__ void __launch_bounds__(256) router_dx_v4_k(int64_t n, int d, const float* __restrict__ dlog,
                                                      const float* __restrict__ router, float* __restrict__ dx,
                                                      int64_t lddx) {
  const int c = (blockIdx.y * 256 + threadIdx.x) * 4;
  if (c >= d) return;
  float r[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 a = *reinterpret_cast<const float4*>(router + (int64_t)(c + q) * 8);
    const float4 b = *reinterpret_cast<const float4*>(router + (int64_t)(c + q) * 8 + 4);
    r[q][0] = a.x, r[q][1] = a.y, r[q][2] = a.z, r[q][3] = a.w;
    r[q][4] = b.x, r[q][5] = b.y, r[q][6] = b.z, r[q][7] = b.w;
  }
  const int64_t t0 = (int64_t)blockIdx.x * kRouterDxTok, t1 = min(n, t0 + kRouterDxTok);
#pragma unroll 2
  for (int64_t t = t0; t < t1; ++t) {
    const float4 g0 = *reinterpret_cast<const float4*>(dlog + t * 8);
    const float4 g1 = *reinterpret_cast<const float4*>(dlog + t * 8 + 4);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float4* o = reinterpret_cast<float4*>(dx + t * lddx + c);
    float4 v = *o;
    float sq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(g[e], r[q][e], acc);
      sq[q] = acc;
    }
    v.x += sq[0];
    v.y += sq[1];
    v.z += sq[2];
    v.w += sq[3];
    *o = v;
  }
}

// ------------------------------------------------------------- padded expert layout
// The grouped expert GEMMs (cb_gemm_grouped / cb_gemm_gated_*_grouped) need every expert's
// rows to start on a 256-row boundary: expert e owns padded rows [poff[e], poff[e+1]),
// poff[e+1] - poff[e] = roundup(count_e, 256); its first count_e rows are its assignments in
// the stable sorted order, the rest are zero.  Everything stays on the device (no host sync).
__global__ void pad_offsets_k(int E, const int* __restrict__ off, int* __restrict__ poff) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int acc = 0;
    poff[0] = 0;
    for (int e = 0; e < E; ++e) {
      acc += (off[e + 1] - off[e] + 255) / 256 * 256;
      poff[e + 1] = acc;
    }
  }
}

// one warp per padded row r < poff[E], 16-byte chunks (d * sizeof(T) % 16 == 0):
// xe[r] = x[perm[off[e] + j] / k] and pinv[assignment] = r for the expert's real rows, zero
// for its pad rows
template <typename T>
__global__ void __launch_bounds__(256) pad_rows_k(int cap, int d, int E, int k, const int* __restrict__ off,
                                                  const int* __restrict__ poff, const int32_t* __restrict__ perm,
                                                  const T* __restrict__ x, int64_t ldx, T* __restrict__ out,
                                                  int64_t ldo, int32_t* __restrict__ pinv) {
  __shared__ int s_po[65], s_o[65];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    s_po[i] = poff[i];
    s_o[i] = off[i];
  }
  __syncthreads();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= s_po[E] || r >= cap) return;  // beyond the last expert: never read by the grouped GEMMs
  int e = 0;
  while (e + 1 < E && s_po[e + 1] <= r) ++e;
  const int j = r - s_po[e];
  const int chunks = d * (int)sizeof(T) / 16;
  uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)r * ldo);
  if (j < s_o[e + 1] - s_o[e]) {
    const int a = perm[s_o[e] + j];
    if (lane == 0) pinv[a] = r;
    const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)(a / k) * ldx);
    for (int c = lane; c < chunks; c += 32) dst[c] = src[c];
  } else {
    for (int c = lane; c < chunks; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
  }
}

// zero only the pad rows: block e walks expert e's rows [poff[e] + count_e, poff[e+1])
__global__ void __launch_bounds__(256) zero_pad_k(int d_bytes, int E, const int* __restrict__ off,
                                                  const int* __restrict__ poff, uint8_t* __restrict__ buf,
                                                  int64_t ld_bytes) {
  const int e = blockIdx.x;
  if (e >= E) return;
  const int r0 = poff[e] + (off[e + 1] - off[e]), r1 = poff[e + 1];
  const int chunks = d_bytes / 16;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = r0 + w; r < r1; r += nw) {
    uint4* dst = reinterpret_cast<uint4*>(buf + (int64_t)r * ld_bytes);
    for (int c = lane; c < chunks; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
  }
}

extern "C" int cb_moe_dispatch_padded(int64_t nk, int dim, int experts, int top_k, const int* offsets,
                                      const int32_t* perm, const void* x, int64_t ldx, int dtype, int* poff,
                                      int32_t* pinv, void* xe, int64_t ldxe, int cap, void* stream) {
  if (experts < 1 || experts > 64) return fail(CB_ERR_ARG, "moe dispatch: 1..64 experts");
  if ((int64_t)cap < nk + (int64_t)experts * 255) return fail(CB_ERR_SHAPE, "moe dispatch: capacity %d too small", cap);
  const int es = dtype == CB_DT_F32 ? 4 : 2;
  if ((dim * es) % 16 || ((ldx * es) | (ldxe * es)) % 16 || ((reinterpret_cast<uintptr_t>(x) |
                                                              reinterpret_cast<uintptr_t>(xe)) & 15))
    return fail(CB_ERR_ARG, "moe dispatch: rows must be whole, 16-byte aligned chunks");
  cudaStream_t st = (cudaStream_t)stream;
  pad_offsets_k<<<1, 32, 0, st>>>(experts, offsets, poff);
  if (int r = check_launch("moe_pad_offsets")) return r;
  if (cap <= 0) return CB_OK;
  const int blocks = (cap + 7) / 8;  // one warp per padded row, 8 per block
  if (dtype == CB_DT_F32)
    pad_rows_k<float><<<blocks, 256, 0, st>>>(cap, dim, experts, top_k, offsets, poff, perm, (const float*)x, ldx,
                                              (float*)xe, ldxe, pinv);
  else
    pad_rows_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(cap, dim, experts, top_k, offsets, poff, perm,
                                                      (const __nv_bfloat16*)x, ldx, (__nv_bfloat16*)xe, ldxe, pinv);
  return check_launch("moe_dispatch_padded");
}

extern "C" int cb_moe_zero_pad_rows(int cap, int dim, int experts, const int* offsets, const int* poff, void* buf,
                                    int64_t ld, int dtype, void* stream) {
  if (cap <= 0) return CB_OK;
  if (experts < 1 || experts > 64) return fail(CB_ERR_ARG, "moe zero pad: 1..64 experts");
  const int es = dtype == CB_DT_F32 ? 4 : 2;
  if ((dim * es) % 16 || (ld * es) % 16 || (reinterpret_cast<uintptr_t>(buf) & 15))
    return fail(CB_ERR_ARG, "moe zero pad: rows must be whole, 16-byte aligned chunks");
  zero_pad_k<<<experts, 256, 0, (cudaStream_t)stream>>>(dim * es, experts, offsets, poff, (uint8_t*)buf, ld * es);
  return check_launch("moe_zero_pad_rows");
}

// inv[perm[j]] = j
__global__ void invert_perm_k(int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) inv[perm[j]] = (int32_t)j;
}

// int32 -> int64 widening (expert ids feed cb_sort_ids)
__global__ void widen_k(int64_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) b[j] = a[j];
}

extern "C" int cb_invert_perm(int64_t n, const int32_t* perm, int32_t* inv, void* stream) {
  if (n <= 0) return CB_OK;
  invert_perm_k<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, perm, inv);
  return check_launch("invert_perm");
}

extern "C" int cb_widen_i32(int64_t n, const int32_t* a, int64_t* b, void* stream) {
  if (n <= 0) return CB_OK;
  widen_k<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, a, b);
  return check_launch("widen_i32");
}

// drouter (+)= x^T dlog (deterministic: fixed token blocks + ordered column reduction);
// dx += dlog router^T.  workspace: ceil(n / 128) * dim * experts floats.
extern "C" int cb_moe_router_bwd_gemms(int64_t n, int dim, int experts, const void* x, int64_t ldx, int x_dtype,
                                       const float* dlogits, const float* router, float* drouter, float* dx,
                                       int64_t lddx, float* workspace, void* stream) {
  if (experts < 1 || experts > kMaxExperts) return fail(CB_ERR_UNSUPPORTED, "moe: experts must be in [1, %d]", kMaxExperts);
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int tpb = 128;  // tokens per block: 4x the blocks of 512 for load-latency hiding
  const int nblk = (int)((n + tpb - 1) / tpb);
  dim3 grid(nblk, (dim + 255) / 256);
  const bool small = experts <= 8;
  if (x_dtype == CB_DT_F32) {
    if (small)
      router_wgrad_k<float, 8><<<grid, 256, 0, st>>>(n, dim, experts, tpb, (const float*)x, ldx, dlogits, workspace);
    else
      router_wgrad_k<float, kMaxExperts><<<grid, 256, 0, st>>>(n, dim, experts, tpb, (const float*)x, ldx, dlogits,
                                                               workspace);
  } else {
    if (small)
      router_wgrad_k<__nv_bfloat16, 8><<<grid, 256, 0, st>>>(n, dim, experts, tpb, (const __nv_bfloat16*)x, ldx,
                                                             dlogits, workspace);
    else
      router_wgrad_k<__nv_bfloat16, kMaxExperts><<<grid, 256, 0, st>>>(n, dim, experts, tpb,
                                                                       (const __nv_bfloat16*)x, ldx, dlogits,
                                                                       workspace);
  }
  if (int s = check_launch("moe_router_wgrad")) return s;
  if (int s = cb_col_reduce(nblk, dim * experts, workspace, drouter, 1, stream)) return s;
  const bool vec = experts == 8 && (reinterpret_cast<uintptr_t>(router) & 15) == 0;
  if (vec && dim % 4 == 0 && lddx % 4 == 0 && !(reinterpret_cast<uintptr_t>(dx) & 15) &&
      !(reinterpret_cast<uintptr_t>(dlogits) & 15)) {
    dim3 g2((unsigned)((n + kRouterDxTok - 1) / kRouterDxTok), (unsigned)((dim + 1023) / 1024));
    router_dx_v4_k<<<g2, 256, 0, st>>>(n, dim, dlogits, router, dx, lddx);
  } else if (vec)
    router_dx_k<8><<<(int)n, 256, 0, st>>>(n, dim, experts, dlogits, router, dx, lddx);
  else
    router_dx_k<kMaxExperts><<<(int)n, 256, 0, st>>>(n, dim, experts, dlogits, router, dx, lddx);
  return check_launch("moe_router_dx");
}
