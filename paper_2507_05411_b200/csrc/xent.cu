// Next-token softmax cross-entropy, forward + backward in one pass over the logits
// (reference layers.py:638-651: loss = -mean over B*(T-1) of log_softmax(logits[:, :-1])
// at targets tokens[:, 1:]; log_softmax as reference layers.py:86-88).
//
// Row r = b*T + t of the [B*T, V] logits predicts tokens[b, t+1]; rows with t = T-1 have
// no target: their gradient is zero and they do not enter the mean.  The per-row loss
// is kept in f32; the batch mean is a deterministic single-CTA f64 reduction.
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

template <typename TL, typename TG>
__global__ void __launch_bounds__(512) xent_k(int T, int V, const TL* __restrict__ logits, int64_t ld,
                                              const int64_t* __restrict__ tokens, float* __restrict__ row_loss,
                                              TG* __restrict__ dlogits, int64_t ldg, float grad_scale) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const int t = (int)(row % T);
  const TL* lr = logits + row * ld;
  TG* gr = dlogits ? dlogits + row * ldg : nullptr;
  if (t == T - 1) {
    if (gr)
      for (int i = threadIdx.x; i < V; i += blockDim.x) gr[i] = from_f32<TG>(0.f);
    if (threadIdx.x == 0) row_loss[row] = 0.f;
    return;
  }
  const int64_t target = tokens[row + 1];
  // read the target logit before any thread can overwrite it (dlogits may alias logits)
  const float target_logit = threadIdx.x == 0 ? to_f32(lr[target]) : 0.f;
  // pass 1: online max / sum of exp
  float m = -INFINITY, s = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = to_f32(lr[i]);
    if (v > m) {
      s = s * __expf(m - v) + 1.f;
      m = v;
    } else {
      s += __expf(v - m);
    }
  }
  // combine (m, s) across the block
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  __shared__ float sm[32], ss[32];
  if (lane == 0) {
    sm[wid] = m;
    ss[wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    m = lane < nw ? sm[lane] : -INFINITY;
    s = lane < nw ? ss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      sm[0] = m;
      ss[0] = s;
    }
  }
  __syncthreads();
  m = sm[0];
  s = ss[0];
  const float lse = m + logf(s);
  if (threadIdx.x == 0) row_loss[row] = lse - target_logit;
  (void)red;
  if (gr) {
    const float inv = 1.f / s;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      float p = __expf(to_f32(lr[i]) - m) * inv;
      if (i == target) p -= 1.f;
      gr[i] = from_f32<TG>(p * grad_scale);
    }
  }
}

// Single-HBM-pass variant for f32 logits: the row lives in registers (NV4 float4 per thread,
// V <= NV4 * 4 * 1024), so logits are read once and dlogits written once.
__device__ __forceinline__ void combine_ms(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
  m = mm;
}

template <int NV4, int NT, typename TG>
__global__ void __launch_bounds__(NT) xent_reg_k(int T, int V, const float* __restrict__ logits, int64_t ld,
                                                   const int64_t* __restrict__ tokens, float* __restrict__ row_loss,
                                                   TG* __restrict__ dlogits, int64_t ldg, float grad_scale) {
  __shared__ float sm[32], ss[32];
  const int64_t row = blockIdx.x;
  const int t = (int)(row % T);
  const float* lr = logits + row * ld;
  TG* gr = dlogits ? dlogits + row * ldg : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int V4 = V >> 2;
  if (t == T - 1) {
    if (gr)
      for (int i = tid; i < V; i += blockDim.x) gr[i] = from_f32<TG>(0.f);
    if (tid == 0) row_loss[row] = 0.f;
    return;
  }
  const int64_t target = tokens[row + 1];
  const float target_logit = tid == 0 ? lr[target] : 0.f;
  float4 r[NV4];
  float m = -INFINITY, s = 0.f;
  // every load of the row in flight before any arithmetic
#pragma unroll
  for (int i = 0; i < NV4; ++i) {
    const int j = i * NT + tid;
    r[i] = j < V4 ? __ldcs(reinterpret_cast<const float4*>(lr) + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // the thread's max, then exp(x - max) kept in place of the logits: the gradient pass needs
  // a single exp per thread (the rescale to the row max)
#pragma unroll
  for (int i = 0; i < NV4; ++i)
    if (i * NT + tid < V4) m = fmaxf(m, fmaxf(fmaxf(r[i].x, r[i].y), fmaxf(r[i].z, r[i].w)));
#pragma unroll
  for (int i = 0; i < NV4; ++i) {
    if (i * NT + tid < V4) {
      r[i] = make_float4(__expf(r[i].x - m), __expf(r[i].y - m), __expf(r[i].z - m), __expf(r[i].w - m));
      s += (r[i].x + r[i].y) + (r[i].z + r[i].w);
    }
  }
  const float tmax = m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) combine_ms(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) {
    sm[wid] = m;
    ss[wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
    m = lane < (int)(blockDim.x >> 5) ? sm[lane] : -INFINITY;
    s = lane < (int)(blockDim.x >> 5) ? ss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) combine_ms(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) {
      sm[0] = m;
      ss[0] = s;
    }
  }
  __syncthreads();
  m = sm[0];
  s = ss[0];
  if (tid == 0) row_loss[row] = m + logf(s) - target_logit;
  if (!gr) return;
  const float inv = grad_scale / s;
  const float sc = tmax == -INFINITY ? 0.f : __expf(tmax - m) * inv;
#pragma unroll
  for (int i = 0; i < NV4; ++i) {
    const int j = i * NT + tid;
    if (j < V4) {
      const int base = j * 4;
      // the one-hot term by comparison (a dynamic index would put p[] in local memory)
      float p[4] = {r[i].x * sc - (target == base ? grad_scale : 0.f),
                    r[i].y * sc - (target == base + 1 ? grad_scale : 0.f),
                    r[i].z * sc - (target == base + 2 ? grad_scale : 0.f),
                    r[i].w * sc - (target == base + 3 ? grad_scale : 0.f)};
      if constexpr (sizeof(TG) == 2) {  // one 8-byte store of 4 bf16
        __nv_bfloat162 lo = __floats2bfloat162_rn(p[0], p[1]), hi = __floats2bfloat162_rn(p[2], p[3]);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(gr + base) = pk;
      } else {
        *reinterpret_cast<float4*>(gr + base) = make_float4(p[0], p[1], p[2], p[3]);
      }
    }
  }
}

// Deterministic mean of row losses (rows with t == T-1 are zero and excluded from the count).
__global__ void __launch_bounds__(1024) loss_reduce_k(int64_t rows, int64_t count, const float* __restrict__ row_loss,
                                                      double* __restrict__ out64, float* __restrict__ out32) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) acc += (double)row_loss[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) {
      const double mean = acc / (double)count;
      if (out64) *out64 = mean;
      if (out32) *out32 = (float)mean;
    }
  }
}

}  // namespace cb

using namespace cb;

extern "C" int cb_xent_fwd_bwd(int batch, int seq_len, int vocab, const void* logits, int64_t ld, int l_dtype,
                               const int64_t* tokens, float* row_loss, void* dlogits, int64_t ldg, int g_dtype,
                               float grad_scale, double* loss64, float* loss32, void* stream) {
  if (seq_len < 2 || batch <= 0) return fail(CB_ERR_SHAPE, "trainer expects tokens of shape [batch, seq>=2]");
  if (vocab <= 0) return fail(CB_ERR_SHAPE, "xent: vocab must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = (int64_t)batch * seq_len;
  const int64_t gal = g_dtype == CB_DT_F32 ? 16 : 8;  // vector store of 4 gradients
  const bool reg_ok = l_dtype == CB_DT_F32 && vocab % 4 == 0 && vocab <= 8 * 4 * 1024 && (ld % 4) == 0 &&
                      !(reinterpret_cast<uintptr_t>(logits) & 15) && (!dlogits || dlogits != logits) &&
                      (!dlogits || ((ldg % 4) == 0 && (reinterpret_cast<uintptr_t>(dlogits) % gal) == 0));
  if (reg_ok) {
    if (g_dtype == CB_DT_F32)
      xent_reg_k<8, 1024, float><<<rows, 1024, 0, st>>>(seq_len, vocab, (const float*)logits, ld, tokens, row_loss,
                                                        (float*)dlogits, ldg, grad_scale);
    else
      xent_reg_k<8, 1024, __nv_bfloat16><<<rows, 1024, 0, st>>>(seq_len, vocab, (const float*)logits, ld, tokens,
                                                                row_loss, (__nv_bfloat16*)dlogits, ldg, grad_scale);
  } else if (l_dtype == CB_DT_F32 && g_dtype == CB_DT_F32)
    xent_k<float, float><<<rows, 512, 0, st>>>(seq_len, vocab, (const float*)logits, ld, tokens, row_loss,
                                               (float*)dlogits, ldg, grad_scale);
  else if (l_dtype == CB_DT_F32)
    xent_k<float, __nv_bfloat16><<<rows, 512, 0, st>>>(seq_len, vocab, (const float*)logits, ld, tokens, row_loss,
                                                       (__nv_bfloat16*)dlogits, ldg, grad_scale);
  else if (g_dtype == CB_DT_F32)
    xent_k<__nv_bfloat16, float><<<rows, 512, 0, st>>>(seq_len, vocab, (const __nv_bfloat16*)logits, ld, tokens,
                                                       row_loss, (float*)dlogits, ldg, grad_scale);
  else
    xent_k<__nv_bfloat16, __nv_bfloat16><<<rows, 512, 0, st>>>(seq_len, vocab, (const __nv_bfloat16*)logits, ld,
                                                               tokens, row_loss, (__nv_bfloat16*)dlogits, ldg,
                                                               grad_scale);
  if (int s = check_launch("xent")) return s;
  loss_reduce_k<<<1, 1024, 0, st>>>(rows, (int64_t)batch * (seq_len - 1), row_loss, loss64, loss32);
  return check_launch("loss_reduce");
}
