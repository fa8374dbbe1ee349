// Elementwise kernels of the decoder step.
//
//  * RoPE (reference layers.py:235-257): interleaved pairs (x[2i], x[2i+1]) of each head
//    rotated by pos * base^(-2i/hd); cos/sin come from an f32 table the host derives in
//    f64 (angles in f32 lose ~1e-4 at T=4096).  The inverse rotation is the backward.
//  * activations (reference layers.py:55-77 ACTIVATIONS, :405-416 gated FFN): linear,
//    relu, silu = x*sigmoid(x) with the overflow-safe two-branch sigmoid, sigmoid, tanh;
//    gated form act0(a) * act1(g) and its backward.
//  * cast / strided copy.
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

enum Act { ACT_LINEAR = 0, ACT_RELU = 1, ACT_SILU = 2, ACT_SIGMOID = 3, ACT_TANH = 4 };

__device__ __forceinline__ float act_f(int a, float x) {
  switch (a) {
    case ACT_RELU: return fmaxf(x, 0.f);
    case ACT_SILU: return x * stable_sigmoid(x);
    case ACT_SIGMOID: return stable_sigmoid(x);
    case ACT_TANH: return tanhf(x);
    default: return x;
  }
}
__device__ __forceinline__ float act_df(int a, float x) {
  switch (a) {
    case ACT_RELU: return x > 0.f ? 1.f : 0.f;
    case ACT_SILU: {
      const float s = stable_sigmoid(x);
      return s * (1.f + x * (1.f - s));
    }
    case ACT_SIGMOID: {
      const float s = stable_sigmoid(x);
      return s * (1.f - s);
    }
    case ACT_TANH: {
      const float t = tanhf(x);
      return 1.f - t * t;
    }
    default: return 1.f;
  }
}

template <typename T>
__global__ void rope_k(int64_t rows, int T_, int heads, int hd, T* __restrict__ x, int64_t ld,
                       const float* __restrict__ cs, const float* __restrict__ sn, int inverse) {
  const int half = hd >> 1;
  const int64_t total = rows * heads * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(i % half);
    const int64_t rh = i / half;
    const int h = (int)(rh % heads);
    const int64_t r = rh / heads;
    const int t = (int)(r % T_);
    T* px = x + r * ld + (int64_t)h * hd + 2 * p;
    const float e = to_f32(px[0]), o = to_f32(px[1]);
    const float c = cs[(int64_t)t * half + p];
    const float s = inverse ? -sn[(int64_t)t * half + p] : sn[(int64_t)t * half + p];
    px[0] = from_f32<T>(e * c - o * s);
    px[1] = from_f32<T>(e * s + o * c);
  }
}

template <typename T>
__global__ void gated_fwd_k(int64_t rows, int cols, int a0, int a1, const T* __restrict__ a, int64_t lda,
                            const T* __restrict__ g, int64_t ldg, T* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int c = (int)(i - r * cols);
    float v = act_f(a0, to_f32(a[r * lda + c]));
    if (g) v *= act_f(a1, to_f32(g[r * ldg + c]));
    out[r * ldo + c] = from_f32<T>(v);
  }
}

template <typename T>
__global__ void gated_bwd_k(int64_t rows, int cols, int a0, int a1, const T* __restrict__ a, int64_t lda,
                            const T* __restrict__ g, int64_t ldg, const T* __restrict__ dout, int64_t lddo,
                            T* __restrict__ da, int64_t ldda, T* __restrict__ dg, int64_t lddg) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int c = (int)(i - r * cols);
    const float x = to_f32(a[r * lda + c]);
    const float d = to_f32(dout[r * lddo + c]);
    if (g) {
      const float y = to_f32(g[r * ldg + c]);
      const float fy = act_f(a1, y);
      da[r * ldda + c] = from_f32<T>(d * fy * act_df(a0, x));
      dg[r * lddg + c] = from_f32<T>(d * act_f(a0, x) * act_df(a1, y));
    } else {
      da[r * ldda + c] = from_f32<T>(d * act_df(a0, x));
    }
  }
}

template <typename TI, typename TO>
__global__ void copy2d_k(int64_t rows, int cols, const TI* __restrict__ in, int64_t ldi, TO* __restrict__ out,
                         int64_t ldo, float alpha, int accumulate) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int c = (int)(i - r * cols);
    float v = alpha * to_f32(in[r * ldi + c]);
    if (accumulate) v += to_f32(out[r * ldo + c]);
    out[r * ldo + c] = from_f32<TO>(v);
  }
}

static inline int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)kNumSMs * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace cb

using namespace cb;

extern "C" int cb_rope(int64_t rows, int seq_len, int heads, int head_dim, void* x, int64_t ld, int dtype,
                       const float* cos_t, const float* sin_t, int inverse, void* stream) {
  if (head_dim % 2) return fail(CB_ERR_SHAPE, "rotary embedding needs an even dim, got %d", head_dim);
  if (rows <= 0) return CB_OK;
  const int64_t n = rows * heads * (head_dim / 2);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32)
    rope_k<float><<<grid_for(n), 256, 0, st>>>(rows, seq_len, heads, head_dim, (float*)x, ld, cos_t, sin_t, inverse);
  else
    rope_k<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(rows, seq_len, heads, head_dim, (__nv_bfloat16*)x, ld, cos_t,
                                                       sin_t, inverse);
  return check_launch("rope");
}

extern "C" int cb_act_fwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                          int64_t ldg, void* out, int64_t ldo, int dtype, void* stream) {
  if (act0 < 0 || act0 > 4 || act1 < 0 || act1 > 4) return fail(CB_ERR_ARG, "unknown activation id");
  if (rows <= 0 || cols <= 0) return CB_OK;
  const int64_t n = rows * cols;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32)
    gated_fwd_k<float><<<grid_for(n), 256, 0, st>>>(rows, cols, act0, act1, (const float*)a, lda, (const float*)g, ldg,
                                                    (float*)out, ldo);
  else
    gated_fwd_k<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(rows, cols, act0, act1, (const __nv_bfloat16*)a, lda,
                                                            (const __nv_bfloat16*)g, ldg, (__nv_bfloat16*)out, ldo);
  return check_launch("act_fwd");
}

extern "C" int cb_act_bwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                          int64_t ldg, const void* dout, int64_t lddo, void* da, int64_t ldda, void* dg, int64_t lddg,
                          int dtype, void* stream) {
  if (act0 < 0 || act0 > 4 || act1 < 0 || act1 > 4) return fail(CB_ERR_ARG, "unknown activation id");
  if (rows <= 0 || cols <= 0) return CB_OK;
  const int64_t n = rows * cols;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32)
    gated_bwd_k<float><<<grid_for(n), 256, 0, st>>>(rows, cols, act0, act1, (const float*)a, lda, (const float*)g, ldg,
                                                    (const float*)dout, lddo, (float*)da, ldda, (float*)dg, lddg);
  else
    gated_bwd_k<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(
        rows, cols, act0, act1, (const __nv_bfloat16*)a, lda, (const __nv_bfloat16*)g, ldg,
        (const __nv_bfloat16*)dout, lddo, (__nv_bfloat16*)da, ldda, (__nv_bfloat16*)dg, lddg);
  return check_launch("act_bwd");
}

extern "C" int cb_copy2d(int64_t rows, int cols, const void* in, int64_t ldi, int in_dtype, void* out, int64_t ldo,
                         int out_dtype, float alpha, int accumulate, void* stream) {
  if (rows <= 0 || cols <= 0) return CB_OK;
  const int64_t n = rows * cols;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n);
  if (in_dtype == CB_DT_F32 && out_dtype == CB_DT_F32)
    copy2d_k<float, float><<<g, 256, 0, st>>>(rows, cols, (const float*)in, ldi, (float*)out, ldo, alpha, accumulate);
  else if (in_dtype == CB_DT_F32 && out_dtype == CB_DT_BF16)
    copy2d_k<float, __nv_bfloat16><<<g, 256, 0, st>>>(rows, cols, (const float*)in, ldi, (__nv_bfloat16*)out, ldo,
                                                      alpha, accumulate);
  else if (in_dtype == CB_DT_BF16 && out_dtype == CB_DT_F32)
    copy2d_k<__nv_bfloat16, float><<<g, 256, 0, st>>>(rows, cols, (const __nv_bfloat16*)in, ldi, (float*)out, ldo,
                                                      alpha, accumulate);
  else
    copy2d_k<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(rows, cols, (const __nv_bfloat16*)in, ldi,
                                                              (__nv_bfloat16*)out, ldo, alpha, accumulate);
  return check_launch("copy2d");
}

extern "C" int cb_memset_zero(void* ptr, int64_t bytes, void* stream) {
  if (bytes <= 0) return CB_OK;
  cudaError_t e = cudaMemsetAsync(ptr, 0, (size_t)bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(CB_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  return CB_OK;
}
