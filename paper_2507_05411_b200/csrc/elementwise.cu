// Elementwise kernels of the decoder step (HBM-bound; 16-byte vector accesses when the
// row strides and base pointers allow it, a scalar path otherwise).
//
//  * RoPE (reference layers.py:235-257): interleaved pairs (x[2i], x[2i+1]) of each head
//    rotated by pos * base^(-2i/hd); cos/sin come from an f32 table the host derives in
//    f64 (angles in f32 lose ~1e-4 at T=4096).  The inverse rotation is the backward.
//  * activations (reference layers.py:55-77 ACTIVATIONS, :405-416 gated FFN): linear,
//    relu, silu = x*sigmoid(x) with the overflow-safe two-branch sigmoid, sigmoid, tanh;
//    gated form act0(a) * act1(g) and its backward.
//  * cast / strided copy / accumulate.
//
// Grids are 1-D over (row, column-chunk) blocks: one 256-thread block covers 256 vectors
// of one row, so the only integer division is per block.
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

// ---- vector helpers: 16-byte packets of T (8 x bf16 or 4 x f32) ----------------------
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 t;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = t;
  }
};

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// blocks: rows * cb, cb = ceil(cols / (256 * VEC)) chunks per row
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) gated_fwd_k(int cols, int cb, int a0, int a1, const T* __restrict__ a,
                                                   int64_t lda, const T* __restrict__ g, int64_t ldg, T* __restrict__ out,
                                                   int64_t ldo) {
  constexpr int W = VEC ? Vec<T>::N : 1;
  const int64_t r = blockIdx.x / cb;
  const int c = ((int)(blockIdx.x % cb) * 256 + threadIdx.x) * W;
  if (c >= cols) return;
  const T* ar = a + r * lda;
  const T* gr = g ? g + r * ldg : nullptr;
  T* orow = out + r * ldo;
  if constexpr (VEC) {
    float x[W], y[W];
    Vec<T>::load(ar + c, x);
    if (gr) Vec<T>::load(gr + c, y);
#pragma unroll
    for (int i = 0; i < W; ++i) x[i] = act_f(a0, x[i]) * (gr ? act_f(a1, y[i]) : 1.f);
    Vec<T>::store(orow + c, x);
  } else {
    float v = act_f(a0, to_f32(ar[c]));
    if (gr) v *= act_f(a1, to_f32(gr[c]));
    orow[c] = from_f32<T>(v);
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) gated_bwd_k(int cols, int cb, int a0, int a1, const T* __restrict__ a,
                                                   int64_t lda, const T* __restrict__ g, int64_t ldg,
                                                   const T* __restrict__ dout, int64_t lddo, T* __restrict__ da,
                                                   int64_t ldda, T* __restrict__ dg, int64_t lddg) {
  constexpr int W = VEC ? Vec<T>::N : 1;
  const int64_t r = blockIdx.x / cb;
  const int c = ((int)(blockIdx.x % cb) * 256 + threadIdx.x) * W;
  if (c >= cols) return;
  float x[W], y[W], d[W], ra[W], rg[W];
  if constexpr (VEC) {
    Vec<T>::load(a + r * lda + c, x);
    Vec<T>::load(dout + r * lddo + c, d);
    if (g) Vec<T>::load(g + r * ldg + c, y);
  } else {
    x[0] = to_f32(a[r * lda + c]);
    d[0] = to_f32(dout[r * lddo + c]);
    if (g) y[0] = to_f32(g[r * ldg + c]);
  }
  if (g && a0 == ACT_LINEAR && a1 == ACT_SILU) {
    // SwiGLU: one sigmoid per element serves silu(g) and silu'(g)
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float s = stable_sigmoid(y[i]);
      const float sg = y[i] * s;
      ra[i] = d[i] * sg;
      rg[i] = d[i] * x[i] * (s + sg * (1.f - s));
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      if (g) {
        ra[i] = d[i] * act_f(a1, y[i]) * act_df(a0, x[i]);
        rg[i] = d[i] * act_f(a0, x[i]) * act_df(a1, y[i]);
      } else {
        ra[i] = d[i] * act_df(a0, x[i]);
      }
    }
  }
  if constexpr (VEC) {
    Vec<T>::store(da + r * ldda + c, ra);
    if (g) Vec<T>::store(dg + r * lddg + c, rg);
  } else {
    da[r * ldda + c] = from_f32<T>(ra[0]);
    if (g) dg[r * lddg + c] = from_f32<T>(rg[0]);
  }
}

// out (+)= alpha * in; VEC path moves 4 elements per thread (f32 or bf16 either side)
template <typename TI, typename TO, bool VEC>
__global__ void __launch_bounds__(256) copy2d_k(int cols, int cb, const TI* __restrict__ in, int64_t ldi,
                                                TO* __restrict__ out, int64_t ldo, float alpha, int accumulate) {
  constexpr int W = VEC ? 4 : 1;
  const int64_t r = blockIdx.x / cb;
  const int c = ((int)(blockIdx.x % cb) * 256 + threadIdx.x) * W;
  if (c >= cols) return;
  const TI* ip = in + r * ldi + c;
  TO* op = out + r * ldo + c;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    float v = alpha * to_f32(ip[i]);
    if (accumulate) v += to_f32(op[i]);
    op[i] = from_f32<TO>(v);
  }
}

// RoPE: one thread per 4 pairs (8 values) of one head of one row.
template <typename T>
__global__ void __launch_bounds__(256) rope_k(int64_t rows, int T_, int heads, int hd, T* __restrict__ x, int64_t ld,
                                              const float* __restrict__ cs, const float* __restrict__ sn, int inverse) {
  const int half = hd >> 1;
  const int per_row = heads * hd / 8;  // 8-value chunks per row (hd % 8 == 0 on this path)
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * per_row) return;
  const int64_t r = idx / per_row;
  const int ch = (int)(idx - r * per_row);
  const int col = ch * 8;
  const int p0 = (col % hd) >> 1;
  const int t = (int)(r % T_);
  T* px = x + r * ld + col;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = to_f32(px[i]);
  const float* ct = cs + (int64_t)t * half + p0;
  const float* st = sn + (int64_t)t * half + p0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float c = ct[i], s = inverse ? -st[i] : st[i];
    const float e = v[2 * i], o = v[2 * i + 1];
    v[2 * i] = e * c - o * s;
    v[2 * i + 1] = e * s + o * c;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) px[i] = from_f32<T>(v[i]);
}

// generic RoPE (any even hd)
template <typename T>
__global__ void rope_scalar_k(int64_t rows, int T_, int heads, int hd, T* __restrict__ x, int64_t ld,
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

}  // namespace cb

using namespace cb;

extern "C" int cb_rope(int64_t rows, int seq_len, int heads, int head_dim, void* x, int64_t ld, int dtype,
                       const float* cos_t, const float* sin_t, int inverse, void* stream) {
  if (head_dim % 2) return fail(CB_ERR_SHAPE, "rotary embedding needs an even dim, got %d", head_dim);
  if (rows <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim % 8 == 0) {
    const int64_t n = rows * heads * head_dim / 8;
    const int blocks = (int)((n + 255) / 256);
    if (dtype == CB_DT_F32)
      rope_k<float><<<blocks, 256, 0, st>>>(rows, seq_len, heads, head_dim, (float*)x, ld, cos_t, sin_t, inverse);
    else
      rope_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(rows, seq_len, heads, head_dim, (__nv_bfloat16*)x, ld, cos_t,
                                                    sin_t, inverse);
  } else {
    const int64_t n = rows * heads * (head_dim / 2);
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
    if (dtype == CB_DT_F32)
      rope_scalar_k<float><<<blocks, 256, 0, st>>>(rows, seq_len, heads, head_dim, (float*)x, ld, cos_t, sin_t, inverse);
    else
      rope_scalar_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(rows, seq_len, heads, head_dim, (__nv_bfloat16*)x, ld,
                                                           cos_t, sin_t, inverse);
  }
  return check_launch("rope");
}

template <typename T>
static int act_fwd_t(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g, int64_t ldg,
                     void* out, int64_t ldo, cudaStream_t st) {
  constexpr int W = Vec<T>::N;
  const bool vec = cols % W == 0 && lda % W == 0 && (!g || ldg % W == 0) && ldo % W == 0 && al16(a) &&
                   (!g || al16(g)) && al16(out);
  const int cb = (cols + 256 * (vec ? W : 1) - 1) / (256 * (vec ? W : 1));
  const int64_t blocks = rows * cb;
  if (vec)
    gated_fwd_k<T, true><<<blocks, 256, 0, st>>>(cols, cb, act0, act1, (const T*)a, lda, (const T*)g, ldg, (T*)out, ldo);
  else
    gated_fwd_k<T, false><<<blocks, 256, 0, st>>>(cols, cb, act0, act1, (const T*)a, lda, (const T*)g, ldg, (T*)out, ldo);
  return check_launch("act_fwd");
}

extern "C" int cb_act_fwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                          int64_t ldg, void* out, int64_t ldo, int dtype, void* stream) {
  if (act0 < 0 || act0 > 4 || act1 < 0 || act1 > 4) return fail(CB_ERR_ARG, "unknown activation id");
  if (rows <= 0 || cols <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32) return act_fwd_t<float>(rows, cols, act0, act1, a, lda, g, ldg, out, ldo, st);
  return act_fwd_t<__nv_bfloat16>(rows, cols, act0, act1, a, lda, g, ldg, out, ldo, st);
}

template <typename T>
static int act_bwd_t(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g, int64_t ldg,
                     const void* dout, int64_t lddo, void* da, int64_t ldda, void* dg, int64_t lddg, cudaStream_t st) {
  constexpr int W = Vec<T>::N;
  const bool vec = cols % W == 0 && lda % W == 0 && lddo % W == 0 && ldda % W == 0 && al16(a) && al16(dout) &&
                   al16(da) && (!g || (ldg % W == 0 && lddg % W == 0 && al16(g) && al16(dg)));
  const int cb = (cols + 256 * (vec ? W : 1) - 1) / (256 * (vec ? W : 1));
  const int64_t blocks = rows * cb;
  if (vec)
    gated_bwd_k<T, true><<<blocks, 256, 0, st>>>(cols, cb, act0, act1, (const T*)a, lda, (const T*)g, ldg,
                                                 (const T*)dout, lddo, (T*)da, ldda, (T*)dg, lddg);
  else
    gated_bwd_k<T, false><<<blocks, 256, 0, st>>>(cols, cb, act0, act1, (const T*)a, lda, (const T*)g, ldg,
                                                  (const T*)dout, lddo, (T*)da, ldda, (T*)dg, lddg);
  return check_launch("act_bwd");
}

extern "C" int cb_act_bwd(int64_t rows, int cols, int act0, int act1, const void* a, int64_t lda, const void* g,
                          int64_t ldg, const void* dout, int64_t lddo, void* da, int64_t ldda, void* dg, int64_t lddg,
                          int dtype, void* stream) {
  if (act0 < 0 || act0 > 4 || act1 < 0 || act1 > 4) return fail(CB_ERR_ARG, "unknown activation id");
  if (rows <= 0 || cols <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CB_DT_F32) return act_bwd_t<float>(rows, cols, act0, act1, a, lda, g, ldg, dout, lddo, da, ldda, dg, lddg, st);
  return act_bwd_t<__nv_bfloat16>(rows, cols, act0, act1, a, lda, g, ldg, dout, lddo, da, ldda, dg, lddg, st);
}

template <typename TI, typename TO>
static int copy_t(int64_t rows, int cols, const void* in, int64_t ldi, void* out, int64_t ldo, float alpha,
                  int accumulate, cudaStream_t st) {
  const bool vec = cols % 4 == 0 && ldi % 4 == 0 && ldo % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(in) % (4 * sizeof(TI))) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) % (4 * sizeof(TO))) == 0;
  const int cb = (cols + 256 * (vec ? 4 : 1) - 1) / (256 * (vec ? 4 : 1));
  const int64_t blocks = rows * cb;
  if (vec)
    copy2d_k<TI, TO, true><<<blocks, 256, 0, st>>>(cols, cb, (const TI*)in, ldi, (TO*)out, ldo, alpha, accumulate);
  else
    copy2d_k<TI, TO, false><<<blocks, 256, 0, st>>>(cols, cb, (const TI*)in, ldi, (TO*)out, ldo, alpha, accumulate);
  return check_launch("copy2d");
}

extern "C" int cb_copy2d(int64_t rows, int cols, const void* in, int64_t ldi, int in_dtype, void* out, int64_t ldo,
                         int out_dtype, float alpha, int accumulate, void* stream) {
  if (rows <= 0 || cols <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  using B = __nv_bfloat16;
  if (in_dtype == CB_DT_F32 && out_dtype == CB_DT_F32) return copy_t<float, float>(rows, cols, in, ldi, out, ldo, alpha, accumulate, st);
  if (in_dtype == CB_DT_F32) return copy_t<float, B>(rows, cols, in, ldi, out, ldo, alpha, accumulate, st);
  if (out_dtype == CB_DT_F32) return copy_t<B, float>(rows, cols, in, ldi, out, ldo, alpha, accumulate, st);
  return copy_t<B, B>(rows, cols, in, ldi, out, ldo, alpha, accumulate, st);
}

extern "C" int cb_memset_zero(void* ptr, int64_t bytes, void* stream) {
  if (bytes <= 0) return CB_OK;
  cudaError_t e = cudaMemsetAsync(ptr, 0, (size_t)bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(CB_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  return CB_OK;
}

// ---- FSDP gradient reduce-scatter, local half -------------------------------------------
// out[i] = scale * sum_q parts[q][i], q = 0..nparts-1 in order (every rank sums its slice in
// rank order: deterministic).  The peers' slices arrive by copy-engine reads of their
// symmetric-memory gradient buffers (engine.FSDPProvider._rs); this is the only SM work of
// the reduce-scatter.  HBM-bound: (nparts + 1) * 4 bytes per element.
struct SumParts {
  const float* p[8];
};

__global__ void __launch_bounds__(256) sum_parts_k(SumParts s, int nparts, int64_t n4, float* __restrict__ out,
                                                   float scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(s.p[0]) + i);
    for (int q = 1; q < nparts; ++q) {
      const float4 b = __ldcs(reinterpret_cast<const float4*>(s.p[q]) + i);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    a.x *= scale;
    a.y *= scale;
    a.z *= scale;
    a.w *= scale;
    reinterpret_cast<float4*>(out)[i] = a;
  }
}

extern "C" int cb_sum_parts(int nparts, int64_t n, const void* parts, void* out, float scale, void* stream) {
  if (n <= 0) return CB_OK;
  if (nparts < 1 || nparts > 8) return fail(CB_ERR_SHAPE, "sum_parts: nparts %d not in [1, 8]", nparts);
  if (n % 4) return fail(CB_ERR_SHAPE, "sum_parts: n %lld not a multiple of 4", (long long)n);
  SumParts s{};
  const float* const* hp = reinterpret_cast<const float* const*>(parts);
  for (int q = 0; q < nparts; ++q) {
    s.p[q] = hp[q];
    if (reinterpret_cast<uintptr_t>(hp[q]) & 15) return fail(CB_ERR_SHAPE, "sum_parts: part %d not 16-byte aligned", q);
  }
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(CB_ERR_SHAPE, "sum_parts: out not 16-byte aligned");
  const int64_t n4 = n / 4;
  const int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
  sum_parts_k<<<blocks, 256, 0, (cudaStream_t)stream>>>(s, nparts, n4, (float*)out, scale);
  return check_launch("sum_parts");
}

// f32 -> three bf16 terms x = x1 + x2 + x3 (+ O(2^-24 |x|)): the operand split of the f32 parity
// mode's GEMMs on the tcgen05 engine (six bf16 products, the "BF16x6" FP32 emulation).
// src is a row-major [rows][cols] view with row stride ld; the three outputs are contiguous.
__global__ void __launch_bounds__(256) split_bf16x3_k(int64_t rows, int cols, const float* __restrict__ src,
                                                      int64_t ld, __nv_bfloat16* __restrict__ d1,
                                                      __nv_bfloat16* __restrict__ d2, __nv_bfloat16* __restrict__ d3) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const float x = src[r * ld + (i - r * cols)];
    const __nv_bfloat16 a = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(a);
    const __nv_bfloat16 b = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(b);
    d1[i] = a;
    d2[i] = b;
    d3[i] = __float2bfloat16_rn(r2);
  }
}

extern "C" int cb_split_bf16x3(int64_t rows, int cols, const float* src, int64_t ld, void* d1, void* d2, void* d3,
                               void* stream) {
  if (rows <= 0 || cols <= 0) return CB_OK;
  if (ld < cols) return fail(CB_ERR_SHAPE, "split_bf16x3: ld %lld < cols %d", (long long)ld, cols);
  const int64_t n = rows * cols;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  split_bf16x3_k<<<blocks, 256, 0, (cudaStream_t)stream>>>(rows, cols, src, ld, (__nv_bfloat16*)d1,
                                                           (__nv_bfloat16*)d2, (__nv_bfloat16*)d3);
  return check_launch("split_bf16x3");
}
