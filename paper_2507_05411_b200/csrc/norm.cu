// RMSNorm forward/backward (reference layers.py:176-193: x / sqrt(mean(x^2) + eps) * scale).
//
// Forward: one CTA per row; f32 statistics; writes y in the GEMM input dtype and the
// per-row reciprocal RMS (the only statistic the backward needs).  Rows whose width is a
// multiple of 256 keep their 8 values per thread in registers (one HBM read of x).
// Backward (one pass over x, dy, dres):
//   dx     = dres + r*s*dy - x * r^3/D * sum(s*dy*x)     (dres: the residual branch)
//   dx_bf  = bf16(dx) (optional second output: the next GEMM's operand, saves a cast pass)
//   dscale = sum_rows dy * x * r  — each CTA owns a fixed set of rows and keeps its
//            column partials in registers; a fixed-order column reduction finishes it
//            (deterministic, no atomics).
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 t = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float (&v)[8]);
template <>
__device__ __forceinline__ void store8<float>(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 t;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = t;
}

// ---------------------------------------------------------------- forward
template <typename TX, typename TY>
__global__ void __launch_bounds__(1024) rmsnorm_fwd_vec_k(int dim, const TX* __restrict__ x, int64_t ldx,
                                                          const float* __restrict__ scale, float eps, TY* __restrict__ y,
                                                          int64_t ldy, float* __restrict__ rstd) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const int c = threadIdx.x * 8;
  float v[8], s[8];
  load8(x + row * ldx + c, v);
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / (float)dim + eps);
  if (threadIdx.x == 0 && rstd) rstd[row] = r;
  load8(scale + c, s);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = v[i] * r * s[i];
  store8(y + row * ldy + c, v);
}

template <typename TX, typename TY>
__global__ void __launch_bounds__(256) rmsnorm_fwd_k(int dim, const TX* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ scale, float eps, TY* __restrict__ y,
                                                     int64_t ldy, float* __restrict__ rstd) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const TX* xr = x + row * ldx;
  float ss = 0.f;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    const float v = to_f32(xr[i]);
    ss = fmaf(v, v, ss);
  }
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / (float)dim + eps);
  if (threadIdx.x == 0 && rstd) rstd[row] = r;
  TY* yr = y + row * ldy;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) yr[i] = from_f32<TY>(to_f32(xr[i]) * r * scale[i]);
}

// ---------------------------------------------------------------- backward
// grid: P CTAs, CTA p handles rows p, p+P, ...; partial[p][dim] gets its dscale share.
template <typename TX, typename TG>
__global__ void __launch_bounds__(1024) rmsnorm_bwd_vec_k(int rows, int dim, const TX* __restrict__ x, int64_t ldx,
                                                          const float* __restrict__ scale,
                                                          const float* __restrict__ rstd, const TG* __restrict__ dy,
                                                          int64_t lddy, const float* __restrict__ dres, int64_t lddres,
                                                          float* __restrict__ dx, int64_t lddx,
                                                          __nv_bfloat16* __restrict__ dxb, int64_t lddxb,
                                                          float* __restrict__ partial) {
  __shared__ float red[32];
  const int c = threadIdx.x * 8;
  float s[8], ps[8];
  load8(scale + c, s);
#pragma unroll
  for (int i = 0; i < 8; ++i) ps[i] = 0.f;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    float xv[8], g[8];
    load8(x + (int64_t)row * ldx + c, xv);
    load8(dy + (int64_t)row * lddy + c, g);
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      dot = fmaf(g[i] * s[i], xv[i], dot);
      ps[i] = fmaf(g[i] * r, xv[i], ps[i]);
    }
    dot = block_sum(dot, red);
    const float k = dot * r * r * r / (float)dim;
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = r * s[i] * g[i] - xv[i] * k;
    if (dres) {
      float d[8];
      load8(dres + (int64_t)row * lddres + c, d);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] += d[i];
    }
    store8(dx + (int64_t)row * lddx + c, o);
    if (dxb) store8(dxb + (int64_t)row * lddxb + c, o);
  }
  if (partial) store8(partial + (int64_t)blockIdx.x * dim + c, ps);
}

template <typename TX, typename TG>
__global__ void __launch_bounds__(256) rmsnorm_bwd_k(int dim, const TX* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ scale, const float* __restrict__ rstd,
                                                     const TG* __restrict__ dy, int64_t lddy,
                                                     const float* __restrict__ dres, int64_t lddres,
                                                     float* __restrict__ dx, int64_t lddx,
                                                     __nv_bfloat16* __restrict__ dxb, int64_t lddxb) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const TX* xr = x + row * ldx;
  const TG* gr = dy + row * lddy;
  const float r = rstd[row];
  float dot = 0.f;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) dot = fmaf(to_f32(gr[i]) * scale[i], to_f32(xr[i]), dot);
  dot = block_sum(dot, red);
  const float c = dot * r * r * r / (float)dim;
  float* dxr = dx + row * lddx;
  const float* dr = dres ? dres + row * lddres : nullptr;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    float v = r * scale[i] * to_f32(gr[i]) - to_f32(xr[i]) * c;
    if (dr) v += dr[i];
    dxr[i] = v;
    if (dxb) dxb[row * lddxb + i] = __float2bfloat16_rn(v);
  }
}

// partial[chunk][col] = sum over rows in chunk of dy*x*r (scalar path)
template <typename TX, typename TG>
__global__ void __launch_bounds__(256) rmsnorm_dscale_partial_k(int rows, int dim, int rows_per_chunk,
                                                                const TX* __restrict__ x, int64_t ldx,
                                                                const float* __restrict__ rstd,
                                                                const TG* __restrict__ dy, int64_t lddy,
                                                                float* __restrict__ partial) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (col >= dim) return;
  const int r0 = chunk * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r) acc = fmaf(to_f32(dy[(int64_t)r * lddy + col]) * rstd[r], to_f32(x[(int64_t)r * ldx + col]), acc);
  partial[(int64_t)chunk * dim + col] = acc;
}

// 256 threads = 32 columns x 8 row lanes; lane r sums parts r, r+8, ... in order, then
// lane 0 adds the 8 lane sums in order: a fixed summation order (deterministic).
__global__ void __launch_bounds__(256) col_reduce_k(int nparts, int dim, const float* __restrict__ partial,
                                                    float* __restrict__ out, int accumulate) {
  __shared__ float red[8][33];
  const int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + c;
  float acc = 0.f;
  if (col < dim)
    for (int p = r; p < nparts; p += 8) acc += partial[(int64_t)p * dim + col];
  red[r][c] = acc;
  __syncthreads();
  if (r == 0 && col < dim) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += red[i][c];
    out[col] = accumulate ? out[col] + s : s;
  }
}

static bool vec_ok(int dim, const void* const* ptrs, const int64_t* lds, int n, int elem_align = 8) {
  if (dim % 256 != 0 || dim > 8192) return false;
  for (int i = 0; i < n; ++i) {
    if (ptrs[i] && ((reinterpret_cast<uintptr_t>(ptrs[i]) & 31) || (lds[i] % elem_align))) return false;
  }
  return true;
}

constexpr int kBwdCtas = 4 * kNumSMs;

}  // namespace cb

using namespace cb;

#define DISPATCH_XY(xdt, ydt, FN, ...)                                   \
  ((xdt) == CB_DT_F32 ? ((ydt) == CB_DT_F32 ? FN<float, float>(__VA_ARGS__) \
                                            : FN<float, __nv_bfloat16>(__VA_ARGS__)) \
                      : ((ydt) == CB_DT_F32 ? FN<__nv_bfloat16, float>(__VA_ARGS__) \
                                            : FN<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__)))

template <typename TX, typename TY>
static int launch_fwd(int rows, int dim, const void* x, int64_t ldx, const float* scale, float eps, void* y,
                      int64_t ldy, float* rstd, cudaStream_t st) {
  const void* ptrs[3] = {x, y, scale};
  const int64_t lds[3] = {ldx, ldy, 8};
  if (vec_ok(dim, ptrs, lds, 3)) {
    rmsnorm_fwd_vec_k<TX, TY><<<rows, dim / 8, 0, st>>>(dim, (const TX*)x, ldx, scale, eps, (TY*)y, ldy, rstd);
  } else {
    rmsnorm_fwd_k<TX, TY><<<rows, 256, 0, st>>>(dim, (const TX*)x, ldx, scale, eps, (TY*)y, ldy, rstd);
  }
  return check_launch("rmsnorm_fwd");
}

extern "C" int cb_rmsnorm_fwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale,
                              float eps, void* y, int64_t ldy, int y_dtype, float* rstd, void* stream) {
  if (rows < 0 || dim <= 0) return fail(CB_ERR_SHAPE, "rmsnorm: bad extents rows=%d dim=%d", rows, dim);
  if (rows == 0) return CB_OK;
  return DISPATCH_XY(x_dtype, y_dtype, launch_fwd, rows, dim, x, ldx, scale, eps, y, ldy, rstd, (cudaStream_t)stream);
}

template <typename TX, typename TG>
static int launch_bwd(int rows, int dim, const void* x, int64_t ldx, const float* scale, const float* rstd,
                      const void* dy, int64_t lddy, const float* dres, int64_t lddres, float* dx, int64_t lddx,
                      void* dxb, int64_t lddxb, float* dscale, float* workspace, cudaStream_t st) {
  const void* ptrs[6] = {x, dy, dres, dx, dxb, scale};
  const int64_t lds[6] = {ldx, lddy, lddres, lddx, lddxb, 8};
  if (vec_ok(dim, ptrs, lds, 6)) {
    const int P = std::min(rows, kBwdCtas);
    rmsnorm_bwd_vec_k<TX, TG><<<P, dim / 8, 0, st>>>(rows, dim, (const TX*)x, ldx, scale, rstd, (const TG*)dy, lddy,
                                                    dres, lddres, dx, lddx, (__nv_bfloat16*)dxb, lddxb,
                                                    dscale ? workspace : nullptr);
    if (int s = check_launch("rmsnorm_bwd")) return s;
    if (dscale) {
      col_reduce_k<<<(dim + 31) / 32, 256, 0, st>>>(P, dim, workspace, dscale, 1);
      return check_launch("rmsnorm_dscale_reduce");
    }
    return CB_OK;
  }
  rmsnorm_bwd_k<TX, TG><<<rows, 256, 0, st>>>(dim, (const TX*)x, ldx, scale, rstd, (const TG*)dy, lddy, dres, lddres,
                                             dx, lddx, (__nv_bfloat16*)dxb, lddxb);
  if (int s = check_launch("rmsnorm_bwd")) return s;
  if (dscale) {
    const int rpc = 64;
    const int chunks = (rows + rpc - 1) / rpc;
    dim3 grid((dim + 255) / 256, chunks);
    rmsnorm_dscale_partial_k<TX, TG><<<grid, 256, 0, st>>>(rows, dim, rpc, (const TX*)x, ldx, rstd, (const TG*)dy,
                                                          lddy, workspace);
    if (int s = check_launch("rmsnorm_dscale_partial")) return s;
    col_reduce_k<<<(dim + 31) / 32, 256, 0, st>>>(chunks, dim, workspace, dscale, 1);
    return check_launch("rmsnorm_dscale_reduce");
  }
  return CB_OK;
}

extern "C" int cb_rmsnorm_bwd_workspace(int rows, int dim, int64_t* bytes) {
  const int64_t a = (int64_t)std::min(rows, kBwdCtas) * dim * 4;
  const int64_t b = (int64_t)((rows + 63) / 64) * dim * 4;
  *bytes = a > b ? a : b;
  return CB_OK;
}

extern "C" int cb_rmsnorm_bwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale,
                              const float* rstd, const void* dy, int64_t lddy, int dy_dtype, const float* dres,
                              int64_t lddres, float* dx, int64_t lddx, void* dx_bf16, int64_t lddxb, float* dscale,
                              float* workspace, void* stream) {
  if (rows < 0 || dim <= 0) return fail(CB_ERR_SHAPE, "rmsnorm_bwd: bad extents");
  if (rows == 0) return CB_OK;
  if (dscale && !workspace) return fail(CB_ERR_ARG, "rmsnorm_bwd: dscale needs a workspace");
  return DISPATCH_XY(x_dtype, dy_dtype, launch_bwd, rows, dim, x, ldx, scale, rstd, dy, lddy, dres, lddres, dx, lddx,
                     dx_bf16, lddxb, dscale, workspace, (cudaStream_t)stream);
}

extern "C" int cb_col_reduce(int nparts, int dim, const float* partial, float* out, int accumulate, void* stream) {
  if (nparts <= 0 || dim <= 0) return CB_OK;
  col_reduce_k<<<(dim + 31) / 32, 256, 0, (cudaStream_t)stream>>>(nparts, dim, partial, out, accumulate);
  return check_launch("col_reduce");
}
