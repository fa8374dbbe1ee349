// RMSNorm forward/backward (reference layers.py:176-193: x / sqrt(mean(x^2) + eps) * scale).
//
// Forward: one CTA per row, f32 statistics, writes y in the GEMM input dtype and the
// per-row reciprocal RMS (the only statistic the backward needs).
// Backward: dx = dres + r*s*dy - x * r^3/D * sum(s*dy*x)   (dres = the residual branch)
//           dscale = sum_rows dy * x * r   (deterministic two-level column reduction)
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

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

template <typename TX, typename TG>
__global__ void __launch_bounds__(256) rmsnorm_bwd_k(int dim, const TX* __restrict__ x, int64_t ldx,
                                                     const float* __restrict__ scale, const float* __restrict__ rstd,
                                                     const TG* __restrict__ dy, int64_t lddy,
                                                     const float* __restrict__ dres, int64_t lddres,
                                                     float* __restrict__ dx, int64_t lddx) {
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
  }
}

// partial[chunk][col] = sum over rows in chunk of dy*x*r
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

__global__ void col_reduce_k(int nparts, int dim, const float* __restrict__ partial, float* __restrict__ out,
                             int accumulate) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= dim) return;
  float acc = 0.f;
  for (int p = 0; p < nparts; ++p) acc += partial[(int64_t)p * dim + col];
  out[col] = accumulate ? out[col] + acc : acc;
}

}  // namespace cb

using namespace cb;

#define DISPATCH_XY(xdt, ydt, KERNEL, ...)                                                                   \
  do {                                                                                                      \
    if (xdt == CB_DT_F32 && ydt == CB_DT_F32)                                                               \
      KERNEL<float, float>(__VA_ARGS__);                                                                    \
    else if (xdt == CB_DT_F32 && ydt == CB_DT_BF16)                                                         \
      KERNEL<float, __nv_bfloat16>(__VA_ARGS__);                                                            \
    else if (xdt == CB_DT_BF16 && ydt == CB_DT_BF16)                                                        \
      KERNEL<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                                                    \
    else                                                                                                    \
      KERNEL<__nv_bfloat16, float>(__VA_ARGS__);                                                            \
  } while (0)

template <typename TX, typename TY>
static void launch_fwd(int rows, int dim, const void* x, int64_t ldx, const float* scale, float eps, void* y,
                       int64_t ldy, float* rstd, cudaStream_t st) {
  rmsnorm_fwd_k<TX, TY><<<rows, 256, 0, st>>>(dim, (const TX*)x, ldx, scale, eps, (TY*)y, ldy, rstd);
}

extern "C" int cb_rmsnorm_fwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale,
                              float eps, void* y, int64_t ldy, int y_dtype, float* rstd, void* stream) {
  if (rows < 0 || dim <= 0) return fail(CB_ERR_SHAPE, "rmsnorm: bad extents rows=%d dim=%d", rows, dim);
  if (rows == 0) return CB_OK;
  DISPATCH_XY(x_dtype, y_dtype, launch_fwd, rows, dim, x, ldx, scale, eps, y, ldy, rstd, (cudaStream_t)stream);
  return check_launch("rmsnorm_fwd");
}

template <typename TX, typename TG>
static void launch_bwd(int rows, int dim, const void* x, int64_t ldx, const float* scale, const float* rstd,
                       const void* dy, int64_t lddy, const float* dres, int64_t lddres, float* dx, int64_t lddx,
                       float* dscale, float* workspace, cudaStream_t st) {
  rmsnorm_bwd_k<TX, TG><<<rows, 256, 0, st>>>(dim, (const TX*)x, ldx, scale, rstd, (const TG*)dy, lddy, dres, lddres,
                                             dx, lddx);
  if (dscale) {
    const int rpc = 64;
    const int chunks = (rows + rpc - 1) / rpc;
    dim3 grid((dim + 255) / 256, chunks);
    rmsnorm_dscale_partial_k<TX, TG><<<grid, 256, 0, st>>>(rows, dim, rpc, (const TX*)x, ldx, rstd, (const TG*)dy,
                                                          lddy, workspace);
    col_reduce_k<<<(dim + 255) / 256, 256, 0, st>>>(chunks, dim, workspace, dscale, 1);
  }
}

extern "C" int cb_rmsnorm_bwd_workspace(int rows, int dim, int64_t* bytes) {
  *bytes = (int64_t)((rows + 63) / 64) * dim * 4;
  return CB_OK;
}

extern "C" int cb_rmsnorm_bwd(int rows, int dim, const void* x, int64_t ldx, int x_dtype, const float* scale,
                              const float* rstd, const void* dy, int64_t lddy, int dy_dtype, const float* dres,
                              int64_t lddres, float* dx, int64_t lddx, float* dscale, float* workspace,
                              void* stream) {
  if (rows < 0 || dim <= 0) return fail(CB_ERR_SHAPE, "rmsnorm_bwd: bad extents");
  if (rows == 0) return CB_OK;
  if (dscale && !workspace) return fail(CB_ERR_ARG, "rmsnorm_bwd: dscale needs a workspace");
  DISPATCH_XY(x_dtype, dy_dtype, launch_bwd, rows, dim, x, ldx, scale, rstd, dy, lddy, dres, lddres, dx, lddx, dscale,
              workspace, (cudaStream_t)stream);
  return check_launch("rmsnorm_bwd", dscale ? 3 : 1);
}

extern "C" int cb_col_reduce(int nparts, int dim, const float* partial, float* out, int accumulate, void* stream) {
  if (nparts <= 0 || dim <= 0) return CB_OK;
  col_reduce_k<<<(dim + 255) / 256, 256, 0, (cudaStream_t)stream>>>(nparts, dim, partial, out, accumulate);
  return check_launch("col_reduce");
}
