// Microbenchmarks for the attention kernels' CUDA-core side on sm_100a: TMEM load/store
// throughput per SM, MUFU ex2 throughput, FMA throughput.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2507_05411_b200/csrc scripts/ubench.cu -o /tmp/ubench
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace cb;

constexpr int kIters = 2048;

template <int NW, int BATCH>
__global__ void __launch_bounds__(NW * 32, 1) tmem_ld_bench(unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    uint32_t v[BATCH][32];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) tmem_ld32(tm + b * 32, v[b]);
    tmem_ld_wait();
#pragma unroll
    for (int b = 0; b < BATCH; ++b)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[b][i];
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) tmem_st_bench(unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t p[16];
  for (int i = 0; i < 16; ++i) p[i] = threadIdx.x * i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    tmem_st16(tm, p);
    tmem_st16(tm + 16, p);
    tmem_st_wait();
    p[it & 15] += 1;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = p[3];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) alu_bench(unsigned long long* cyc, float* sink) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
        x[i] = y - 1.0f;
      } else if (MODE == 2) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(r);
      } else if (MODE == 4) {
        uint32_t h2, r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h2) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h2));
        x[i] = __uint_as_float(r) - 1.0f;
      } else if (MODE == 5) {
        uint32_t r;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(__float_as_uint(x[i])));
        x[i] = __uint_as_float(r & 0xbfffbfffu);
      } else if (MODE == 3) {
        float y, z;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[(i + 3) & 7]), "f"(x[(i + 1) & 7]));
        z = __uint_as_float(r);
        x[i] = y - z;
      } else {
        x[i] = fmaf(x[i], 0.999f, -0.0001f);
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static unsigned long long* d_cyc;
static void* d_sink;

template <typename K>
static double run(K kern, int nthreads) {
  kern<<<148, nthreads>>>(d_cyc, (uint32_t*)d_sink);
  cudaDeviceSynchronize();
  kern<<<148, nthreads>>>(d_cyc, (uint32_t*)d_sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return -1;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  return s / 148;
}

template <typename K>
static double runf(K kern, int nthreads) {
  kern<<<148, nthreads>>>(d_cyc, (float*)d_sink);
  cudaDeviceSynchronize();
  kern<<<148, nthreads>>>(d_cyc, (float*)d_sink);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  return s / 148;
}

int main() {
  cudaMalloc(&d_cyc, 148 * 8);
  cudaMalloc(&d_sink, 148 * 1024 * 4);
#define LD(NW, B)                                                                                         \
  {                                                                                                       \
    double c = run(tmem_ld_bench<NW, B>, NW * 32);                                                         \
    printf("tmem_ld  warps=%2d batch=%d: %8.0f cyc  %6.1f B/clk/SM\n", NW, B, c,                          \
           (double)NW * 32 * 32 * 4 * B * kIters / c);                                                    \
  }
  LD(4, 1) LD(4, 2) LD(4, 4) LD(8, 1) LD(8, 2) LD(8, 4) LD(16, 1) LD(16, 2)
#define ST(NW)                                                                                            \
  {                                                                                                       \
    double c = run(tmem_st_bench<NW>, NW * 32);                                                            \
    printf("tmem_st  warps=%2d: %8.0f cyc  %6.1f B/clk/SM\n", NW, c, (double)NW * 32 * 32 * 4 * kIters / c); \
  }
  ST(4) ST(8) ST(16)
#define ALU(NW, M)                                                                                        \
  {                                                                                                       \
    double c = runf(alu_bench<NW, M>, NW * 32);                                                            \
    printf("%s warps=%2d: %8.0f cyc  %6.1f ops/clk/SM\n", M == 0 ? "ex2 " : M == 2 ? "f2fp" : M == 3 ? "ex2+f2fp" : M == 4 ? "cvt+ex2.f16x2" : M == 5 ? "ex2.f16x2" : "fma ", NW, c, \
           (double)NW * 32 * 8 * kIters / c);                                                             \
  }
  ALU(4, 0) ALU(8, 0) ALU(8, 4) ALU(16, 4) ALU(8, 5) ALU(16, 5)
  return 0;
}
