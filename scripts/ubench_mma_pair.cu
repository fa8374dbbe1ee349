// tcgen05.mma throughput of the CTA-pair form (cta_group::2, M = 256 over two SMs) against the
// single-CTA form (M = 128) at N = 64 / 128 / 256, SS operands, K- or MN-major B: cycles per
// instruction (K = 16) measured by the issuing thread over a long chain of MMAs into one
// accumulator, then the per-SM rate.  Question it answers (DESIGN (f) 1): does a pair MMA at
// N = 128 run at the single-CTA rate per SM (as the 256-wide GEMM tiles do at N = 256)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2507_05411_b200/csrc \
//     -I include scripts/ubench_mma_pair.cu -o scripts/bin/ubench_mma_pair
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace cb;
constexpr int kIters = 1024;

__device__ __forceinline__ void umma_ts_pair(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

// PAIR: cta_group::2 (cluster of 2, leader issues) or cta_group::1; BMN: B MN-major; TS: A from
// TMEM (columns 256.., the accumulator at column 0)
template <int PAIR, int N, int BMN, int TS = 0>
__global__ void __launch_bounds__(128, 1) mma_bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_async_smem();
  if (warp == 0) {
    if (PAIR)
      tmem_alloc_pair(&slot, 512);
    else
      tmem_alloc(&slot, 512);
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool leader = !PAIR || cluster_ctarank() == 0;
  if (threadIdx.x == 0 && leader) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N, 0, BMN);
    const uint64_t ad = sw128_desc(a, 16, 1024);
    const uint64_t bd = BMN ? sw128_desc(b, 8192, 1024) : sw128_desc(b, 16, 1024);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
      if (TS && PAIR)
        umma_ts_pair(tmem, tmem + 256, bd, idesc, it > 0);
      else if (TS)
        umma_f16_ts(tmem, tmem + 256, bd, idesc, it > 0);
      else if (PAIR)
        umma_f16_ss_pair(tmem, ad, bd, idesc, it > 0);
      else
        umma_f16_ss(tmem, ad, bd, idesc, it > 0);
    }
    if (PAIR)
      umma_commit_pair_mc(&bar, 0x3);
    else
      umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (threadIdx.x == 0 && PAIR) {
    mbar_wait(&bar, 0);  // the leader's commit is multicast to both CTAs
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (PAIR)
      tmem_dealloc_pair(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

template <int PAIR, int N, int BMN, int TS = 0>
void run(const char* name, int ctas) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * ctas);
  cudaMemset(d, 0, sizeof(unsigned long long) * ctas);
  const int smem_bytes = 98304;
  cudaFuncSetAttribute(mma_bench<PAIR, N, BMN, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, mma_bench<PAIR, N, BMN, TS>, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      return;
    }
  }
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
  double sum = 0;
  int cnt = 0;
  for (int i = 0; i < ctas; ++i)
    if (h[i]) {
      sum += h[i];
      ++cnt;
    }
  const double cyc = sum / cnt / kIters;
  // per-SM MACs per cycle: a pair instruction covers 256 x N x 16 on two SMs
  const double macs_per_sm = (PAIR ? 128.0 : 128.0) * N * 16 / cyc;
  printf("%-34s %7.1f cycles/MMA  %7.0f MAC/clk/SM  (%d issuing CTAs)\n", name, cyc, macs_per_sm, cnt);
  cudaFree(d);
}

int main() {
  for (int ctas : {2, 296}) {
    printf("--- %d CTAs\n", ctas);
    run<0, 64, 0>("1-CTA  M128 N64  B K-major", ctas);
    run<0, 128, 0>("1-CTA  M128 N128 B K-major", ctas);
    run<0, 256, 0>("1-CTA  M128 N256 B K-major", ctas);
    run<1, 64, 0>("pair   M256 N64  B K-major", ctas);
    run<1, 128, 0>("pair   M256 N128 B K-major", ctas);
    run<1, 256, 0>("pair   M256 N256 B K-major", ctas);
    run<1, 128, 1>("pair   M256 N128 B MN-major", ctas);
    run<1, 256, 1>("pair   M256 N256 B MN-major", ctas);
    run<0, 128, 1, 1>("1-CTA  M128 N128 TS B MN-major", ctas);
    run<1, 128, 1, 1>("pair   M256 N128 TS B MN-major", ctas);
    run<1, 128, 0, 1>("pair   M256 N128 TS B K-major", ctas);
  }
  return 0;
}
