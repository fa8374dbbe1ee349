// tcgen05.mma issue/throughput microbenchmark (kind::f16, M=128, cta_group::1): cycles per
// instruction for SS vs TS (A from TMEM) operands, K- vs MN-major B, N = 128 / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2507_05411_b200/csrc \
//     -I include scripts/ubench_mma.cu -o scripts/bin/ubench_mma
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace cb;
constexpr int kIters = 512;

// MODE 0: SS K-major B; 1: SS MN-major B; 2: TS + MN-major B; 3: TS + K-major B
// COMMIT > 0: a tcgen05.commit (to a barrier nobody waits on) after every COMMIT MMAs
template <int MODE, int N, int LDW, int COMMIT = 0>
__global__ void __launch_bounds__(384, 1) mma_bench(unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) stop = 0;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_mbar_init();
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, (MODE == 1 || MODE == 2) ? 1 : 0);
    const unsigned long long t0 = clock64();
    if (MODE == 9) {
      // dq-like: per iteration S (SS -> cols 0..127), dP (SS -> 128..255), dQ (TS A = cols 0..63 -> 384..511)
      const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);
      for (int it = 0; it < kIters / 24; ++it) {
        for (int k = 0; k < 8; ++k)
          umma_f16_ss(tmem + 0, sw128_desc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                      sw128_desc(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), idesc, k > 0);
        umma_commit(&bar2);
        for (int k = 0; k < 8; ++k)
          umma_f16_ss(tmem + 128, sw128_desc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                      sw128_desc(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), idesc, k > 0);
        umma_commit(&bar2);
        for (int k = 0; k < 8; ++k)
          umma_f16_ts(tmem + 384, tmem + (k >> 2) * 64 + (k & 3) * 8, sw128_desc(b + k * 2048, 16384, 1024), id_acc, 1);
        umma_commit(&bar2);
      }
    }
    for (int it = 0; it < (MODE == 9 ? 0 : kIters); ++it) {
      const int k = it & 7;
      const uint64_t bd = (MODE == 1 || MODE == 2) ? sw128_desc(b + k * 2048, 16384, 1024)
                                                  : sw128_desc(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      if (MODE >= 2)
        umma_f16_ts(tmem + 256, tmem + k * 8, bd, idesc, 1);
      else
        umma_f16_ss(tmem + 256, sw128_desc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc, 1);
      if (COMMIT > 0 && (it % COMMIT) == COMMIT - 1) umma_commit(&bar2);
    }
    const unsigned long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t2 = clock64();
    cyc[blockIdx.x * 2] = t1 - t0;
    cyc[blockIdx.x * 2 + 1] = t2 - t0;
    stop = 1;
  }
  if (LDW < 0 && warp >= 4 && warp < 8) {
    // shared-memory store traffic from other warps (region 48..64 KB, unused by the MMAs)
    uint4* dst = reinterpret_cast<uint4*>(smem + 49152) + (threadIdx.x & 127);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i * 128 % 1024] = v;
      v.x += 1;
    }
  }
  if (LDW > 0 && warp >= 4 && warp < 4 + LDW) {
    // TMEM traffic from other warps (columns 0..255, the MMA accumulates into 256..)
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp - 4) >> 2) * 64;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[32];
      tmem_ld32(base, v);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) acc += v[i];
      if (LDW > 4) {
        uint32_t p[16];
        for (int i = 0; i < 16; ++i) p[i] = v[i] ^ acc;
        tmem_st16(base + 32, p);
        tmem_st_wait();
      }
    }
    if (acc == 0x12345) cyc[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE, int N, int LDW = 0, int COMMIT = 0>
void run(const char* name, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(mma_bench<MODE, N, LDW, COMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  mma_bench<MODE, N, LDW, COMMIT><<<grid, 384, 65536 + 1024>>>(d);
  mma_bench<MODE, N, LDW, COMMIT><<<grid, 384, 65536 + 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  unsigned long long h[296];
  cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
  double issue = 0, done = 0;
  for (int i = 0; i < grid; ++i) {
    issue += h[2 * i];
    done += h[2 * i + 1];
  }
  printf("%-28s ldw=%d commit/%d N=%3d grid=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (ideal %d)\n", name, LDW, COMMIT, N, grid,
         issue / grid / kIters, done / grid / kIters, 128 * N / 256);
  cudaFree(d);
}

int main() {
  for (int grid : {148}) {
    run<0, 128>("SS", grid);
    run<9, 128>("dq pattern (kIters/24*24)", grid);
  }
  return 0;
}
