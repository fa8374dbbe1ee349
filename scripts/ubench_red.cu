// Microbenchmark: throughput of accumulating 128x128 f32 tiles (64 KB) into L2-resident
// global memory from every SM — the dQ reduction a fused attention backward would issue per
// (key tile, query tile).  Modes:
//   0 red.global.add.v4.f32, one tile row per lane (the tcgen05.ld 32x32b register layout)
//   1 red.global.add.v4.f32, coalesced (lanes on consecutive 16-byte chunks of a row)
//   2 ld.v4 + add + st.v4, coalesced (ordered read-modify-write)
//   3 cp.reduce.async.bulk .add.f32 from shared memory (8 x 8 KB per tile, one thread)
//   4 st.v4 coalesced (plain write bandwidth)
//   5 red.global.add.v2.f32 in the tcgen05.ld 16x256b register layout (4 lanes cover 32 B of a row)
//   6 mode 5 + ~2000 cycles of simulated work per tile (spin)
//   7 mode 6 + deterministic ordering: the CTAs of a group of 32 accumulate each tile in CTA
//     order (acquire a per-tile flag == rank, reds, __threadfence, release flag = rank + 1)
// Destinations: "disjoint" (each CTA cycles over its own 8 tiles) or "shared" (the 32 CTAs of
// a group cycle over the same 32 tiles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/ubench_red.cu -o ubench_red
#include <cstdint>
#include <cstdio>

constexpr int kRows = 128, kCols = 128, kTileF = kRows * kCols;
constexpr int kIter = 256;

__device__ __forceinline__ void red4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void red2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ unsigned g_flags[8][kIter];

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float* dst, int shared_dst) {
  extern __shared__ __align__(128) float sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (MODE == 3) {
    for (int i = tid; i < kTileF; i += 256) sm[i] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  for (int it = 0; it < kIter; ++it) {
    const int tile = shared_dst ? (blockIdx.x / 32) * 32 + (it + blockIdx.x) % 32 : blockIdx.x * 8 + it % 8;
    float* t = dst + (size_t)tile * kTileF;
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    if (MODE == 0) {
      // warp w: rows (w % 4) * 32 + lane, columns [64 (w / 4), +64)
      float* r = t + ((warp & 3) * 32 + lane) * kCols + (warp >> 2) * 64;
#pragma unroll
      for (int c = 0; c < 16; ++c) red4(r + 4 * c, v);
    } else if (MODE == 1) {
#pragma unroll 4
      for (int i = tid; i < kTileF / 4; i += 256) red4(t + 4 * i, v);
    } else if (MODE == 2) {
#pragma unroll 4
      for (int i = tid; i < kTileF / 4; i += 256) {
        float4 a = reinterpret_cast<float4*>(t)[i];
        a.x += v.x;
        a.y += v.y;
        a.z += v.z;
        a.w += v.w;
        reinterpret_cast<float4*>(t)[i] = a;
      }
    } else if (MODE >= 5) {
      if (MODE >= 6) {
        const long long t0 = clock64();
        while (clock64() - t0 < 2000) {
        }
      }
      const int grp = blockIdx.x / 32, rank = blockIdx.x % 32;
      if (MODE == 7) {
        if (tid == 0) {
          unsigned f;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(&g_flags[grp][it]));
          } while (f != (unsigned)rank);
        }
        __syncthreads();
      }
      float* tt = MODE == 7 ? dst + (size_t)((grp * kIter + it) % (gridDim.x * 8)) * kTileF : t;
      const int row0 = (warp & 3) * 32, col0 = (warp >> 2) * 64;
#pragma unroll
      for (int rb = 0; rb < 32; rb += 8)
#pragma unroll
        for (int cb = 0; cb < 64; cb += 8)
          red2(tt + (row0 + rb + (lane >> 2)) * kCols + col0 + cb + (lane & 3) * 2, 1.f, 2.f);
      if (MODE == 7) {
        __threadfence();
        __syncthreads();
        if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&g_flags[grp][it]), "r"(rank + 1));
      }
    } else if (MODE == 3) {
      if (tid == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                           t + c * 2048),
                       "r"((uint32_t)__cvta_generic_to_shared(sm + c * 2048)), "r"(8192)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    } else {
#pragma unroll 4
      for (int i = tid; i < kTileF / 4; i += 256) reinterpret_cast<float4*>(t)[i] = v;
    }
  }
  if (MODE == 3 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE>
float run(float* dst, int shared_dst, int nsm) {
  const int smem = MODE == 3 ? kTileF * 4 : 0;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (MODE != 7) k<MODE><<<nsm, 256, smem>>>(dst, shared_dst);
  cudaEvent_t a, b;
  if (MODE == 7) {
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
      static unsigned z[8][kIter];
      cudaMemcpyToSymbol(g_flags, z, sizeof(z));
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<MODE><<<nsm, 256, smem>>>(dst, shared_dst);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float m;
      cudaEventElapsedTime(&m, a, b);
      ms += m;
    }
    return ms / 3;
  }
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<MODE><<<nsm, 256, smem>>>(dst, shared_dst);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  return ms / 5;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* dst;
  cudaMalloc(&dst, (size_t)nsm * 8 * kTileF * 4 + (size_t)160 * kTileF * 4);
  cudaMemset(dst, 0, (size_t)nsm * 8 * kTileF * 4);
  const char* names[8] = {"red.v4 row/lane", "red.v4 coalesced", "ld+add+st", "bulk reduce", "st.v4",
                          "red.v2 16x256b",  "v2 + 2000cyc work", "v2+work+ordered"};
  k<7><<<nsm, 256>>>(dst, 0);  // the first run of mode 7 waits on zeroed flags (static init)
  cudaDeviceSynchronize();
  for (int sh = 0; sh < 2; ++sh)
    for (int m = 0; m < 8; ++m) {
      if (sh && m == 7) continue;
      float ms = 0;
      switch (m) {
        case 0: ms = run<0>(dst, sh, nsm); break;
        case 1: ms = run<1>(dst, sh, nsm); break;
        case 2: ms = run<2>(dst, sh, nsm); break;
        case 3: ms = run<3>(dst, sh, nsm); break;
        case 5: ms = run<5>(dst, sh, nsm); break;
        case 6: ms = run<6>(dst, sh, nsm); break;
        case 7: ms = run<7>(dst, sh, nsm); break;
        default: ms = run<4>(dst, sh, nsm); break;
      }
      const double bytes = (double)nsm * kIter * kTileF * 4;
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("%-8s %-18s %8.3f ms  %7.1f GB/s  %6.0f B/clk/SM @max clock  (%.0f cycles per 64 KB tile at 1.9 GHz)\n",
             sh ? "shared" : "disjoint", names[m], ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / (clk * 1e3) / nsm,
             ms * 1e-3 * 1.9e9 / kIter);
    }
  return 0;
}
