// Pipeline trace of the tcgen05 attention forward: builds attn_tc.cu with CB_ATTN_TRACE and
// prints, for CTA (0,0,0) of a 1B-shape launch, the clock64 of every MMA issue and softmax
// phase per K/V block.  Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE \
//     -I paper_2507_05411_b200/csrc -I include scripts/attn_trace.cu \
//     paper_2507_05411_b200/csrc/runtime.cu -o scripts/bin/attn_trace -lcuda
#include <cstdio>
#include <vector>

#include "../paper_2507_05411_b200/csrc/attn_tc.cu"

int main() {
  const int B = 8, T = 4096, H = 16, hd = 128;
  const size_t n = (size_t)B * T * H * hd;
  std::vector<__nv_bfloat16> h(n);
  uint32_t x = 12345;
  for (size_t i = 0; i < n; ++i) {
    x = x * 1664525u + 1013904223u;
    h[i] = __float2bfloat16(((x >> 8) & 0xffff) / 65536.f - 0.5f);
  }
  void *q, *k, *v, *o;
  float* lse;
  cudaMalloc(&q, n * 2);
  cudaMalloc(&k, n * 2);
  cudaMalloc(&v, n * 2);
  cudaMalloc(&o, n * 2);
  cudaMalloc(&lse, (size_t)B * H * T * 4);
  cudaMemcpy(q, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(k, h.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(v, h.data(), n * 2, cudaMemcpyHostToDevice);
  cb::AttnGeom g{B, T, H, H, hd, H * hd, H * hd, H * hd, H * hd, 0.08838834764831845f};
  for (int it = 0; it < 3; ++it) {
    if (int s = cb::attn_fwd_tc(g, q, k, v, o, lse, 0)) {
      printf("launch failed %d\n", s);
      return 1;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("kernel failed\n");
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) cb::attn_fwd_tc(g, q, k, v, o, lse, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 10;
  printf("emu %d: fwd %.3f ms  %.1f TFLOP/s\n", cb::tca::kEmuPairs, ms, 4.0 * B * T * (double)T * H * hd / ms / 1e9);
  unsigned long long tr[16][64];
  cudaMemcpyFromSymbol(tr, cb::tca::g_trace, sizeof(tr));
  const unsigned long long t0 = tr[0][0];
  const char* names[16] = {"S_A", "S_B", "PV_A", "PV_B", "A.st", "A.mx", "A.end", "B.st",
                           "B.mx", "B.end", "PVAdone", "-", "ld.K", "ld.V", "PVAwait", "PVBdone"};
  printf("  j");
  for (int e = 0; e < 16; ++e)
    if (e != 11) printf(" %7s", names[e]);
  printf("\n");
  for (int j = 0; j < 32; ++j) {
    printf("%3d", j);
    for (int e = 0; e < 16; ++e)
      if (e != 11) printf(" %7lld", (long long)(tr[e][j] - t0));
    printf("\n");
  }
  return 0;
}
