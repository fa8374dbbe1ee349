// Pipeline trace + timing of the tcgen05 attention backward kernels (CB_ATTN_TRACE build),
// 1B step shape.  Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCB_ATTN_TRACE \
//     -I paper_2507_05411_b200/csrc -I include scripts/attn_bwd_trace.cu \
//     paper_2507_05411_b200/csrc/runtime.cu -o scripts/bin/attn_bwd_trace -lcuda
#include <cstdio>
#include <vector>
#include <algorithm>

#include "../paper_2507_05411_b200/csrc/attn_tc.cu"
#include "../paper_2507_05411_b200/csrc/attn_tc_bwd.cu"

int main(int argc, char** argv) {
  // "single" / "pair" (dQ on pairs) / "both" (dQ and dK/dV on pairs)
  cb::tcb::g_dq_pair = argc > 1 && (argv[1][0] == 'p' || argv[1][0] == 'b');
  cb::tcb::g_dkdv_pair = argc > 1 && argv[1][0] == 'b';
  const int B = 8, T = 4096, H = 16, hd = 128;
  const size_t n = (size_t)B * T * H * hd;
  std::vector<__nv_bfloat16> h(n);
  uint32_t x = 12345;
  for (size_t i = 0; i < n; ++i) {
    x = x * 1664525u + 1013904223u;
    h[i] = __float2bfloat16(((x >> 8) & 0xffff) / 65536.f - 0.5f);
  }
  void *q, *k, *v, *o, *g, *dq, *dk, *dv;
  float *lse, *delta;
  for (void** p : {&q, &k, &v, &o, &g, &dq, &dk, &dv}) cudaMalloc(p, n * 2);
  cudaMalloc(&lse, (size_t)B * H * T * 4);
  cudaMalloc(&delta, (size_t)B * H * T * 4);
  cudaMemset(delta, 0, (size_t)B * H * T * 4);
  for (void* p : {q, k, v, g}) cudaMemcpy(p, h.data(), n * 2, cudaMemcpyHostToDevice);
  cb::AttnGeom geo{B, T, H, H, hd, H * hd, H * hd, H * hd, H * hd, 0.08838834764831845f};
  cb::attn_fwd_tc(geo, q, k, v, o, nullptr, lse, 0);
  auto bwd = [&]() {
    return cb::attn_bwd_tc(geo, q, k, v, g, H * hd, lse, delta, dq, H * hd, dk, H * hd, dv, H * hd, 0, nullptr, nullptr,
                           nullptr);
  };
  for (int it = 0; it < 3; ++it)
    if (int s = bwd()) {
      printf("launch failed %d\n", s);
      return 1;
    }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("kernel failed\n");
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) bwd();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 10;
  printf("bwd %.3f ms  %.1f TFLOP/s (5 GEMMs algorithmic)\n", ms, 10.0 * B * T * (double)T * H * hd / ms / 1e9);
  unsigned long long tr[24][64];
  cudaMemcpyFromSymbol(tr, cb::tcb::g_btrace, sizeof(tr));
  const unsigned long long t0 = tr[1][0];
  const char* names[10] = {"dV", "S+1", "dK", "dP+1", "c.S", "c.P", "c.dP", "c.dS", "ld.Q", "ld.dO"};
  printf("  u");
  for (int e = 0; e < 10; ++e) printf(" %7s", names[e]);
  printf("\n");
  for (int j = 0; j < 16; ++j) {
    printf("%3d", j);
    for (int e = 0; e < 10; ++e) printf(" %7lld", (long long)(tr[e][j] - t0));
    printf("\n");
  }
  const unsigned long long t1 = tr[10][0];
  const char* qn[8] = {"S", "dQ", "dP", "c.S", "c.dP", "c.dS", "ld.K", "ld.V"};
  printf("dq kernel\n  j");
  for (int e = 0; e < 8; ++e) printf(" %7s", qn[e]);
  printf("\n");
  for (int j = 0; j < 12; ++j) {
    printf("%3d", j);
    for (int e = 0; e < 8; ++e) printf(" %7lld", (long long)(tr[10 + e][j] - t1));
    printf("\n");
  }
  printf("dq: k_full wait per tile (S issue ready -> K tile present), cycles:");
  for (int j = 4; j < 12; ++j) printf(" %lld", (long long)(tr[10][j] - tr[18][j]));
  printf("\n");
  if (tr[19][0] && tr[21][0])
    printf("dkdv CTA (0,0,0), single-CTA sweep: compute start %lld, last tile's dV issue %lld, last MMA done %lld, "
           "epilogue stores issued %lld (cycles from the first S)\n",
           (long long)(tr[19][0] - t0), (long long)(tr[0][31] - t0), (long long)(tr[20][0] - t0),
           (long long)(tr[21][0] - t0));
  printf("steady-state period (tiles 4..15): dkdv %.0f cycles, dq %.0f cycles\n", (tr[0][15] - tr[0][4]) / 11.0,
         (tr[11][15] - tr[11][4]) / 11.0);
  // per-CTA timeline of the last launch: CTA duration, gap to the next CTA on the same SM
  static unsigned long long ct[2][8192][3];
  cudaMemcpyFromSymbol(ct, cb::tcb::g_cta, sizeof(ct));
  const int ncta = (T / 128) * H * B;
  for (int kk = 0; kk < 2; ++kk) {
    unsigned long long lo = ~0ull, hi = 0;
    double dur = 0, gap = 0;
    int ngap = 0;
    std::vector<std::vector<std::pair<unsigned long long, unsigned long long>>> per(160);
    for (int i = 0; i < ncta; ++i) {
      lo = std::min(lo, ct[kk][i][0]);
      hi = std::max(hi, ct[kk][i][1]);
      dur += (double)(ct[kk][i][1] - ct[kk][i][0]);
      per[ct[kk][i][2] % 160].push_back({ct[kk][i][0], ct[kk][i][1]});
    }
    int nsm = 0;
    double first_start = 0, last_end = 0;
    for (auto& v : per) {
      if (v.empty()) continue;
      ++nsm;
      std::sort(v.begin(), v.end());
      first_start += (double)(v.front().first - lo);
      last_end += (double)(hi - v.back().second);
      for (size_t j = 1; j < v.size(); ++j) {
        gap += (double)v[j].first - (double)v[j - 1].second;
        ++ngap;
      }
    }
    printf("%s: span %.1f us, %d SMs, %d CTAs, mean CTA %.2f us, mean gap between CTAs on an SM %.2f us, "
           "mean first start %.2f us, mean idle tail %.2f us\n",
           kk ? "dq" : "dkdv", (hi - lo) / 1e3, nsm, ncta, dur / ncta / 1e3, ngap ? gap / ngap / 1e3 : 0.0,
           first_start / nsm / 1e3, last_end / nsm / 1e3);
  }
  return 0;
}
