// GEMM for every contraction on the decoder step:  D = alpha * op(A) @ op(B) (+ D) (+ R)
//
// Replaces the reference's `x @ param(...)` products (reference layers.py:167, 340-348,
// 412-416, 516, 597) and supplies the backward products the reference never runs.
//
// Two engines behind one entry point (cb_gemm):
//   * gemm_tc   — bf16 operands, f32 accumulation in TMEM, tcgen05.mma issued by one
//                 thread, operands staged by TMA into 128B-swizzled shared memory, a
//                 persistent warp-specialised CTA per SM (TMA warp, MMA warp, 4 epilogue
//                 warps) with a 2-deep TMEM accumulator so the epilogue of tile i overlaps
//                 the MMAs of tile i+1.  Both K-major and MN-major operands are native
//                 (UMMA descriptor major bits), so forward (x@W), dgrad (dY@W^T) and wgrad
//                 (X^T@dY) all run on the reference's [in, out] weight layout with no
//                 transposed copies.
//   * gemm_simt — f32 FMA tiles; the fp32 parity mode (1e-5 contract) and shapes TMA
//                 cannot describe (row strides not 16-byte aligned, e.g. hidden 341).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "composer_b200.h"

namespace cb {

struct Epi {
  void* D;
  int64_t ldd;
  int d_f32;
  const void* R;
  int64_t ldr;
  int r_f32;
  float alpha;
  int accumulate;
  int M, N;
  // optional RoPE on output columns [0, rope_cols): rows are tokens (position = row % rope_T),
  // interleaved pairs inside heads of rope_hd columns (reference layers.py:235-257)
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int rope_T = 0, rope_hd = 0, rope_cols = 0;
  // gated-activation epilogues (CTA-pair engine, bf16): glu = 1 forward — the tile's 256
  // columns are 128 columns of the a half and the same 128 of the g half of pre = x @ [W1|Wg]
  // (D = pre [M, 2H]); also writes hidden = act0(a) * act1(g) to glu_out [M, H].
  // glu = 2 backward — the accumulator is dhidden [M, H] (never stored); reads pre from
  // glu_pre and writes dpre = [da | dg] to glu_out [M, 2H].
  int glu = 0, glu_h = 0, glu_a0 = 0, glu_a1 = 0;
  void* glu_out = nullptr;
  int64_t ld_glu_out = 0;
  const void* glu_pre = nullptr;
  int64_t ld_glu_pre = 0;
  // AdamW fused into a weight-gradient GEMM (cb_gemm_adamw): the accumulator is the whole
  // gradient of the output elements (D is only the address frame, never read or written); the
  // epilogue applies the update to the f32 master / m / v and writes the bf16 working copy,
  // all laid out like D (same row stride).  g = fma(acc, alpha, 0) — the value the unfused
  // path stores into a cleared gradient buffer — then adam_elem exactly as cb_adamw.
  float* ad_p = nullptr;
  float* ad_m = nullptr;
  float* ad_v = nullptr;
  __nv_bfloat16* ad_bf = nullptr;
  float ad_lr = 0.f, ad_b1 = 0.f, ad_b2 = 0.f, ad_eps = 0.f, ad_wd = 0.f, ad_bc1 = 1.f, ad_bc2 = 1.f;
};

// L2 prefetch of one output row's optimizer state (master / m / v) over a tile's columns: the
// fused-AdamW epilogue issues it for the next tile while the current one drains, so the
// epilogue's loads hit L2 instead of waiting on HBM with only 4 warps of loads in flight.
__device__ __forceinline__ void epi_adam_prefetch(const Epi& e, int row, int col0, int ncols) {
  if (!e.ad_p || row >= e.M) return;
  const int64_t base = (int64_t)row * e.ldd + col0;
  for (int c = 0; c < ncols && col0 + c < e.N; c += 32) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(e.ad_p + base + c));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(e.ad_m + base + c));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(e.ad_v + base + c));
  }
}

__device__ __forceinline__ void epi_adam1(const Epi& e, int64_t di, float acc) {
  float p = e.ad_p[di], m = e.ad_m[di], v = e.ad_v[di];
  adam_elem(p, __fmul_rn(__fmaf_rn(acc, e.alpha, 0.f), 1.f), m, v, e.ad_lr, e.ad_b1, e.ad_b2, e.ad_eps, e.ad_wd,
            e.ad_bc1, e.ad_bc2);
  e.ad_p[di] = p;
  e.ad_m[di] = m;
  e.ad_v[di] = v;
  if (e.ad_bf) e.ad_bf[di] = __float2bfloat16_rn(p);
}

__device__ __forceinline__ float epi_load(const void* p, int64_t idx, int f32) {
  return f32 ? reinterpret_cast<const float*>(p)[idx] : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
}

__device__ __forceinline__ void epi_store1(const Epi& e, int r, int c, float v) {
  if (e.ad_p) {
    epi_adam1(e, (int64_t)r * e.ldd + c, v);
    return;
  }
  v *= e.alpha;
  const int64_t di = (int64_t)r * e.ldd + c;
  if (e.accumulate) v += epi_load(e.D, di, e.d_f32);
  if (e.R) v += epi_load(e.R, (int64_t)r * e.ldr + c, e.r_f32);
  if (e.d_f32)
    reinterpret_cast<float*>(e.D)[di] = v;
  else
    reinterpret_cast<__nv_bfloat16*>(e.D)[di] = __float2bfloat16_rn(v);
}

// ======================================================================================
// tcgen05 engine
// ======================================================================================
namespace tc {
// 1 (default): the CTA-pair engine's epilogues go through the per-warp shared-memory stage
// (coalesced global I/O); 0: per-lane stores (A/B and tests, cb_gemm_set_staged_epilogue)
// bits: kStagedBf16 | kStagedGlu (default: both)
__constant__ int g_epi_staged = 3;
constexpr int kStagedBf16 = 1, kStagedGlu = 2;
constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kThreads = 256;
constexpr int kGroupM = 16;  // raster: 16 M-tiles share each N column step (L2 reuse)
// raster group height actually used (cb_gemm_set_raster; A/B of the L2 reuse pattern)
__constant__ int g_group_m = kGroupM;

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
};

struct Args {
  int M, N, K;
  int a_mn, b_mn;
  int tiles_m, tiles_n;
  Epi e;
  // split-K (CTA-pair engine): slice s of every tile covers k-blocks [s*nk/S, (s+1)*nk/S)
  // and stores its raw f32 partial to ws[s] ([M][N]); splitk_reduce_k sums the slices in
  // order and applies the epilogue (deterministic: no atomics)
  int splits = 1;
  float* ws = nullptr;
  // grouped launch (all MoE experts in one persistent launch, CTA-pair engine only):
  // grp_off = device [G+1] row offsets, each a multiple of 256, read by the kernel (no host
  // round trip).  grp_mode 1: the groups split the rows of A and D; the tiles of group g read
  // B at a coordinate offset g * b_grp_stride along K (MN-major B, stacked [G*K][N]) or along
  // N (K-major B, stacked [G*N][K]); tiles_m is taken from grp_off[G].  grp_mode 2: the groups
  // split the K rows of A and B (both MN-major, stacked along K); group g writes D rows
  // [g*M, (g+1)*M) and an empty group writes nothing.
  const int* grp_off = nullptr;
  int grp_mode = 0, G = 0;
  int64_t b_grp_stride = 0;
};
constexpr int kMaxGroups = 64;

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int gmx = g_group_m;
  const int per_group = gmx * tiles_n;
  const int g = t / per_group;
  const int r = t - g * per_group;
  const int gm0 = g * gmx;
  const int gsz = min(gmx, tiles_m - gm0);
  tm = gm0 + r % gsz;
  tn = r / gsz;
}

// One 32-column accumulator chunk of one output row through the epilogue: optional RoPE
// rotation of the columns [0, rope_cols), then alpha / accumulate / residual and the store.
__device__ __forceinline__ void epi_chunk(const Epi& e, uint32_t (&v)[32], int row, int col0) {
  if (e.rope_cos && col0 < e.rope_cols) {
    // 32 columns = 16 pairs of one head (rope_hd % 32 == 0 is required on this path)
    const int half = e.rope_hd >> 1;
    const int p0 = (col0 % e.rope_hd) >> 1;
    const int64_t tb = (int64_t)(row % e.rope_T) * half + p0;
    const float4* cs4 = reinterpret_cast<const float4*>(e.rope_cos + tb);
    const float4* sn4 = reinterpret_cast<const float4*>(e.rope_sin + tb);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 cq = cs4[j], sq = sn4[j];
      const float cc[4] = {cq.x, cq.y, cq.z, cq.w}, ss[4] = {sq.x, sq.y, sq.z, sq.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = (j * 4 + i) * 2;
        const float ev = __uint_as_float(v[k]), od = __uint_as_float(v[k + 1]);
        v[k] = __float_as_uint(ev * cc[i] - od * ss[i]);
        v[k + 1] = __float_as_uint(ev * ss[i] + od * cc[i]);
      }
    }
  }
  const bool full_chunk = col0 + 32 <= e.N;
  if (e.ad_p) {
    const int64_t di = (int64_t)row * e.ldd + col0;
    const bool v4 = full_chunk && (e.ldd & 7) == 0 &&
                    !((reinterpret_cast<uintptr_t>(e.ad_p) | reinterpret_cast<uintptr_t>(e.ad_m) |
                       reinterpret_cast<uintptr_t>(e.ad_v)) & 15) && !(reinterpret_cast<uintptr_t>(e.ad_bf) & 15);
    if (v4) {
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) {
        const int64_t i = di + g8 * 8;
        float4 P[2], Mv[2], V[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          P[h] = reinterpret_cast<const float4*>(e.ad_p + i)[h];
          Mv[h] = reinterpret_cast<const float4*>(e.ad_m + i)[h];
          V[h] = reinterpret_cast<const float4*>(e.ad_v + i)[h];
        }
        float* pp = &P[0].x;
        float* mm = &Mv[0].x;
        float* vv = &V[0].x;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          adam_elem(pp[j], __fmul_rn(__fmaf_rn(__uint_as_float(v[g8 * 8 + j]), e.alpha, 0.f), 1.f), mm[j], vv[j],
                    e.ad_lr, e.ad_b1, e.ad_b2, e.ad_eps, e.ad_wd, e.ad_bc1, e.ad_bc2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          reinterpret_cast<float4*>(e.ad_p + i)[h] = P[h];
          reinterpret_cast<float4*>(e.ad_m + i)[h] = Mv[h];
          reinterpret_cast<float4*>(e.ad_v + i)[h] = V[h];
        }
        if (e.ad_bf) {
          uint4 t;
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
          for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(pp[2 * j], pp[2 * j + 1]);
          *reinterpret_cast<uint4*>(e.ad_bf + i) = t;
        }
      }
    } else {
      const int lim = min(32, e.N - col0);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < lim) epi_adam1(e, di + j, __uint_as_float(v[j]));
    }
    return;
  }
  const bool fast = full_chunk && !e.accumulate && !e.R && e.alpha == 1.f && !e.d_f32 && ((e.ldd & 7) == 0) &&
                    ((reinterpret_cast<uintptr_t>(e.D) & 15) == 0);
  const bool vec = full_chunk && ((e.ldd & 7) == 0) && ((reinterpret_cast<uintptr_t>(e.D) & 31) == 0) &&
                   (!e.R || (((e.ldr & 7) == 0) && ((reinterpret_cast<uintptr_t>(e.R) & 31) == 0)));
  if (!fast && vec && e.d_f32 && ((e.R && e.r_f32) != (bool)e.accumulate)) {
    // f32 output plus exactly one f32 addend (the residual R, or D itself when accumulating):
    // all of the chunk's addend loads are issued before any store (one memory latency per
    // chunk instead of one per 8 columns)
    const int64_t di = (int64_t)row * e.ldd + col0;
    const float4* src = e.accumulate
                            ? reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.D) + di)
                            : reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.R) + (int64_t)row * e.ldr + col0);
    float4 add[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) add[i] = src[i];
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.D) + di);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      d[i] = make_float4(fmaf(__uint_as_float(v[4 * i]), e.alpha, add[i].x),
                         fmaf(__uint_as_float(v[4 * i + 1]), e.alpha, add[i].y),
                         fmaf(__uint_as_float(v[4 * i + 2]), e.alpha, add[i].z),
                         fmaf(__uint_as_float(v[4 * i + 3]), e.alpha, add[i].w));
  } else if (!fast && vec) {
    // general epilogue, 8 columns (one 16/32-byte vector) at a time
#pragma unroll
    for (int g8 = 0; g8 < 4; ++g8) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = __uint_as_float(v[g8 * 8 + i]) * e.alpha;
      const int64_t di = (int64_t)row * e.ldd + col0 + g8 * 8;
      if (e.accumulate) {
        if (e.d_f32) {
          const float4* s = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.D) + di);
          const float4 a = s[0], b = s[1];
          o[0] += a.x; o[1] += a.y; o[2] += a.z; o[3] += a.w; o[4] += b.x; o[5] += b.y; o[6] += b.z; o[7] += b.w;
        } else {
          const uint4 t = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.D) + di);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h2[i]);
            o[2 * i] += f.x;
            o[2 * i + 1] += f.y;
          }
        }
      }
      if (e.R) {
        const int64_t ri = (int64_t)row * e.ldr + col0 + g8 * 8;
        if (e.r_f32) {
          const float4* s = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.R) + ri);
          const float4 a = s[0], b = s[1];
          o[0] += a.x; o[1] += a.y; o[2] += a.z; o[3] += a.w; o[4] += b.x; o[5] += b.y; o[6] += b.z; o[7] += b.w;
        } else {
          const uint4 t = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.R) + ri);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h2[i]);
            o[2 * i] += f.x;
            o[2 * i + 1] += f.y;
          }
        }
      }
      if (e.d_f32) {
        float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.D) + di);
        d[0] = make_float4(o[0], o[1], o[2], o[3]);
        d[1] = make_float4(o[4], o[5], o[6], o[7]);
      } else {
        uint4 t;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
        for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.D) + di) = t;
      }
    }
  } else if (fast) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.D) + (int64_t)row * e.ldd + col0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 pk;
      uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[j * 8 + 2 * h]), __uint_as_float(v[j * 8 + 2 * h + 1]));
        w[h] = *reinterpret_cast<uint32_t*>(&b2);
      }
      dst[j] = pk;
    }
  } else {
    const int lim = min(32, e.N - col0);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < lim) epi_store1(e, row, col0 + j, __uint_as_float(v[j]));
  }
}

// MC = 1: one CTA per 128 x BN tile.  MC = 2: a cluster of two CTAs computes two vertically
// adjacent tiles that share the B (weight) tile; each CTA loads half of B and multicasts it
// to both, so the L2->SM operand traffic per FLOP drops by a third (the kernel is L2-
// bandwidth-limited at 1-CTA: ~96 B/cycle/SM needed at peak MMA rate).
template <int BN, int MC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Args args) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = MC == 2 ? (int)cluster_ctarank() : 0;
  const int tiles_mg = (args.tiles_m + MC - 1) / MC;  // M-tile groups (pairs when MC == 2)
  const int num_units = tiles_mg * args.tiles_n;
  const int unit0 = MC == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int unit_stride = MC == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nk = (args.K + BK - 1) / BK;
  auto coords = [&](int u, int& tm, int& tn) {
    int tg;
    tile_coords(u, tiles_mg, args.tiles_n, tg, tn);
    tm = tg * MC + rank;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // both CTAs' MMAs must release a stage (multicast B lands in both)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  if (MC == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (whole warp, one elected lane issues) ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int u = unit0; u < num_units; u += unit_stride) {
      int tm, tn;
      coords(u, tm, tn);
      const int m0 = tm * BM, n0 = tn * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* a_dst = sA + stage * C::kABytes;
        uint8_t* b_dst = sB + stage * C::kBBytes;
        const int k0 = kb * BK;
        if (elect_one()) {
          mbar_expect_tx(&full[stage], C::kStageBytes);
          if (!args.a_mn) {
            tma_load_2d(a_dst, &tmA, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(a_dst + j * 8192, &tmA, &full[stage], m0 + 64 * j, k0);
          }
          if (MC == 1) {
            if (!args.b_mn) {
              tma_load_2d(b_dst, &tmB, &full[stage], k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_2d(b_dst + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
            }
          } else {
            // this CTA's half of B (rows [rank*BN/2, (rank+1)*BN/2) of the tile), to both CTAs
            constexpr int kHalf = BN / 2;
            uint8_t* hb = b_dst + rank * (kHalf * BK * 2);
            if (!args.b_mn) {
              tma_load_2d_mc(hb, &tmB, &full[stage], k0, n0 + rank * kHalf, 0x3);
            } else {
#pragma unroll
              for (int j = 0; j < kHalf / 64; ++j)
                tma_load_2d_mc(hb + j * 8192, &tmB, &full[stage], n0 + rank * kHalf + 64 * j, k0, 0x3);
            }
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // the whole warp walks the schedule (descriptors stay warp-uniform, in uniform
    // registers); one elected lane issues each k-block's MMAs
    const uint32_t idesc = idesc_bf16_f32(BM, BN, args.a_mn, args.b_mn);
    const uint64_t a0 = args.a_mn ? sw128_desc(smem_u32(sA), 8192, 1024) : sw128_desc(smem_u32(sA), 16, 1024);
    const uint64_t b0 = args.b_mn ? sw128_desc(smem_u32(sB), 8192, 1024) : sw128_desc(smem_u32(sB), 16, 1024);
    // per-K=16-step descriptor advance (16-byte units): MN-major +2048 B, K-major +32 B
    const uint64_t a_step = args.a_mn ? 128 : 2, b_step = args.b_mn ? 128 : 2;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = unit0; u < num_units; u += unit_stride, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = a0 + (uint64_t)(stage * (C::kABytes >> 4));
        const uint64_t bd = b0 + (uint64_t)(stage * (C::kBBytes >> 4));
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_f16_ss(d_tmem, ad + kk * a_step, bd + kk * b_step, idesc, (kb | kk) != 0);
          if (MC == 2)
            umma_commit_mc(&empty[stage], 0x3);  // release the stage in both CTAs (B is shared)
          else
            umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const Epi& e = args.e;
    int it = 0;
    if (e.ad_p && unit0 < num_units) {
      int tm, tn;
      coords(unit0, tm, tn);
      epi_adam_prefetch(e, tm * BM + q * 32 + lane, tn * BN, BN);
    }
    for (int u = unit0; u < num_units; u += unit_stride, ++it) {
      int tm, tn;
      coords(u, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (e.ad_p && u + unit_stride < num_units) {  // the next tile's optimizer state into L2
        int tm2, tn2;
        coords(u + unit_stride, tm2, tn2);
        epi_adam_prefetch(e, tm2 * BM + q * 32 + lane, tn2 * BN, BN);
      }
      const int row = tm * BM + q * 32 + lane;
      const bool row_ok = row < e.M;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        tmem_ld_wait();
        const int col0 = tn * BN + c * 32;
        if (!row_ok || col0 >= e.N) continue;
        epi_chunk(e, v, row, col0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  if (MC == 2)
    cluster_sync();  // no CTA leaves while its peer may still multicast into / commit to it
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// bf16 pack / unpack of 8 values (one 16-byte vector)
__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 t;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  return t;
}
__device__ __forceinline__ void unpack8(uint4 t, float* v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
// Gated activation act0(a) * act1(g) and its partials with the activation ids as template
// parameters (a runtime switch per element compiles to jump tables in the epilogue loop).
// (A0 / A1 = -1: the runtime ids r0 / r1 of the other pairs.)
template <int A0, int A1>
__device__ __forceinline__ float glu_f(float a, float g, int r0, int r1) {
  return act_f(A0 < 0 ? r0 : A0, a) * act_f(A1 < 0 ? r1 : A1, g);
}
template <int A0, int A1>
__device__ __forceinline__ void glu_df(float d, float a, float g, float& da, float& dg, int r0, int r1) {
  if (A0 == ACT_LINEAR && A1 == ACT_SILU) {  // SwiGLU: one sigmoid serves silu and silu'
    const float sg = stable_sigmoid(g);
    const float sl = g * sg;
    da = d * sl;
    dg = d * a * (sg + sl * (1.f - sg));
  } else {
    const int x0 = A0 < 0 ? r0 : A0, x1 = A1 < 0 ? r1 : A1;
    da = d * act_df(x0, a) * act_f(x1, g);
    dg = d * act_f(x0, a) * act_df(x1, g);
  }
}

// The gated epilogues' operands, passed by value (in registers) to the out-of-line tile
// functions.
struct Glu {
  __nv_bfloat16* pre;  // fwd: pre output (D); bwd: unused
  int64_t ldpre;
  __nv_bfloat16* out;  // fwd: hidden; bwd: dpre
  int64_t ldout;
  const __nv_bfloat16* pin;  // bwd: pre input
  int64_t ldpin;
  int h, n, a0, a1;
};

// forward gated epilogue for 32 columns: va / vg are the a / g accumulators of columns
// [col, col + 32) of each half; values are rounded to bf16 first, exactly as the unfused
// path reads them back from pre.
template <int A0, int A1>
__device__ __forceinline__ void glu_fwd_chunk(const Glu& q, const uint32_t (&va)[32], const uint32_t (&vg)[32],
                                              int row, int col) {
  __nv_bfloat16* pre = q.pre + (int64_t)row * q.ldpre;
  __nv_bfloat16* hid = q.out + (int64_t)row * q.ldout;
#pragma unroll
  for (int g8 = 0; g8 < 4; ++g8) {
    float a[8], g[8], h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __uint_as_float(va[g8 * 8 + i]);
      g[i] = __uint_as_float(vg[g8 * 8 + i]);
    }
    const uint4 pa = pack8(a), pg = pack8(g);
    *reinterpret_cast<uint4*>(pre + col + g8 * 8) = pa;
    *reinterpret_cast<uint4*>(pre + q.h + col + g8 * 8) = pg;
    unpack8(pa, a);
    unpack8(pg, g);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = glu_f<A0, A1>(a[i], g[i], q.a0, q.a1);
    *reinterpret_cast<uint4*>(hid + col + g8 * 8) = pack8(h);
  }
}
// backward gated epilogue for 32 columns of dhidden (rounded to bf16 like the stored dhidden
// of the unfused path); pa / pg hold the chunk's pre values (loaded ahead)
template <int A0, int A1>
__device__ __forceinline__ void glu_bwd_chunk(const Glu& q, const uint32_t (&vd)[32], const uint4 (&pa)[4],
                                              const uint4 (&pg)[4], int row, int col) {
  __nv_bfloat16* dpre = q.out + (int64_t)row * q.ldout;
#pragma unroll
  for (int g8 = 0; g8 < 4; ++g8) {
    float d[8], a[8], g[8], da[8], dg[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = __uint_as_float(vd[g8 * 8 + i]);
    unpack8(pack8(d), d);
    unpack8(pa[g8], a);
    unpack8(pg[g8], g);
#pragma unroll
    for (int i = 0; i < 8; ++i) glu_df<A0, A1>(d[i], a[i], g[i], da[i], dg[i], q.a0, q.a1);
    *reinterpret_cast<uint4*>(dpre + col + g8 * 8) = pack8(da);
    *reinterpret_cast<uint4*>(dpre + q.h + col + g8 * 8) = pack8(dg);
  }
}
__device__ __forceinline__ void glu_load(const Glu& q, int row, int col, bool ok, uint4 (&pa)[4], uint4 (&pg)[4]) {
  if (!ok) return;
  const uint4* a = reinterpret_cast<const uint4*>(q.pin + (int64_t)row * q.ldpin + col);
  const uint4* g = reinterpret_cast<const uint4*>(q.pin + (int64_t)row * q.ldpin + q.h + col);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    pa[i] = __ldg(a + i);
    pg[i] = __ldg(g + i);
  }
}

// One tile of the gated epilogues for a fixed activation pair (out of line: keeps the
// register allocation of the main epilogue loop unaffected).
template <int A0, int A1>
__device__ __noinline__ void glu_tile(const Glu q, int glu, uint32_t tbase, int row, bool row_ok, int tn) {
  if (glu == 1) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t va[32], vg[32];
      tmem_ld32(tbase + c * 32, va);
      tmem_ld32(tbase + 128 + c * 32, vg);
      tmem_ld_wait_regs(va);
      reg_fence(vg);
      const int col = tn * 128 + c * 32;
      if (row_ok && col < q.h) glu_fwd_chunk<A0, A1>(q, va, vg, row, col);
    }
  } else {
    // pre for chunk c + 1 is in flight while chunk c is computed
    uint4 ca[4], cg[4], na[4], ng[4];
    const int n0 = tn * 256;
    glu_load(q, row, n0, row_ok && n0 < q.n, ca, cg);
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
      const int col = n0 + c * 32;
      glu_load(q, row, col + 32, c + 1 < 8 && row_ok && col + 32 < q.n, na, ng);
      uint32_t v[32];
      tmem_ld32(tbase + c * 32, v);
      tmem_ld_wait_regs(v);
      if (row_ok && col < q.n) glu_bwd_chunk<A0, A1>(q, v, ca, cg, row, col);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ca[i] = na[i];
        cg[i] = ng[i];
      }
    }
  }
}

// ---- coalesced epilogue I/O through a per-warp shared-memory stage -------------------------
// The accumulator layout puts one output row in each lane, so direct stores touch 32 rows per
// instruction (32 L2 requests of 16 bytes: the epilogue of the wide GEMMs was L2-request bound,
// tensor pipe ~55% busy).  Instead each lane writes its row piece to the stage and the warp
// moves the 32 rows with lanes along rows: 4 (128-byte rows) or 8 (64-byte rows) requests per
// instruction.  A staged row is RB = 64 or 128 bytes; with RB = 128, bytes [0, 64) of row r
// live at g0 + r * ld and bytes [64, 128) at g1 + r * ld (g1 = g0 + 64: one contiguous piece).
constexpr int kStagePitch = 144;  // 16-byte pad: the lanes' own-row accesses are conflict-free

template <int RB>
__device__ __forceinline__ const uint8_t* stage_src(const uint8_t* g0, const uint8_t* g1, int c) {
  return RB == 128 && c >= 4 ? g1 + (c - 4) * 16 : g0 + c * 16;
}
// global -> registers (lanes along rows); rows >= nrows are skipped
template <int RB>
__device__ __forceinline__ void stage_gload(uint4 (&v)[RB / 16], int lane, const void* g0, const void* g1, int64_t ld,
                                            int nrows) {
  constexpr int LPR = RB / 16;  // lanes per row
#pragma unroll
  for (int i = 0; i < RB / 16; ++i) {
    const int r = i * (32 / LPR) + lane / LPR, c = lane % LPR;
    if (r < nrows)
      v[i] = __ldg(reinterpret_cast<const uint4*>(
          stage_src<RB>(reinterpret_cast<const uint8_t*>(g0), reinterpret_cast<const uint8_t*>(g1), c) + r * ld));
  }
}
// registers (from stage_gload) -> stage
template <int RB>
__device__ __forceinline__ void stage_put(uint8_t* st, const uint4 (&v)[RB / 16], int lane) {
  constexpr int LPR = RB / 16;
#pragma unroll
  for (int i = 0; i < RB / 16; ++i) {
    const int r = i * (32 / LPR) + lane / LPR, c = lane % LPR;
    *reinterpret_cast<uint4*>(st + r * kStagePitch + c * 16) = v[i];
  }
}
// stage -> global (lanes along rows); rows >= nrows are skipped
template <int RB>
__device__ __forceinline__ void stage_gstore(const uint8_t* st, int lane, void* g0, void* g1, int64_t ld, int nrows) {
  constexpr int LPR = RB / 16;
#pragma unroll
  for (int i = 0; i < RB / 16; ++i) {
    const int r = i * (32 / LPR) + lane / LPR, c = lane % LPR;
    const uint4 v = *reinterpret_cast<const uint4*>(st + r * kStagePitch + c * 16);
    if (r < nrows)
      *reinterpret_cast<uint4*>(
          const_cast<uint8_t*>(stage_src<RB>(reinterpret_cast<const uint8_t*>(g0), reinterpret_cast<const uint8_t*>(g1), c)) +
          r * ld) = v;
  }
}
__device__ __forceinline__ uint4 stage_own(const uint8_t* st, int lane, int j) {
  return *reinterpret_cast<const uint4*>(st + lane * kStagePitch + j * 16);
}
__device__ __forceinline__ void stage_set_own(uint8_t* st, int lane, int j, uint4 v) {
  *reinterpret_cast<uint4*>(st + lane * kStagePitch + j * 16) = v;
}

// Backward gated epilogue of one tile through the stage: per 32-column chunk of dhidden the
// warp loads the chunk's pre rows (a | g, 64 + 64 bytes) coalesced (the next chunk's loads in
// flight during this one), and stores dpre (da | dg) coalesced.  row0 = the warp's first row.
template <int A0, int A1>
__device__ __noinline__ void glu_bwd_tile_staged(const Glu q, uint32_t tbase, int row0, int nrows, int tn,
                                                 uint8_t* st, int lane) {
  const int n0 = tn * 256;
  const int64_t ldi = q.ldpin * 2, ldo = q.ldout * 2;
  const __nv_bfloat16* pin = q.pin + (int64_t)row0 * q.ldpin;
  __nv_bfloat16* pout = q.out + (int64_t)row0 * q.ldout;
  uint4 nxt[8];
  stage_gload<128>(nxt, lane, pin + n0, pin + q.h + n0, ldi, nrows);
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    const int col = n0 + c * 32;
    if (col >= q.n) break;  // warp-uniform (q.n % 32 == 0 on this path)
    stage_put<128>(st, nxt, lane);
    if (c + 1 < 8 && col + 32 < q.n) stage_gload<128>(nxt, lane, pin + col + 32, pin + q.h + col + 32, ldi, nrows);
    uint32_t v[32];
    tmem_ld32(tbase + c * 32, v);
    __syncwarp();
    uint4 pa[4], pg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pa[j] = stage_own(st, lane, j);
      pg[j] = stage_own(st, lane, 4 + j);
    }
    tmem_ld_wait_regs(v);
#pragma unroll
    for (int g8 = 0; g8 < 4; ++g8) {
      float d[8], a[8], g[8], da[8], dg[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = __uint_as_float(v[g8 * 8 + i]);
      unpack8(pack8(d), d);
      unpack8(pa[g8], a);
      unpack8(pg[g8], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) glu_df<A0, A1>(d[i], a[i], g[i], da[i], dg[i], q.a0, q.a1);
      stage_set_own(st, lane, g8, pack8(da));
      stage_set_own(st, lane, 4 + g8, pack8(dg));
    }
    __syncwarp();
    stage_gstore<128>(st, lane, pout + col, pout + q.h + col, ldo, nrows);
    __syncwarp();
  }
}

// RoPE rotation of one 32-column chunk held in registers (columns [0, rope_cols) only)
__device__ __forceinline__ void epi_rope(const Epi& e, uint32_t (&v)[32], int row, int col0) {
  if (!(e.rope_cos && col0 < e.rope_cols)) return;
  const int half = e.rope_hd >> 1;
  const int p0 = (col0 % e.rope_hd) >> 1;
  const int64_t tb = (int64_t)(row % e.rope_T) * half + p0;
  const float4* cs4 = reinterpret_cast<const float4*>(e.rope_cos + tb);
  const float4* sn4 = reinterpret_cast<const float4*>(e.rope_sin + tb);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 cq = cs4[j], sq = sn4[j];
    const float cc[4] = {cq.x, cq.y, cq.z, cq.w}, ss[4] = {sq.x, sq.y, sq.z, sq.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = (j * 4 + i) * 2;
      const float ev = __uint_as_float(v[k]), od = __uint_as_float(v[k + 1]);
      v[k] = __float_as_uint(ev * cc[i] - od * ss[i]);
      v[k + 1] = __float_as_uint(ev * ss[i] + od * cc[i]);
    }
  }
}

// Whether a GEMM's output takes the staged epilogue: bf16 output without addend (alpha and
// RoPE allowed), whole 32-column chunks, 16-byte aligned rows.  f32 outputs keep the per-lane
// epilogue: staging them measured ~10% slower on the O projection (each lane's eight 16-byte
// residual loads already hit one L1 line; the stage round trips lengthen the chunk chain).
__host__ __device__ __forceinline__ bool staged_ok(const Epi& e) {
  return e.N % 32 == 0 && (e.ldd & 7) == 0 && (reinterpret_cast<uintptr_t>(e.D) & 15) == 0 && !e.d_f32 &&
         !e.accumulate && !e.R;
}

// One 128-row x BN tile (bf16 output) of this warp's 32 rows through the stage.
template <int BN>
__device__ __noinline__ void epi_tile_staged(const Epi e, uint32_t tbase, int row0, int nrows, int tn, uint8_t* st,
                                             int lane) {
  const int row = row0 + lane;
  const int c0 = tn * BN;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    const int col0 = c0 + c * 32;
    if (col0 >= e.N) break;
    uint32_t v[32];
    tmem_ld32(tbase + c * 32, v);
    tmem_ld_wait_regs(v);
    epi_rope(e, v, row, col0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = __uint_as_float(v[j * 8 + i]) * e.alpha;
      stage_set_own(st, lane, j, pack8(o));
    }
    __syncwarp();
    __nv_bfloat16* g = reinterpret_cast<__nv_bfloat16*>(e.D) + (int64_t)row0 * e.ldd + col0;
    stage_gstore<64>(st, lane, g, g, e.ldd * 2, nrows);
    __syncwarp();
  }
}

// CTA-pair engine (cta_group::2): a cluster of two CTAs computes one 256 x 256 tile with a
// single tcgen05.mma stream issued by the leader.  Each CTA stages its own 128 rows of A and
// its own 128 columns of B (the hardware feeds each SM's tensor core the other half of B from
// the peer), so per SM the shared-memory operand traffic per FLOP is a third lower than the
// 1-CTA 128 x 256 tile and the two SMs share one MMA issue stream.  Each CTA's TMEM holds the
// 128 x 256 accumulator of its rows (double-buffered: 512 columns).
struct Cfg2 {
  static constexpr int kStages = 6;
  static constexpr int kABytes = BM * BK * 2;  // 16 KB: this CTA's 128 rows of A
  static constexpr int kBBytes = 128 * BK * 2; // 16 KB: this CTA's 128 columns of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiBytes = 4 * 32 * 144;  // per epilogue warp: 32 staged rows (see stage_*)
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + 1024 + 256;
};

// GLU: instantiation with the gated-activation epilogues (kept out of the plain kernel so its
// register allocation is not inflated by them)
template <bool GLU>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Args args) {
  using C = Cfg2;
  constexpr int BN = 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const bool leader = rank == 0;
  __shared__ int s_goff[kMaxGroups + 1];
  const int gm = args.grp_mode;
  if (gm) {
    for (int i = threadIdx.x; i <= args.G; i += blockDim.x) s_goff[i] = args.grp_off[i];
    __syncthreads();
  }
  // 256-row tile pairs (grouped over M: the padded row count comes from the device offsets)
  const int tiles_mg = gm == 1 ? s_goff[args.G] / (2 * BM) : (args.tiles_m + 1) / 2;
  const int S = args.splits;
  const int per_group = tiles_mg * args.tiles_n;
  const int num_units = gm == 2 ? args.G * per_group : per_group * S;
  const int unit0 = (int)(blockIdx.x >> 1), unit_stride = (int)(gridDim.x >> 1);
  const int nk_all = (args.K + BK - 1) / BK;
  // tile (tm, tn) of unit u and its group g (0 when not grouped)
  auto coords = [&](int u, int& tm, int& tn, int& g) {
    int tg;
    g = 0;
    if (gm == 2) {
      g = u / per_group;
      tile_coords(u - g * per_group, tiles_mg, args.tiles_n, tg, tn);
    } else {
      tile_coords(u / S, tiles_mg, args.tiles_n, tg, tn);
    }
    tm = tg * 2 + rank;
    if (gm == 1) {  // the group whose rows hold this 256-row tile
      const int r = tg * 2 * BM;
      while (g + 1 < args.G && s_goff[g + 1] <= r) ++g;
    }
  };
  // k-block range of unit u (its split-K slice, or its group's K rows)
  auto krange = [&](int u, int& kb0, int& kb1) {
    if (gm == 2) {
      const int g = u / per_group;
      kb0 = s_goff[g] / BK;
      kb1 = s_goff[g + 1] / BK;
      return;
    }
    const int sl = u % S;
    kb0 = (int)((int64_t)sl * nk_all / S);
    kb1 = (int)((int64_t)(sl + 1) * nk_all / S);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);   // leader: its expect_tx arrive; both CTAs' loads complete_tx here
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast to both CTAs)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // leader's copy: 4 epilogue warps of each CTA
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; completions land on the leader's barrier) ----
    int stage = 0;
    uint32_t phase = 0;
    for (int u = unit0; u < num_units; u += unit_stride) {
      int tm, tn, g;
      coords(u, tm, tn, g);
      const int m0 = tm * BM;
      // B columns this CTA stages: its half of the 256-column tile, or (gated forward) the
      // tile's 128 columns of the a half (rank 0) / of the g half (rank 1)
      int nb = args.e.glu == 1 ? rank * args.e.glu_h + tn * 128 : tn * BN + rank * 128;
      // grouped over M: group g's B block (stacked along K for MN-major B, along N otherwise)
      const int bk_off = (gm == 1 && args.b_mn) ? (int)(g * args.b_grp_stride) : 0;
      if (gm == 1 && !args.b_mn) nb += (int)(g * args.b_grp_stride);
      int kb0, kb1;
      krange(u, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* a_dst = sA + stage * C::kABytes;
        uint8_t* b_dst = sB + stage * C::kBBytes;
        const int k0 = kb * BK;
        if (elect_one()) {
          const uint32_t fb = leader_addr(&full[stage]);
          if (leader) mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
          if (!args.a_mn) {
            tma_load_2d_pair(a_dst, &tmA, fb, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(a_dst + j * 8192, &tmA, fb, m0 + 64 * j, k0);
          }
          if (!args.b_mn) {
            tma_load_2d_pair(b_dst, &tmB, fb, k0, nb);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma_load_2d_pair(b_dst + j * 8192, &tmB, fb, nb + 64 * j, k0 + bk_off);
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (leader) {
      const uint32_t idesc = idesc_bf16_f32(2 * BM, BN, args.a_mn, args.b_mn);
      const uint64_t a0 = args.a_mn ? sw128_desc(smem_u32(sA), 8192, 1024) : sw128_desc(smem_u32(sA), 16, 1024);
      const uint64_t b0 = args.b_mn ? sw128_desc(smem_u32(sB), 8192, 1024) : sw128_desc(smem_u32(sB), 16, 1024);
      const uint64_t a_step = args.a_mn ? 128 : 2, b_step = args.b_mn ? 128 : 2;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = unit0; u < num_units; u += unit_stride) {
        int kb0, kb1;
        krange(u, kb0, kb1);
        if (kb1 <= kb0) continue;  // an empty group (grouped over K): no tile
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a0 + (uint64_t)(stage * (C::kABytes >> 4));
          const uint64_t bd = b0 + (uint64_t)(stage * (C::kBBytes >> 4));
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_f16_ss_pair(d_tmem, ad + kk * a_step, bd + kk * b_step, idesc, (kb > kb0 || kk) ? 1u : 0u);
            umma_commit_pair_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair_mc(&tfull[acc], 0x3);
        __syncwarp();
        ++it;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs: each drains its own 128 rows) ----------------
    const int q = warp & 3;
    const Epi& e0 = args.e;
    const uint32_t tempty_leader0 = leader_addr(&tempty[0]);
    uint8_t* stg = smem + C::kStages * C::kStageBytes + 256 + q * 32 * kStagePitch;  // this warp's stage
    const bool staged = S == 1 && staged_ok(e0) && (g_epi_staged & kStagedBf16);
    // gated backward through the stage: pre / dpre rows 16-byte aligned, whole 32-column chunks
    const bool glu_staged = GLU && e0.glu == 2 && e0.N % 32 == 0 && e0.glu_h % 8 == 0 && (e0.ld_glu_pre & 7) == 0 &&
                            (e0.ld_glu_out & 7) == 0 && (reinterpret_cast<uintptr_t>(e0.glu_pre) & 15) == 0 &&
                            (reinterpret_cast<uintptr_t>(e0.glu_out) & 15) == 0;
    int it = 0;
    const bool adam_pf = e0.ad_p && gm == 0;
    if (adam_pf && unit0 < num_units) {
      int tm, tn, g;
      coords(unit0, tm, tn, g);
      epi_adam_prefetch(e0, tm * BM + q * 32 + lane, tn * BN, BN);
    }
    for (int u = unit0; u < num_units; u += unit_stride) {
      int tm, tn, g;
      coords(u, tm, tn, g);
      if (gm == 2) {
        int kb0, kb1;
        krange(u, kb0, kb1);
        if (kb1 <= kb0) continue;  // an empty group: its D rows are left untouched
      }
      const int acc = it & 1;
      ++it;
      mbar_wait(&tfull[acc], ((it - 1) >> 1) & 1);
      tc_fence_after();
      if (adam_pf && u + unit_stride < num_units) {  // the next tile's optimizer state into L2
        int tm2, tn2, g2;
        coords(u + unit_stride, tm2, tn2, g2);
        epi_adam_prefetch(e0, tm2 * BM + q * 32 + lane, tn2 * BN, BN);
      }
      Epi eg = e0;
      if (gm == 2)  // group g's rows of the stacked output
        eg.D = reinterpret_cast<char*>(eg.D) + (int64_t)g * eg.M * eg.ldd * (eg.d_f32 ? 4 : 2);
      const Epi& e = eg;
      const int row0 = tm * BM + q * 32;
      const int row = row0 + lane;
      const bool row_ok = row < e.M;
      const int nrows = max(0, min(32, e.M - row0));
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (GLU) {
        const Glu gq{reinterpret_cast<__nv_bfloat16*>(e.D), e.ldd, reinterpret_cast<__nv_bfloat16*>(e.glu_out),
                     e.ld_glu_out, reinterpret_cast<const __nv_bfloat16*>(e.glu_pre), e.ld_glu_pre, e.glu_h, e.N,
                     e.glu_a0, e.glu_a1};
        if (glu_staged && (g_epi_staged & kStagedGlu)) {
          if (e.glu_a0 == ACT_LINEAR && e.glu_a1 == ACT_SILU)  // SwiGLU
            glu_bwd_tile_staged<ACT_LINEAR, ACT_SILU>(gq, tbase, row0, nrows, tn, stg, lane);
          else
            glu_bwd_tile_staged<-1, -1>(gq, tbase, row0, nrows, tn, stg, lane);
        } else if (e.glu_a0 == ACT_LINEAR && e.glu_a1 == ACT_SILU) {  // SwiGLU
          glu_tile<ACT_LINEAR, ACT_SILU>(gq, e.glu, tbase, row, row_ok, tn);
        } else {
          glu_tile<-1, -1>(gq, e.glu, tbase, row, row_ok, tn);
        }
      } else if (staged) {
        epi_tile_staged<BN>(e, tbase, row0, nrows, tn, stg, lane);
      } else if (S > 1) {
        // split-K slice: raw f32 partial to ws[slice] (the reduce kernel applies the epilogue)
        float* part = args.ws + (int64_t)(u % S) * e.M * e.N + (int64_t)row * e.N;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + c * 32, v);
          tmem_ld_wait();
          const int col0 = tn * BN + c * 32;
          if (!row_ok || col0 >= e.N) continue;
          if (col0 + 32 <= e.N) {
            float4* dst = reinterpret_cast<float4*>(part + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                   __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          } else {
            const int lim = e.N - col0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < lim) part[col0 + j] = __uint_as_float(v[j]);
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + c * 32, v);
          tmem_ld_wait();
          const int col0 = tn * BN + c * 32;
          if (!row_ok || col0 >= e.N) continue;
          epi_chunk(e, v, row, col0);
        }
      }
      tc_fence_before();
      __syncwarp();
      // the accumulator buffer is free once this warp's tcgen05.ld completed (fence above);
      // its global stores need no ordering with the next tile's MMAs
      if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader0 + acc * 8);
    }
  }
  tc_fence_before();
  cluster_sync();  // neither CTA leaves while the pair's MMAs / multicasts may still target it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

// Split-K reduction: D = alpha * sum_s ws[s] (+ D) (+ R), slices summed in order s = 0..S-1
// (deterministic), 4 columns per thread.
__global__ void __launch_bounds__(256) splitk_reduce_k(const float* __restrict__ ws, int S, const Epi e) {
  const int64_t q = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int nq = (e.N + 3) >> 2;
  const int64_t row = q / nq;
  const int col = (int)(q - row * nq) * 4;
  if (row >= e.M) return;
  const int64_t mn = (int64_t)e.M * e.N, base = row * e.N + col;
  if (col + 4 <= e.N && (e.N & 3) == 0) {
    float4 acc = *reinterpret_cast<const float4*>(ws + base);
    for (int sl = 1; sl < S; ++sl) {
      const float4 t = *reinterpret_cast<const float4*>(ws + sl * mn + base);
      acc.x += t.x;
      acc.y += t.y;
      acc.z += t.z;
      acc.w += t.w;
    }
    const float v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) epi_store1(e, (int)row, col + j, v[j]);
  } else {
    for (int j = 0; j < 4 && col + j < e.N; ++j) {
      float v = 0.f;
      for (int sl = 0; sl < S; ++sl) v += ws[sl * mn + base + j];
      epi_store1(e, (int)row, col + j, v);
    }
  }
}

// Caller-provided split-K workspace (cb_gemm_set_workspace; PyTorch owns the buffer).
static float* g_ws = nullptr;
static int64_t g_ws_bytes = 0;

// Number of split-K slices for a CTA-pair GEMM: more slices only when the tile count leaves
// the last wave of the 74 pairs mostly empty and K is long enough to split, trading the
// saved MMA wave time against the f32 partial round trip through HBM.
static int choose_splits(const Args& a) {
  if (!g_ws || a.e.glu || a.e.rope_cos) return 1;
  const int P = kNumSMs / 2;
  const int units = ((a.tiles_m + 1) / 2) * a.tiles_n;
  const int nk = (a.K + BK - 1) / BK;
  if (units >= 4 * P || nk < 32) return 1;
  const double kblock_s = 0.4e-6;  // one 256x256x64 k-block on a pair, ~1.5 GHz
  const double hbm = 5.5e12;       // B/s for the partial write + reduce read
  double best_t = std::ceil((double)units / P) * nk * kblock_s;
  int best = 1;
  for (int S = 2; S <= 8; ++S) {
    if (nk / S < 16) break;
    const double bytes = 4.0 * S * (double)a.M * a.N;
    if (bytes > (double)g_ws_bytes) break;
    const double t = std::ceil((double)units * S / P) * ((double)nk / S) * kblock_s + 2.0 * bytes / hbm;
    if (t < 0.97 * best_t) {
      best_t = t;
      best = S;
    }
  }
  return best;
}

static int g_gemm_mc = 3;  // 3: CTA-pair MMA, 2: B-multicast cluster pairs, 1: single CTA

int launch_pair(const Args& a, const void* A, int64_t lda, const void* B, int64_t ldb, cudaStream_t st) {
  using C = Cfg2;
  CUtensorMap ta, tb;
  int s;
  // grouped over M: B holds every group's block, stacked along K (MN-major) or N (K-major)
  const int64_t bK = a.grp_mode == 1 && a.b_mn ? (int64_t)a.G * a.K : a.K;
  const int64_t bN = a.grp_mode == 1 && !a.b_mn ? (int64_t)a.G * a.N : a.N;
  if (!a.a_mn)
    s = make_tmap_2d_bf16(&ta, A, a.M, a.K, lda, BM, BK);
  else
    s = make_tmap_2d_bf16(&ta, A, a.K, a.M, lda, BK, 64);
  if (s) return s;
  if (!a.b_mn)
    s = make_tmap_2d_bf16(&tb, B, bN, a.K, ldb, 128, BK);
  else
    s = make_tmap_2d_bf16(&tb, B, bK, a.N, ldb, BK, 64);
  if (s) return s;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    cudaFuncSetAttribute(gemm_tc2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr_set = true;
  }
  Args args = a;
  args.splits = a.grp_mode ? 1 : choose_splits(a);
  args.ws = args.splits > 1 ? g_ws : nullptr;
  const int pairs = ((a.tiles_m + 1) / 2) * a.tiles_n * args.splits * (a.grp_mode == 2 ? a.G : 1);
  const int grid = 2 * std::min(pairs, kNumSMs / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = a.e.glu ? cudaLaunchKernelEx(&cfg, gemm_tc2<true>, ta, tb, args)
                          : cudaLaunchKernelEx(&cfg, gemm_tc2<false>, ta, tb, args);
  if (e != cudaSuccess) return fail(CB_ERR_CUDA, "gemm_tc2 cluster launch: %s", cudaGetErrorString(e));
  if (int r = check_launch("gemm_tc_pair")) return r;
  if (args.splits == 1) return CB_OK;
  const int64_t quads = (int64_t)a.M * ((a.N + 3) / 4);
  splitk_reduce_k<<<(unsigned)((quads + 255) / 256), 256, 0, st>>>(g_ws, args.splits, a.e);
  return check_launch("gemm_splitk_reduce");
}

template <int BN>
int launch(const Args& a, const void* A, int64_t lda, const void* B, int64_t ldb, cudaStream_t st) {
  using C = Cfg<BN>;
  if (BN == 256 && g_gemm_mc == 3 && a.tiles_m >= 2) return launch_pair(a, A, lda, B, ldb, st);
  const int mc = (g_gemm_mc >= 2 && a.tiles_m >= 2) ? 2 : 1;
  CUtensorMap ta, tb;
  int s;
  // A: op(A) is MxK.  K-major -> stored [M][K]; MN-major -> stored [K][M].
  if (!a.a_mn)
    s = make_tmap_2d_bf16(&ta, A, a.M, a.K, lda, BM, BK);
  else
    s = make_tmap_2d_bf16(&ta, A, a.K, a.M, lda, BK, 64);
  if (s) return s;
  // B: op(B) is KxN.  K-major -> stored [N][K] (box rows = the BN/mc rows one CTA loads);
  // MN-major -> stored [K][N].
  if (!a.b_mn)
    s = make_tmap_2d_bf16(&tb, B, a.N, a.K, ldb, BN / mc, BK);
  else
    s = make_tmap_2d_bf16(&tb, B, a.K, a.N, ldb, BK, 64);
  if (s) return s;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc<BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    cudaFuncSetAttribute(gemm_tc<BN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr_set = true;
  }
  if (mc == 1) {
    const int grid = std::min(a.tiles_m * a.tiles_n, kNumSMs);
    gemm_tc<BN, 1><<<grid, kThreads, C::kSmem, st>>>(ta, tb, a);
    return check_launch("gemm_tc");
  }
  Args args = a;
  args.splits = a.grp_mode ? 1 : choose_splits(a);
  args.ws = args.splits > 1 ? g_ws : nullptr;
  const int pairs = ((a.tiles_m + 1) / 2) * a.tiles_n * args.splits * (a.grp_mode == 2 ? a.G : 1);
  const int grid = 2 * std::min(pairs, kNumSMs / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_tc<BN, 2>, ta, tb, a);
  if (e != cudaSuccess) return fail(CB_ERR_CUDA, "gemm_tc cluster launch: %s", cudaGetErrorString(e));
  return check_launch("gemm_tc_mc");
}
}  // namespace tc

// ======================================================================================
// SIMT engine (f32 parity mode; unaligned bf16 shapes)
// ======================================================================================
namespace simt {
constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt(int M, int N, int K, const T* __restrict__ A, int64_t sam, int64_t sak,
                                                 const T* __restrict__ B, int64_t sbk, int64_t sbn, Epi e) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int i = 0; i < (TK * TM) / 256; ++i) {
      const int idx = threadIdx.x + i * 256;
      // walk the contiguous dimension with consecutive threads where possible
      int kk, mm;
      if (sak == 1) {
        kk = idx % TK;
        mm = idx / TK;
      } else {
        mm = idx % TM;
        kk = idx / TM;
      }
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? to_f32(A[(int64_t)gm * sam + (int64_t)gk * sak]) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < (TK * TN) / 256; ++i) {
      const int idx = threadIdx.x + i * 256;
      int kk, nn;
      if (sbn == 1) {
        nn = idx % TN;
        kk = idx / TN;
      } else {
        kk = idx % TK;
        nn = idx / TK;
      }
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? to_f32(B[(int64_t)gk * sbk + (int64_t)gn * sbn]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = m0 + ty + 16 * i, c = n0 + tx + 16 * j;
      if (r < M && c < N) epi_store1(e, r, c, acc[i][j]);
    }
}
}  // namespace simt

static int g_gemm_path = 0;  // 0 auto, 1 force SIMT, 2 force tcgen05
static thread_local int g_last_gemm_tc = 0;  // did the last gemm_impl call run on tcgen05?

}  // namespace cb

using namespace cb;

// Gated-activation FFN GEMMs on the CTA-pair engine (bf16).  Both return
// CB_ERR_UNSUPPORTED — without launching anything — when the fused form does not apply
// (shape / alignment / engine disabled); the caller then runs cb_gemm + cb_act_fwd/bwd.
static bool glu_ok(int M, int H, int K, const void* A, int64_t lda, const void* B, int64_t ldb, const void* p0,
                   int64_t ld0, const void* p1, int64_t ld1) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return tc::g_gemm_mc == 3 && g_gemm_path != 1 && M >= 2 * tc::BM && K > 0 && H % 32 == 0 && al(A) && al(B) &&
         al(p0) && al(p1) && ((lda | ldb | ld0 | ld1) & 7) == 0;
}

extern "C" int cb_gemm_gated_fwd(int M, int H, int K, const void* A, int64_t lda, int trans_a, const void* B,
                                 int64_t ldb, int trans_b, void* pre, int64_t ldpre, void* hidden, int64_t ldh,
                                 int act0, int act1, void* stream) {
  if (M < 0 || H < 0 || K < 0) return fail(CB_ERR_SHAPE, "gemm_gated_fwd: negative extent");
  if (H % 128 != 0 || !glu_ok(M, H, K, A, lda, B, ldb, pre, ldpre, hidden, ldh))
    return fail(CB_ERR_UNSUPPORTED, "gemm_gated_fwd: fused epilogue not applicable (M=%d H=%d K=%d)", M, H, K);
  tc::Args a;
  a.M = M;
  a.N = 2 * H;
  a.K = K;
  a.a_mn = trans_a ? 1 : 0;
  a.b_mn = trans_b ? 0 : 1;
  a.tiles_m = (M + tc::BM - 1) / tc::BM;
  a.tiles_n = H / 128;
  a.e = Epi{pre, ldpre, 0, nullptr, 0, 0, 1.f, 0, M, 2 * H};
  a.e.glu = 1;
  a.e.glu_h = H;
  a.e.glu_a0 = act0;
  a.e.glu_a1 = act1;
  a.e.glu_out = hidden;
  a.e.ld_glu_out = ldh;
  return tc::launch_pair(a, A, lda, B, ldb, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int cb_gemm_gated_bwd(int M, int H, int K, const void* A, int64_t lda, int trans_a, const void* B,
                                 int64_t ldb, int trans_b, const void* pre, int64_t ldpre, void* dpre, int64_t lddpre,
                                 int act0, int act1, void* stream) {
  if (M < 0 || H < 0 || K < 0) return fail(CB_ERR_SHAPE, "gemm_gated_bwd: negative extent");
  if (!glu_ok(M, H, K, A, lda, B, ldb, pre, ldpre, dpre, lddpre))
    return fail(CB_ERR_UNSUPPORTED, "gemm_gated_bwd: fused epilogue not applicable (M=%d H=%d K=%d)", M, H, K);
  tc::Args a;
  a.M = M;
  a.N = H;
  a.K = K;
  a.a_mn = trans_a ? 1 : 0;
  a.b_mn = trans_b ? 0 : 1;
  a.tiles_m = (M + tc::BM - 1) / tc::BM;
  a.tiles_n = (H + 255) / 256;
  a.e = Epi{dpre, lddpre, 0, nullptr, 0, 0, 1.f, 0, M, H};
  a.e.glu = 2;
  a.e.glu_h = H;
  a.e.glu_a0 = act0;
  a.e.glu_a1 = act1;
  a.e.glu_out = dpre;
  a.e.ld_glu_out = lddpre;
  a.e.glu_pre = pre;
  a.e.ld_glu_pre = ldpre;
  return tc::launch_pair(a, A, lda, B, ldb, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- grouped (MoE experts)
static int grouped_check(int groups, const int* grp_off, const char* who) {
  if (groups < 1 || groups > tc::kMaxGroups) return fail(CB_ERR_ARG, "%s: 1..%d groups", who, tc::kMaxGroups);
  if (!grp_off) return fail(CB_ERR_ARG, "%s: null group offsets", who);
  if (tc::g_gemm_mc != 3 || g_gemm_path == 1) return fail(CB_ERR_UNSUPPORTED, "%s: needs the CTA-pair engine", who);
  return CB_OK;
}
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int cb_gemm_grouped(int mode, int groups, const int* grp_off, int M, int N, int K, const void* A,
                               int64_t lda, int trans_a, const void* B, int64_t ldb, int trans_b, void* D, int64_t ldd,
                               int d_dtype, float alpha, int accumulate, void* stream) {
  if (int s = grouped_check(groups, grp_off, "gemm_grouped")) return s;
  if (mode != 1 && mode != 2) return fail(CB_ERR_ARG, "gemm_grouped: mode 1 (rows) or 2 (K)");
  if (M <= 0 || N <= 0 || K <= 0) return fail(CB_ERR_SHAPE, "gemm_grouped: empty extent");
  if ((mode == 1 && M % 256) || (mode == 2 && K % 256))
    return fail(CB_ERR_SHAPE, "gemm_grouped: the grouped extent must be a multiple of 256");
  if (mode == 2 && (!trans_a || trans_b)) return fail(CB_ERR_ARG, "gemm_grouped mode 2: A^T @ B (rows along K)");
  if (!aligned16(A) || !aligned16(B) || ((lda | ldb) & 7))
    return fail(CB_ERR_UNSUPPORTED, "gemm_grouped: 16-byte aligned operands");
  tc::Args a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.a_mn = trans_a ? 1 : 0;
  a.b_mn = trans_b ? 0 : 1;
  a.tiles_m = (M + tc::BM - 1) / tc::BM;
  a.tiles_n = (N + 255) / 256;
  a.e = Epi{D, ldd, d_dtype == CB_DT_F32, nullptr, 0, 0, alpha, accumulate, M, N};
  a.grp_off = grp_off;
  a.grp_mode = mode;
  a.G = groups;
  a.b_grp_stride = trans_b ? N : K;
  return tc::launch_pair(a, A, lda, B, ldb, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int cb_gemm_gated_fwd_grouped(int groups, const int* grp_off, int M, int H, int K, const void* A,
                                         int64_t lda, const void* B, int64_t ldb, void* pre, int64_t ldpre,
                                         void* hidden, int64_t ldh, int act0, int act1, void* stream) {
  if (int s = grouped_check(groups, grp_off, "gemm_gated_fwd_grouped")) return s;
  if (M % 256 || H % 128 || !glu_ok(M, H, K, A, lda, B, ldb, pre, ldpre, hidden, ldh))
    return fail(CB_ERR_UNSUPPORTED, "gemm_gated_fwd_grouped: not applicable (M=%d H=%d K=%d)", M, H, K);
  tc::Args a;
  a.M = M;
  a.N = 2 * H;
  a.K = K;
  a.a_mn = 0;
  a.b_mn = 1;
  a.tiles_m = M / tc::BM;
  a.tiles_n = H / 128;
  a.e = Epi{pre, ldpre, 0, nullptr, 0, 0, 1.f, 0, M, 2 * H};
  a.e.glu = 1;
  a.e.glu_h = H;
  a.e.glu_a0 = act0;
  a.e.glu_a1 = act1;
  a.e.glu_out = hidden;
  a.e.ld_glu_out = ldh;
  a.grp_off = grp_off;
  a.grp_mode = 1;
  a.G = groups;
  a.b_grp_stride = K;  // B = [W1|Wg] of every group stacked along K: [groups*K][2H]
  return tc::launch_pair(a, A, lda, B, ldb, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int cb_gemm_gated_bwd_grouped(int groups, const int* grp_off, int M, int H, int K, const void* A,
                                         int64_t lda, const void* B, int64_t ldb, const void* pre, int64_t ldpre,
                                         void* dpre, int64_t lddpre, int act0, int act1, void* stream) {
  if (int s = grouped_check(groups, grp_off, "gemm_gated_bwd_grouped")) return s;
  if (M % 256 || !glu_ok(M, H, K, A, lda, B, ldb, pre, ldpre, dpre, lddpre))
    return fail(CB_ERR_UNSUPPORTED, "gemm_gated_bwd_grouped: not applicable (M=%d H=%d K=%d)", M, H, K);
  tc::Args a;
  a.M = M;
  a.N = H;
  a.K = K;
  a.a_mn = 0;
  a.b_mn = 0;  // dhidden = dy @ W2^T: W2 of every group stacked [groups*H][K], K-major
  a.tiles_m = M / tc::BM;
  a.tiles_n = (H + 255) / 256;
  a.e = Epi{dpre, lddpre, 0, nullptr, 0, 0, 1.f, 0, M, H};
  a.e.glu = 2;
  a.e.glu_h = H;
  a.e.glu_a0 = act0;
  a.e.glu_a1 = act1;
  a.e.glu_out = dpre;
  a.e.ld_glu_out = lddpre;
  a.e.glu_pre = pre;
  a.e.ld_glu_pre = ldpre;
  a.grp_off = grp_off;
  a.grp_mode = 1;
  a.G = groups;
  a.b_grp_stride = H;
  return tc::launch_pair(a, A, lda, B, ldb, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int cb_gemm_set_workspace(void* ptr, int64_t bytes) {
  if (bytes < 0 || (bytes > 0 && !ptr) || (reinterpret_cast<uintptr_t>(ptr) & 15))
    return fail(CB_ERR_ARG, "gemm workspace: need a 16-byte aligned buffer");
  tc::g_ws = bytes > 0 ? reinterpret_cast<float*>(ptr) : nullptr;
  tc::g_ws_bytes = bytes;
  return CB_OK;
}

extern "C" int cb_gemm_set_staged_epilogue(int enable) {
  const int v = enable == 1 ? 3 : enable < 0 ? 0 : enable & 3;
  if (cudaMemcpyToSymbol(tc::g_epi_staged, &v, sizeof(v)) != cudaSuccess)
    return fail(CB_ERR_CUDA, "cb_gemm_set_staged_epilogue: cudaMemcpyToSymbol failed");
  return CB_OK;
}

extern "C" int cb_gemm_set_raster(int group_m) {
  if (group_m < 1 || group_m > 1024) return fail(CB_ERR_ARG, "gemm raster group must be 1..1024 tile rows");
  if (cudaMemcpyToSymbol(tc::g_group_m, &group_m, sizeof(group_m)) != cudaSuccess)
    return fail(CB_ERR_CUDA, "cb_gemm_set_raster: cudaMemcpyToSymbol failed");
  return CB_OK;
}

extern "C" int cb_gemm_set_multicast(int mode) {
  // 0: single-CTA tiles, 1: default (CTA pair), 2: B-multicast cluster pairs, 3: CTA pair
  if (mode < 0 || mode > 3) return fail(CB_ERR_ARG, "gemm cluster mode must be 0..3");
  tc::g_gemm_mc = mode == 0 ? 1 : mode == 1 ? 3 : mode;
  return CB_OK;
}

extern "C" int cb_gemm_set_path(int path) {
  if (path < 0 || path > 2) return fail(CB_ERR_ARG, "gemm path must be 0 (auto), 1 (simt) or 2 (tcgen05)");
  g_gemm_path = path;
  return CB_OK;
}

static int gemm_impl(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                     int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, const void* R, int64_t ldr,
                     int r_dtype, float alpha, int accumulate, cudaStream_t st, Epi e);

// See include/composer_b200.h for the contract.
extern "C" int cb_gemm(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                       int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, const void* R, int64_t ldr,
                       int r_dtype, float alpha, int accumulate, void* stream) {
  Epi e{D, ldd, d_dtype == CB_DT_F32, R, ldr, r_dtype == CB_DT_F32, alpha, accumulate, M, N};
  return gemm_impl(M, N, K, in_dtype, A, lda, trans_a, B, ldb, trans_b, D, ldd, d_dtype, R, ldr, r_dtype, alpha,
                   accumulate, reinterpret_cast<cudaStream_t>(stream), e);
}

// AdamW fused into a weight-gradient GEMM: the update of the parameters whose gradient is
// alpha * op(A) @ op(B) (their whole gradient this step); D frames the addresses (the
// gradient buffer's view, never read or written), param / exp_avg / exp_avg_sq (f32) and
// param_bf16 (optional) share D's layout.  Bit-identical to cb_gemm(accumulate into a zeroed
// D) followed by cb_adamw on D.
extern "C" int cb_gemm_adamw(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                             int64_t ldb, int trans_b, void* D, int64_t ldd, float alpha, float* param, float* exp_avg,
                             float* exp_avg_sq, void* param_bf16, float lr, float beta1, float beta2, float eps,
                             float weight_decay, int step, void* stream) {
  if (step < 1) return fail(CB_ERR_ARG, "gemm_adamw: step must be >= 1");
  if (!param || !exp_avg || !exp_avg_sq) return fail(CB_ERR_ARG, "gemm_adamw: null optimizer buffer");
  Epi e{D, ldd, 1, nullptr, 0, 0, alpha, 0, M, N};
  e.ad_p = param;
  e.ad_m = exp_avg;
  e.ad_v = exp_avg_sq;
  e.ad_bf = reinterpret_cast<__nv_bfloat16*>(param_bf16);
  e.ad_lr = lr;
  e.ad_b1 = beta1;
  e.ad_b2 = beta2;
  e.ad_eps = eps;
  e.ad_wd = weight_decay;
  e.ad_bc1 = (float)(1.0 - pow((double)beta1, step));  // as cb_adamw
  e.ad_bc2 = (float)(1.0 - pow((double)beta2, step));
  return gemm_impl(M, N, K, in_dtype, A, lda, trans_a, B, ldb, trans_b, D, ldd, CB_DT_F32, nullptr, 0, 0, alpha, 0,
                   reinterpret_cast<cudaStream_t>(stream), e);
}

// D = op(A) @ op(B) with RoPE applied to output columns [0, rope_cols) (the q|k part of a
// fused QKV projection) inside the tcgen05 epilogue; other engines rotate in a second pass.
extern "C" int cb_gemm_rope(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                            int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, int seq_len, int head_dim,
                            int rope_cols, const float* cos_t, const float* sin_t, void* stream) {
  if (head_dim <= 0 || head_dim % 2 || rope_cols % head_dim || rope_cols > N)
    return fail(CB_ERR_SHAPE, "gemm_rope: bad head_dim %d / rope_cols %d", head_dim, rope_cols);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Epi e{D, ldd, d_dtype == CB_DT_F32, nullptr, 0, 0, 1.f, 0, M, N};
  const bool fuse = in_dtype == CB_DT_BF16 && head_dim % 32 == 0 && seq_len > 0 &&
                    !(reinterpret_cast<uintptr_t>(cos_t) & 15) && !(reinterpret_cast<uintptr_t>(sin_t) & 15);
  if (fuse) {
    e.rope_cos = cos_t;
    e.rope_sin = sin_t;
    e.rope_T = seq_len;
    e.rope_hd = head_dim;
    e.rope_cols = rope_cols;
  }
  int s = gemm_impl(M, N, K, in_dtype, A, lda, trans_a, B, ldb, trans_b, D, ldd, d_dtype, nullptr, 0, 0, 1.f, 0, st, e);
  if (s) return s;
  if (fuse && g_last_gemm_tc) return CB_OK;
  // the SIMT engine ignores the rope fields: rotate in a separate pass
  return cb_rope(M, seq_len, rope_cols / head_dim, head_dim, D, ldd, d_dtype, cos_t, sin_t, 0, stream);
}

static int gemm_impl(int M, int N, int K, int in_dtype, const void* A, int64_t lda, int trans_a, const void* B,
                     int64_t ldb, int trans_b, void* D, int64_t ldd, int d_dtype, const void* R, int64_t ldr,
                     int r_dtype, float alpha, int accumulate, cudaStream_t st, Epi e) {
  g_last_gemm_tc = 0;
  if (M < 0 || N < 0 || K < 0) return fail(CB_ERR_SHAPE, "gemm: negative extent (%d,%d,%d)", M, N, K);
  if (!D) return fail(CB_ERR_ARG, "gemm: null output");
  if (M == 0 || N == 0) return CB_OK;
  if (in_dtype != CB_DT_F32 && in_dtype != CB_DT_BF16) return fail(CB_ERR_UNSUPPORTED, "gemm: input dtype %d", in_dtype);
  if (K == 0) {
    // alpha*0 (+D) (+R): route through the SIMT epilogue with an empty reduction
    dim3 grid((N + simt::TN - 1) / simt::TN, (M + simt::TM - 1) / simt::TM);
    simt::gemm_simt<float><<<grid, 256, 0, st>>>(M, N, 0, nullptr, 0, 0, nullptr, 0, 0, e);
    return check_launch("gemm_simt");
  }
  if (!A || !B) return fail(CB_ERR_ARG, "gemm: null operand");
  const int64_t sam = trans_a ? 1 : lda, sak = trans_a ? lda : 1;
  const int64_t sbk = trans_b ? 1 : ldb, sbn = trans_b ? ldb : 1;
  if (in_dtype == CB_DT_BF16) {
    const bool aligned = ((lda & 7) == 0) && ((ldb & 7) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    const double work = (double)M * N * K;
    bool use_tc = aligned && (g_gemm_path == 2 || (g_gemm_path == 0 && work >= (double)(1 << 22)));
    if (g_gemm_path == 2 && !aligned) return fail(CB_ERR_UNSUPPORTED, "gemm: tcgen05 path needs 16-byte aligned operands");
    if (use_tc) {
      tc::Args a;
      a.M = M;
      a.N = N;
      a.K = K;
      a.a_mn = trans_a ? 1 : 0;
      a.b_mn = trans_b ? 0 : 1;
      a.e = e;
      a.tiles_m = (M + tc::BM - 1) / tc::BM;
      g_last_gemm_tc = 1;
      if (N > 128) {
        a.tiles_n = (N + 255) / 256;
        return tc::launch<256>(a, A, lda, B, ldb, st);
      }
      a.tiles_n = (N + 127) / 128;
      return tc::launch<128>(a, A, lda, B, ldb, st);
    }
    dim3 grid((N + simt::TN - 1) / simt::TN, (M + simt::TM - 1) / simt::TM);
    simt::gemm_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(M, N, K, reinterpret_cast<const __nv_bfloat16*>(A), sam, sak,
                                                         reinterpret_cast<const __nv_bfloat16*>(B), sbk, sbn, e);
    return check_launch("gemm_simt_bf16");
  }
  dim3 grid((N + simt::TN - 1) / simt::TN, (M + simt::TM - 1) / simt::TM);
  simt::gemm_simt<float><<<grid, 256, 0, st>>>(M, N, K, reinterpret_cast<const float*>(A), sam, sak,
                                               reinterpret_cast<const float*>(B), sbk, sbn, e);
  return check_launch("gemm_simt_f32");
}
