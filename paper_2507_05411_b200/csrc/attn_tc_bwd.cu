// tcgen05 flash attention backward (bf16, head_dim 128), unmasked, GQA-aware.
//
// Deterministic two-kernel split (no atomics), both recomputing P = exp(S - LSE):
//   dkdv: one CTA per (128-key tile, kv head, batch); sweeps every 128-query tile u of
//         every query head in the kv group:
//           S^T_u  = K Q_u^T      (A = K  smem K-major, B = Q_u  smem K-major)  -> TMEM
//           dP^T_u = V dO_u^T     (A = V  smem K-major, B = dO_u smem K-major)  -> TMEM
//           P^T = exp2(S^T c - lse2), dS^T = P^T (dP^T - delta)   [CUDA cores, per key row]
//           dV += P^T dO_u        (A = P^T from TMEM, B = dO_u smem MN-major)
//           dK += dS^T Q_u        (A = dS^T from TMEM, B = Q_u  smem MN-major)
//         MMA issue order  S(u+1) | dV(u) | dK(u) dP(u+1): S(u+1) as soon as S^T(u) is in
//         registers, dV(u) as soon as P^T(u) is stored, half of dK(u) after the first half of
//         dS^T(u), so the exp and dS passes overlap the MMAs with single-buffered TMEM
//         (S^T | dP^T | dV | dK = 512 columns).
//   dq:   one CTA per (128-query tile, head, batch); sweeps every 128-key tile j:
//           S_j = Q K_j^T (double-buffered), dP_j = dO V_j^T, dS = P (dP - delta),
//           dQ += dS K_j (B = K_j MN-major); S_{j+1} is issued before dQ_j, half of dQ_j
//           after the first half of dS_j.  TMEM: S[2] | dP | dQ.
// Roles: warp 0 TMA, warp 1 MMA (single thread), warp 2 TMEM alloc, warps 4-11 compute
// (warps w and w+4 share TMEM lane quadrant w%4 and split each tile's columns in halves).
#include "attn.cuh"
#include "composer_b200.h"

namespace cb {
namespace tcb {

constexpr int HD = 128;
constexpr int BT = 128;  // tile rows (keys or queries)
constexpr int kThreads = 384;
constexpr int kBox = 128 * 64 * 2;  // one [128][64] bf16 TMA box (16 KB)
constexpr int kTile = 2 * kBox;     // one [128][128] tile (two 64-column atoms)
// dq: Q, dO, K ring [3], V ring [2] = 224 KB (+ alignment slack)
constexpr int kKSlots = 3, kVSlots = 2;
constexpr int kSmemDq = (2 + kKSlots + kVSlots) * kTile + 1024 + 256;
constexpr uint32_t kCols = 512;
constexpr float kLog2e = 1.4426950408889634f;

struct Params {
  int T, H, KVH, B;
  float scale;
  const float* lse;
  const float* delta;
  __nv_bfloat16* o0;  // dk (dkdv) or dq (dq)
  int64_t ld0;
  __nv_bfloat16* o1;  // dv (dkdv)
  int64_t ld1;
  const float* rope_cos;  // optional [T][HD/2]: un-rotate dK / dQ on store
  const float* rope_sin;
};

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// descriptor start-address offset (16-byte units) of the kk-th K=16 step of a K-major
// [128][128] tile (two 64-column swizzle atoms)
__device__ __forceinline__ uint64_t koff(int kk) { return (uint64_t)(((kk >> 2) * kBox + (kk & 3) * 32) >> 4); }

#ifdef CB_ATTN_TRACE
__device__ unsigned long long g_btrace[24][64];
#define BWD_TRACE(ev, j) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64 && (threadIdx.x & 31) == 0) g_btrace[ev][j] = clock64()
// per-CTA timeline: [kernel][cta] = {start ns, end ns, smid}
__device__ unsigned long long g_cta[2][8192][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_TRACE(kern, which)                                                                    \
  if (threadIdx.x == 0) {                                                                         \
    const int id_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);               \
    if (id_ < 8192) {                                                                             \
      g_cta[kern][id_][which] = gtimer();                                                         \
      if (which == 0) {                                                                           \
        unsigned s_;                                                                              \
        asm volatile("mov.u32 %0, %smid;" : "=r"(s_));                                            \
        g_cta[kern][id_][2] = s_;                                                                 \
      }                                                                                           \
    }                                                                                             \
  }
#else
#define CTA_TRACE(kern, which)
#define BWD_TRACE(ev, j)
#endif


// Store `nchunks` x 32 f32 TMEM columns of this thread's row as bf16 (times `mul`); with
// rc/rs (cos/sin of this row's position) first apply the inverse RoPE rotation — the
// backward of the rotation fused into the QKV projection.
__device__ __forceinline__ void store_row(uint32_t taddr, __nv_bfloat16* dst, float mul, bool ok, const float* rc,
                                          const float* rs, int nchunks) {
#pragma unroll 1
  for (int cc = 0; cc < nchunks; ++cc) {
    uint32_t o[32];
    tmem_ld32(taddr + cc * 32, o);
    tmem_ld_wait();
    if (ok && rc) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float c = rc[cc * 16 + i], s = rs[cc * 16 + i];
        const float e = __uint_as_float(o[2 * i]), d = __uint_as_float(o[2 * i + 1]);
        o[2 * i] = __float_as_uint(e * c + d * s);
        o[2 * i + 1] = __float_as_uint(d * c - e * s);
      }
    }
    if (ok) {
      uint4* d = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint4 pk;
        pk.x = pack2(__uint_as_float(o[w * 8 + 0]) * mul, __uint_as_float(o[w * 8 + 1]) * mul);
        pk.y = pack2(__uint_as_float(o[w * 8 + 2]) * mul, __uint_as_float(o[w * 8 + 3]) * mul);
        pk.z = pack2(__uint_as_float(o[w * 8 + 4]) * mul, __uint_as_float(o[w * 8 + 5]) * mul);
        pk.w = pack2(__uint_as_float(o[w * 8 + 6]) * mul, __uint_as_float(o[w * 8 + 7]) * mul);
        d[w] = pk;
      }
    }
  }
}

#ifndef CB_ATTN_EMU_BWD
#define CB_ATTN_EMU_BWD 2
#endif
constexpr int kEmuPairs = CB_ATTN_EMU_BWD;  // of every 8 exp2 pairs, this many on the FMA pipe

// 64 f32 TMEM columns of this thread's row: both loads in flight, one wait
__device__ __forceinline__ void ld64(uint32_t src, uint32_t (&v)[2][32]) {
  tmem_ld32(src, v[0]);
  tmem_ld32(src + 32, v[1]);
  tmem_ld_wait_regs(v[0]);
  reg_fence(v[1]);
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 col2(const uint32_t (&v)[2][32], int i) {  // columns 2i, 2i+1
  return make_float2(__uint_as_float(v[i >> 4][2 * (i & 15)]), __uint_as_float(v[i >> 4][2 * (i & 15) + 1]));
}
__device__ __forceinline__ float2 exp2_pair(float2 a, int i) {
  if ((i & 7) < kEmuPairs) return exp2_poly2(a);
  return make_float2(fast_exp2(a.x), fast_exp2(a.y));
}
// W f32 TMEM columns of this thread's row (W = 32 or 64), all loads in flight, one wait
template <int W>
__device__ __forceinline__ void ldW(uint32_t src, uint32_t (&v)[W / 32][32]) {
#pragma unroll
  for (int i = 0; i < W / 32; ++i) tmem_ld32(src + 32 * i, v[i]);
  tmem_ld_wait_regs(v[0]);
#pragma unroll
  for (int i = 1; i < W / 32; ++i) reg_fence(v[i]);
}
template <int NB>
__device__ __forceinline__ float2 colp(const uint32_t (&v)[NB][32], int i) {  // columns 2i, 2i+1
  return make_float2(__uint_as_float(v[i >> 4][2 * (i & 15)]), __uint_as_float(v[i >> 4][2 * (i & 15) + 1]));
}
// pack NP pairs to bf16 and store them as NP TMEM columns at dst (NP = 16 or 32)
template <int NP>
__device__ __forceinline__ void pack_storeN(uint32_t dst, const float2 (&v)[NP]) {
#pragma unroll
  for (int h = 0; h < NP / 16; ++h) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack2(v[16 * h + i].x, v[16 * h + i].y);
    tmem_st16(dst + 16 * h, pk);
  }
  tmem_st_wait();
}
// pack 32 pairs to bf16 and store them as 32 TMEM columns at dst
__device__ __forceinline__ void pack_store(uint32_t dst, const float2 (&v)[32]) {
  uint32_t pk[2][16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    pk[0][i] = pack2(v[i].x, v[i].y);
    pk[1][i] = pack2(v[16 + i].x, v[16 + i].y);
  }
  tmem_st16(dst, pk[0]);
  tmem_st16(dst + 16, pk[1]);
  tmem_st_wait();
}

// ====================================================================== dK / dV
// 128-query tiles.  TMEM: S^T | dP^T | dV | dK (128 columns each).  Compute warps w and w+4
// share TMEM lane quadrant w%4: half ch takes query columns [64 ch, 64 ch + 64).  A tile's
// S^T is read into registers at once (s_free), so S(u+1) is issued while tile u is still
// being computed; P^T and dS^T (bf16 pairs) are then written over the dP^T region the half
// has already read: P^T at columns [64 ch, 64 ch + 32), dS^T at [64 ch + 32, 64 ch + 64).
// MMA order per tile u:  [s_free(u)] S(u+1) | [p_ready(u)] dV(u) | [ds_part(u)] dK_a(u) |
// [pd_ready(u)] dK_b(u) dP(u+1): P^T is stored (and signalled) before dS^T is computed, so
// dV(u) overlaps the dS math, and dK(u) starts on the first half of each group's dS^T.
// smem: K, V, Q ring [3], dO ring [2], lse/delta ring [2] = 226 KB: this needs the dynamic
// shared-memory base to be 1024-aligned already (checked).
constexpr int kQSlots = 3, kGSlots = 2;
#ifndef CB_DKDV_GROUPS
#define CB_DKDV_GROUPS 2
#endif
constexpr int kDkdvGroups = CB_DKDV_GROUPS;  // 2: 8 compute warps, 4: 16 compute warps
constexpr int kSmemDkdv = (2 + kQSlots + kGSlots) * kTile + 2 * 1024 + 8 * 24;

// TMEM column of the k-th K=16 step of a packed bf16 A operand written by the two halves
__device__ __forceinline__ uint32_t packed_col(int k) { return (uint32_t)((k >> 2) * 64 + (k & 3) * 8); }
// Same with NQ column groups of W = 128 / NQ query columns: group g packs P^T into
// [g W, g W + W/2) and dS^T into [g W + W/2, (g + 1) W) of the dP^T region.
template <int NQ>
__device__ __forceinline__ uint32_t packed_colq(int k) {
  constexpr int W = 128 / NQ;
  return (uint32_t)((k * 16 / W) * W + ((k * 16) % W) / 2);
}

// NQ column groups -> 4 NQ compute warps (warps 4 .. 4 + 4 NQ), 128 + 128 NQ threads.
// DS: also store dS^T (bf16, exactly the dK MMA's operand) to global memory — row
// (b*H + h)*T + key, column query — for the dQ GEMM (dq_gemm_k) that then replaces dq_k's
// S / dP recomputation.  Each compute warp stages its [32 keys][64 queries] block in shared
// memory (128-byte swizzle) and issues its own TMA store; the Q ring drops to two slots to
// make room for the 32 KB stage.
template <int NQ, bool DS>
__global__ void __launch_bounds__(128 + 128 * NQ, 1)
    dkdv_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG,
           const __grid_constant__ CUtensorMap tmS, const Params p) {
  constexpr int kQSlots = DS ? 2 : tcb::kQSlots;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem) & 1023) __trap();  // see kSmemDkdv
  CTA_TRACE(0, 0);
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* sQ = smem + 2 * kTile;                               // [kQSlots]
  uint8_t* sG = sQ + kQSlots * kTile;                           // [kGSlots]
  uint8_t* sStage = sG + kGSlots * kTile;                       // DS: [NQ][128 keys][64 queries]
  float* sLD = reinterpret_cast<float*>(sG + (kGSlots + (DS ? 1 : 0)) * kTile);  // [2] x {lse, delta}
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sLD) + 2048);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;     // [3]
  uint64_t* q_empty = bars + 4;    // [3]
  uint64_t* g_full = bars + 7;     // [2]
  uint64_t* g_empty = bars + 9;    // [2]
  uint64_t* ld_full = bars + 11;   // [2]
  uint64_t* ld_empty = bars + 13;  // [2]
  uint64_t* s_full = bars + 15;
  uint64_t* dp_full = bars + 16;
  uint64_t* s_free = bars + 17;    // the compute warps hold S^T(u) in registers
  uint64_t* pd_ready = bars + 18;  // dS^T(u) is in the dP^T region (after P^T)
  uint64_t* mma_done = bars + 19;
  uint64_t* p_ready = bars + 20;   // P^T(u) is in the dP^T region: dV(u) may start
  uint64_t* ds_part = bars + 21;   // the first half of each group's dS^T(u) is stored
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int group = p.H / p.KVH;
  const int nq = (p.T + BT - 1) / BT;
  const int total = group * nq;  // 128-query tiles to sweep
  const int row0 = b * p.T, k0 = kt * BT;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmG);
    mbar_init(kv_full, 1);
    for (int s = 0; s < kQSlots; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&g_full[s], 1);
      mbar_init(&g_empty[s], 1);
      mbar_init(&ld_full[s], 1);
      mbar_init(&ld_empty[s], 4 * NQ);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(s_free, 4 * NQ);
    mbar_init(pd_ready, 4 * NQ);
    mbar_init(p_ready, 4 * NQ);
    mbar_init(ds_part, 4 * NQ);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cS = 0, cP = 128, cV = 256, cK = 384;

  if (warp == 0) {
    // producer A: K, V once, then the Q tiles (3-slot ring; a slot frees after dK(u))
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * kTile);
      tma_load_2d(sK, &tmK, kv_full, kvh * HD, row0 + k0);
      tma_load_2d(sK + kBox, &tmK, kv_full, kvh * HD + 64, row0 + k0);
      tma_load_2d(sV, &tmV, kv_full, kvh * HD, row0 + k0);
      tma_load_2d(sV + kBox, &tmV, kv_full, kvh * HD + 64, row0 + k0);
      for (int it = 0; it < total; ++it) {
        const int st = it % kQSlots;
        const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
        mbar_wait(&q_empty[st], ((it / kQSlots) & 1) ^ 1);
        BWD_TRACE(8, it);
        mbar_expect_tx(&q_full[st], kTile);
        tma_load_2d(sQ + st * kTile, &tmQ, &q_full[st], h * HD, row0 + q0);
        tma_load_2d(sQ + st * kTile + kBox, &tmQ, &q_full[st], h * HD + 64, row0 + q0);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // producer B: dO tiles (a slot frees after dV(u)) and the lse / delta rows of each tile
    // (bulk copies; a slot frees once the compute warps finished the dS pass)
    if (lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int st = it & 1;
        const uint32_t ph = ((it >> 1) & 1) ^ 1;
        const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
        mbar_wait(&g_empty[st], ph);
        BWD_TRACE(9, it);
        mbar_expect_tx(&g_full[st], kTile);
        tma_load_2d(sG + st * kTile, &tmG, &g_full[st], h * HD, row0 + q0);
        tma_load_2d(sG + st * kTile + kBox, &tmG, &g_full[st], h * HD + 64, row0 + q0);
        const int nvalid = min(BT, p.T - q0);
        const uint32_t bytes = (uint32_t)nvalid * 4u;
        const int64_t li = ((int64_t)b * p.H + h) * p.T + q0;
        mbar_wait(&ld_empty[st], ph);
        // ragged last tile: lse = +inf makes P (hence dS) vanish for query columns past T,
        // so the compute warps need no masking
        for (int i = nvalid; i < BT; ++i) {
          sLD[st * 256 + i] = INFINITY;
          sLD[st * 256 + 128 + i] = 0.f;
        }
        mbar_expect_tx(&ld_full[st], 2 * bytes);
        bulk_load(sLD + st * 256, p.lse + li, bytes, &ld_full[st]);
        bulk_load(sLD + st * 256 + 128, p.delta + li, bytes, &ld_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the schedule (warp-uniform descriptors in uniform
    // registers); one elected lane issues each MMA group
    const uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);    // K-major x K-major
    const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);  // TMEM A x MN-major B
    const uint64_t dK = sw128_desc(smem_u32(sK), 16, 1024), dV = sw128_desc(smem_u32(sV), 16, 1024);
    auto tileQ = [&](int u) { return smem_u32(sQ + (u % kQSlots) * kTile); };
    auto tileG = [&](int u) { return smem_u32(sG + (u & 1) * kTile); };
    auto issue_s = [&](int u) {
      mbar_wait(&q_full[u % kQSlots], (u / kQSlots) & 1);
      tc_fence_after();
      BWD_TRACE(1, u);
      const uint64_t dQ = sw128_desc(tileQ(u), 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cS, dK + koff(kk), dQ + koff(kk), id_s, kk > 0);
        umma_commit(s_full);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int u) {
      mbar_wait(&g_full[u & 1], (u >> 1) & 1);
      tc_fence_after();
      BWD_TRACE(3, u);
      const uint64_t dG = sw128_desc(tileG(u), 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, dV + koff(kk), dG + koff(kk), id_s, kk > 0);
        umma_commit(dp_full);
      }
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    tc_fence_after();
    issue_s(0);
    issue_dp(0);
    for (int u = 0; u < total; ++u) {
      const uint64_t mQ = sw128_desc(tileQ(u), kBox, 1024), mG = sw128_desc(tileG(u), kBox, 1024);
      if (u + 1 < total) {  // S^T region: tile u is in registers
        mbar_wait(s_free, u & 1);
        tc_fence_after();
        issue_s(u + 1);
      }
      mbar_wait(p_ready, u & 1);  // dV(u) runs while the compute warps form dS^T(u)
      tc_fence_after();
      BWD_TRACE(0, u);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          umma_f16_ts(tmem + cV, tmem + cP + packed_colq<NQ>(k), mG + (uint64_t)(k * 128), id_acc, (u | k) != 0);
        umma_commit(&g_empty[u & 1]);  // dO(u) is done (dP(u) and dV(u))
      }
      __syncwarp();
      // dK += dS^T Q in two parts: the K-steps over the first half of each group's query
      // columns once stored (ds_part), the rest after the whole dS pass
      constexpr int KPG = BT / 16 / NQ;  // K-steps per query-column group
      mbar_wait(ds_part, u & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          if (k % KPG < KPG / 2)
            umma_f16_ts(tmem + cK, tmem + cP + 64 / NQ + packed_colq<NQ>(k), mQ + (uint64_t)(k * 128), id_acc,
                        (u | k) != 0);
      }
      __syncwarp();
      mbar_wait(pd_ready, u & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          if (k % KPG >= KPG / 2)
            umma_f16_ts(tmem + cK, tmem + cP + 64 / NQ + packed_colq<NQ>(k), mQ + (uint64_t)(k * 128), id_acc, 1);
        umma_commit(&q_empty[u % kQSlots]);
      }
      __syncwarp();
      BWD_TRACE(2, u);
      if (u + 1 < total) issue_dp(u + 1);  // dP^T region: P^T(u), dS^T(u) consumed (in order)
    }
    if (elect_one()) umma_commit(mma_done);
    __syncwarp();
  } else if (warp >= 4) {
    constexpr int W = 128 / NQ;  // query columns per compute warp
    constexpr int NP = W / 2;    // column pairs
    const int q = warp & 3;
    const int grp = (warp - 4) >> 2;  // query-column group of each tile
    const int t = q * 32 + lane;      // key row inside the tile
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const uint32_t col = (uint32_t)grp * W;
    const float c = p.scale * kLog2e;
    const float2 c2 = make_float2(c, c), nlog2e = make_float2(-kLog2e, -kLog2e);
    if (warp == 4) BWD_TRACE(19, 0);  // compute warps start
    for (int u = 0; u < total; ++u) {
      mbar_wait(&ld_full[u & 1], (u >> 1) & 1);
      const uint32_t sL = smem_u32(sLD + (u & 1) * 256 + grp * W);  // lse; delta at +128 floats
      mbar_wait(s_full, u & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(4, u);
      float2 pr[NP];
      {
        uint32_t sv[W / 32][32];
        ldW<W>(tmem + lo + cS + col, sv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
#pragma unroll
        for (int i = 0; i < NP; i += 2) {
          const float4 l4 = lds4(sL + 8 * i);
          pr[i] = exp2_pair(ffma2(colp(sv, i), c2, fmul2(make_float2(l4.x, l4.y), nlog2e)), i);
          pr[i + 1] = exp2_pair(ffma2(colp(sv, i + 1), c2, fmul2(make_float2(l4.z, l4.w), nlog2e)), i + 1);
        }
      }
      if (warp == 4) BWD_TRACE(5, u);
      mbar_wait(dp_full, u & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(6, u);
      {
        uint32_t dv[W / 32][32];
        ldW<W>(tmem + lo + cP + col, dv);
        // P^T first (over this group's dP^T columns, now in registers), so dV(u) starts while
        // dS^T is formed
        pack_storeN<NP>(tmem + lo + cP + col, pr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready);
        // dS^T next to it, in two halves (ds_part after the first) when a half fills whole
        // 16-column TMEM stores
        constexpr int kParts = NP >= 32 ? 2 : 1;
        // DS: this warp's stage block (32 key rows x 128 bytes); its previous TMA store has
        // finished reading it before it is overwritten
        uint8_t* stg = sStage + grp * (128 * 128) + q * (32 * 128);
        if (DS) {
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll
        for (int part = 0; part < kParts; ++part) {
          float2 ds[NP / kParts];
#pragma unroll
          for (int i = 0; i < NP / kParts; i += 2) {
            const int c2i = part * (NP / kParts) + i;
            const float4 d4 = lds4(sL + 512 + 8 * c2i);
            ds[i] = fmul2(pr[c2i], ffma2(make_float2(d4.x, d4.y), make_float2(-1.f, -1.f), colp(dv, c2i)));
            ds[i + 1] =
                fmul2(pr[c2i + 1], ffma2(make_float2(d4.z, d4.w), make_float2(-1.f, -1.f), colp(dv, c2i + 1)));
          }
          pack_storeN<NP / kParts>(tmem + lo + cP + col + NP + part * (NP / kParts), ds);
          if (DS) {  // the same bf16 pairs, 16-byte chunks at their 128B-swizzled positions
            constexpr int kChunks = NP / kParts / 4;
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
              const int lc = part * kChunks + c;
              uint4 v;
              v.x = pack2(ds[4 * c].x, ds[4 * c].y);
              v.y = pack2(ds[4 * c + 1].x, ds[4 * c + 1].y);
              v.z = pack2(ds[4 * c + 2].x, ds[4 * c + 2].y);
              v.w = pack2(ds[4 * c + 3].x, ds[4 * c + 3].y);
              *reinterpret_cast<uint4*>(stg + lane * 128 + ((lc ^ (lane & 7)) << 4)) = v;
            }
          }
          if (part == 0) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_part);
          }
        }
      }
      if (DS) {
        fence_async_smem();  // the stage's generic-proxy writes, visible to the TMA store
        __syncwarp();
        if (lane == 0) {
          const int hq = kvh * group + u / nq, qs = (u % nq) * BT;
          tma_store_2d(&tmS, sStage + grp * (128 * 128) + q * (32 * 128), qs + grp * W,
                       (b * p.H + hq) * p.T + k0 + q * 32);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 4) BWD_TRACE(7, u);
      if (lane == 0) {
        mbar_arrive(pd_ready);
        mbar_arrive(&ld_empty[u & 1]);
      }
    }
    if (DS && lane == 0) bulk_wait0();  // every dS^T store has landed before the CTA exits
    mbar_wait(mma_done, 0);
    tc_fence_after();
    if (warp == 4) BWD_TRACE(20, 0);  // last MMA done: epilogue starts
    const int krow = k0 + t;
    const bool ok = krow < p.T;
    // the 256 output columns (dK | dV) split evenly over the NQ groups
    constexpr int kCh = 8 / NQ;  // 32-column chunks per group
    const int c0 = grp * kCh * 32;
    if (c0 < 128) {
      const float* rc = p.rope_cos ? p.rope_cos + (int64_t)(ok ? krow : 0) * (HD / 2) + c0 / 2 : nullptr;
      const float* rs = p.rope_sin ? p.rope_sin + (int64_t)(ok ? krow : 0) * (HD / 2) + c0 / 2 : nullptr;
      store_row(tmem + lo + cK + c0, p.o0 + ((int64_t)row0 + krow) * p.ld0 + (int64_t)kvh * HD + c0, p.scale, ok, rc,
                rs, kCh);
    } else {
      store_row(tmem + lo + cV + (c0 - 128), p.o1 + ((int64_t)row0 + krow) * p.ld1 + (int64_t)kvh * HD + (c0 - 128),
                1.f, ok, nullptr, nullptr, kCh);
    }
    if (warp == 4) BWD_TRACE(21, 0);  // epilogue stores issued
  }
  tc_fence_before();
  __syncthreads();
  CTA_TRACE(0, 1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// CTA-pair (cta_group::2) helpers of the pair sweeps below
constexpr int kBoxH = 64 * 64 * 2;  // one [64 rows][64 cols] bf16 box (8 KB)

// descriptor offset of the kk-th K=16 step of a K-major [64][128] half tile (two 64-col boxes)
__device__ __forceinline__ uint64_t koff64(int kk) { return (uint64_t)(((kk >> 2) * kBoxH + (kk & 3) * 32) >> 4); }

__device__ __forceinline__ void umma_f16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// ====================================================================== dK / dV on CTA pairs
// The dK/dV sweep with cta_group::2 MMAs: a cluster of two CTAs owns 256 keys (128 each); for
// every 128-query tile each pair MMA (M = 256, issued by the leader) takes each CTA's own 128
// rows of A (K, V, or P^T / dS^T from its TMEM) and half of B:
//   S^T  = K Q_u^T   : B = its 64 queries of Q_u (all head dims)      [64 x 128, K-major]
//   dP^T = V dO_u^T  : B = its 64 queries of dO_u                     [64 x 128, K-major]
//   dV  += P^T dO_u  : B = all 128 queries of dO_u, its 64 head dims  [128 x 64, MN-major]
//   dK  += dS^T Q_u  : B = all 128 queries of Q_u, its 64 head dims   [128 x 64, MN-major]
// so each SM reads ~192 KB of shared memory per tile instead of ~256 KB (the single-CTA
// sweep's bound, at its 2048-cycle MMA time).  TMA loads of K/V, Q and dO complete on the
// leader's barriers, MMA completions are multicast, the compute warps' signals reach the
// leader's barriers with relaxed cluster arrives (tcgen05 fences order the TMEM accesses).
// lse / delta rows stay per-CTA (bulk copies, local barriers).  Same arithmetic and order as
// dkdv_k<NQ, false>.  Requires T % 256 == 0 (else dkdv_k runs).
template <int NQ>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 128 * NQ, 1)
    dkdv_pair_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQ64,
                const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmG64, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem) & 1023) __trap();  // see kSmemDkdv
  CTA_TRACE(0, 0);
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* sQ = smem + 2 * kTile;      // [kQSlots] {its 64 queries x 128 dims | 128 queries x its 64 dims}
  uint8_t* sG = sQ + kQSlots * kTile;  // [kGSlots] same for dO
  float* sLD = reinterpret_cast<float*>(sG + kGSlots * kTile);  // [2] x {lse, delta}
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sLD) + 2048);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;     // [3]
  uint64_t* q_empty = bars + 4;    // [3]
  uint64_t* g_full = bars + 7;     // [2]
  uint64_t* g_empty = bars + 9;    // [2]
  uint64_t* ld_full = bars + 11;   // [2] (per CTA)
  uint64_t* ld_empty = bars + 13;  // [2] (per CTA)
  uint64_t* s_full = bars + 15;
  uint64_t* dp_full = bars + 16;
  uint64_t* s_free = bars + 17;
  uint64_t* pd_ready = bars + 18;
  uint64_t* mma_done = bars + 19;
  uint64_t* p_ready = bars + 20;
  uint64_t* ds_part = bars + 21;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int kvh = blockIdx.y, b = blockIdx.z;
  const int group = p.H / p.KVH;
  const int nq = p.T / BT;
  const int total = group * nq;
  const int row0 = b * p.T, k0 = (blockIdx.x >> 1) * 2 * BT + (int)rank * BT;
  constexpr int kSig = 2 * 4 * NQ;  // compute-warp signals per phase (both CTAs)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmQ64);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmG);
    tma_prefetch_desc(&tmG64);
    mbar_init(kv_full, 1);
    for (int s = 0; s < kQSlots; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&g_full[s], 1);
      mbar_init(&g_empty[s], 1);
      mbar_init(&ld_full[s], 1);
      mbar_init(&ld_empty[s], 4 * NQ);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(s_free, kSig);
    mbar_init(pd_ready, kSig);
    mbar_init(p_ready, kSig);
    mbar_init(ds_part, kSig);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(slot, kCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cS = 0, cP = 128, cV = 256, cK = 384;

  if (warp == 0) {
    // producer A: its K, V rows once, then per query tile its halves of Q_u
    if (elect_one()) {
      const uint32_t fkv = leader_addr(kv_full);
      if (leader) mbar_expect_tx(kv_full, 2 * 2 * kTile);
      tma_load_2d_pair(sK, &tmK, fkv, kvh * HD, row0 + k0);
      tma_load_2d_pair(sK + kBox, &tmK, fkv, kvh * HD + 64, row0 + k0);
      tma_load_2d_pair(sV, &tmV, fkv, kvh * HD, row0 + k0);
      tma_load_2d_pair(sV + kBox, &tmV, fkv, kvh * HD + 64, row0 + k0);
      for (int it = 0; it < total; ++it) {
        const int st = it % kQSlots;
        const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
        mbar_wait(&q_empty[st], ((it / kQSlots) & 1) ^ 1);
        BWD_TRACE(8, it);
        const uint32_t fq = leader_addr(&q_full[st]);
        if (leader) mbar_expect_tx(&q_full[st], 2 * kTile);
        uint8_t* dst = sQ + st * kTile;
        tma_load_2d_pair(dst, &tmQ64, fq, h * HD, row0 + q0 + (int)rank * 64);
        tma_load_2d_pair(dst + kBoxH, &tmQ64, fq, h * HD + 64, row0 + q0 + (int)rank * 64);
        tma_load_2d_pair(dst + kBox, &tmQ, fq, h * HD + (int)rank * 64, row0 + q0);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // producer B: its halves of dO_u (leader's barriers) and the lse / delta rows (its own)
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int st = it & 1;
        const uint32_t ph = ((it >> 1) & 1) ^ 1;
        const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
        mbar_wait(&g_empty[st], ph);
        BWD_TRACE(9, it);
        const uint32_t fg = leader_addr(&g_full[st]);
        if (leader) mbar_expect_tx(&g_full[st], 2 * kTile);
        uint8_t* dst = sG + st * kTile;
        tma_load_2d_pair(dst, &tmG64, fg, h * HD, row0 + q0 + (int)rank * 64);
        tma_load_2d_pair(dst + kBoxH, &tmG64, fg, h * HD + 64, row0 + q0 + (int)rank * 64);
        tma_load_2d_pair(dst + kBox, &tmG, fg, h * HD + (int)rank * 64, row0 + q0);
        const uint32_t bytes = (uint32_t)BT * 4u;
        const int64_t li = ((int64_t)b * p.H + h) * p.T + q0;
        mbar_wait(&ld_empty[st], ph);
        mbar_expect_tx(&ld_full[st], 2 * bytes);
        bulk_load(sLD + st * 256, p.lse + li, bytes, &ld_full[st]);
        bulk_load(sLD + st * 256 + 128, p.delta + li, bytes, &ld_full[st]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      const uint32_t id_s = idesc_bf16_f32(256, 128, 0, 0);    // K-major x K-major
      const uint32_t id_acc = idesc_bf16_f32(256, 128, 0, 1);  // TMEM A x MN-major B
      const uint64_t dK = sw128_desc(smem_u32(sK), 16, 1024), dV = sw128_desc(smem_u32(sV), 16, 1024);
      auto tileQ = [&](int u) { return smem_u32(sQ + (u % kQSlots) * kTile); };
      auto tileG = [&](int u) { return smem_u32(sG + (u & 1) * kTile); };
      auto issue_s = [&](int u) {
        mbar_wait(&q_full[u % kQSlots], (u / kQSlots) & 1);
        tc_fence_after();
        BWD_TRACE(1, u);
        const uint64_t dQ = sw128_desc(tileQ(u), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            umma_f16_ss_pair(tmem + cS, dK + koff(kk), dQ + koff64(kk), id_s, kk > 0);
          umma_commit_pair_mc(s_full, 0x3);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int u) {
        mbar_wait(&g_full[u & 1], (u >> 1) & 1);
        tc_fence_after();
        BWD_TRACE(3, u);
        const uint64_t dG = sw128_desc(tileG(u), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            umma_f16_ss_pair(tmem + cP, dV + koff(kk), dG + koff64(kk), id_s, kk > 0);
          umma_commit_pair_mc(dp_full, 0x3);
        }
        __syncwarp();
      };
      mbar_wait(kv_full, 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int u = 0; u < total; ++u) {
        // B of dV / dK: all 128 queries x this CTA's 64 head dims (one MN-major atom)
        const uint64_t mQ = sw128_desc(tileQ(u) + kBox, kBox, 1024), mG = sw128_desc(tileG(u) + kBox, kBox, 1024);
        if (u + 1 < total) {
          mbar_wait(s_free, u & 1);
          tc_fence_after();
          issue_s(u + 1);
        }
        mbar_wait(p_ready, u & 1);
        tc_fence_after();
        BWD_TRACE(0, u);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)
            umma_f16_ts_pair(tmem + cV, tmem + cP + packed_colq<NQ>(k), mG + (uint64_t)(k * 128), id_acc,
                             (u | k) != 0);
          umma_commit_pair_mc(&g_empty[u & 1], 0x3);
        }
        __syncwarp();
        constexpr int KPG = BT / 16 / NQ;
        mbar_wait(ds_part, u & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)
            if (k % KPG < KPG / 2)
              umma_f16_ts_pair(tmem + cK, tmem + cP + 64 / NQ + packed_colq<NQ>(k), mQ + (uint64_t)(k * 128), id_acc,
                               (u | k) != 0);
        }
        __syncwarp();
        mbar_wait(pd_ready, u & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)
            if (k % KPG >= KPG / 2)
              umma_f16_ts_pair(tmem + cK, tmem + cP + 64 / NQ + packed_colq<NQ>(k), mQ + (uint64_t)(k * 128), id_acc,
                               1);
          umma_commit_pair_mc(&q_empty[u % kQSlots], 0x3);
        }
        __syncwarp();
        BWD_TRACE(2, u);
        if (u + 1 < total) issue_dp(u + 1);
      }
      if (elect_one()) umma_commit_pair_mc(mma_done, 0x3);
      __syncwarp();
    }
  } else if (warp >= 4) {
    constexpr int W = 128 / NQ;
    constexpr int NP = W / 2;
    const int q = warp & 3;
    const int grp = (warp - 4) >> 2;
    const int t = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const uint32_t col = (uint32_t)grp * W;
    const float c = p.scale * kLog2e;
    const float2 c2 = make_float2(c, c), nlog2e = make_float2(-kLog2e, -kLog2e);
    const uint32_t s_free_l = leader_addr(s_free), p_ready_l = leader_addr(p_ready);
    const uint32_t ds_part_l = leader_addr(ds_part), pd_ready_l = leader_addr(pd_ready);
    for (int u = 0; u < total; ++u) {
      mbar_wait(&ld_full[u & 1], (u >> 1) & 1);
      const uint32_t sL = smem_u32(sLD + (u & 1) * 256 + grp * W);
      mbar_wait(s_full, u & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(4, u);
      float2 pr[NP];
      {
        uint32_t sv[W / 32][32];
        ldW<W>(tmem + lo + cS + col, sv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(s_free_l);
#pragma unroll
        for (int i = 0; i < NP; i += 2) {
          const float4 l4 = lds4(sL + 8 * i);
          pr[i] = exp2_pair(ffma2(colp(sv, i), c2, fmul2(make_float2(l4.x, l4.y), nlog2e)), i);
          pr[i + 1] = exp2_pair(ffma2(colp(sv, i + 1), c2, fmul2(make_float2(l4.z, l4.w), nlog2e)), i + 1);
        }
      }
      if (warp == 4) BWD_TRACE(5, u);
      mbar_wait(dp_full, u & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(6, u);
      {
        uint32_t dv[W / 32][32];
        ldW<W>(tmem + lo + cP + col, dv);
        pack_storeN<NP>(tmem + lo + cP + col, pr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(p_ready_l);
        constexpr int kParts = NP >= 32 ? 2 : 1;
#pragma unroll
        for (int part = 0; part < kParts; ++part) {
          float2 ds[NP / kParts];
#pragma unroll
          for (int i = 0; i < NP / kParts; i += 2) {
            const int c2i = part * (NP / kParts) + i;
            const float4 d4 = lds4(sL + 512 + 8 * c2i);
            ds[i] = fmul2(pr[c2i], ffma2(make_float2(d4.x, d4.y), make_float2(-1.f, -1.f), colp(dv, c2i)));
            ds[i + 1] =
                fmul2(pr[c2i + 1], ffma2(make_float2(d4.z, d4.w), make_float2(-1.f, -1.f), colp(dv, c2i + 1)));
          }
          pack_storeN<NP / kParts>(tmem + lo + cP + col + NP + part * (NP / kParts), ds);
          if (part == 0) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(ds_part_l);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 4) BWD_TRACE(7, u);
      if (lane == 0) {
        mbar_arrive_cluster_relaxed(pd_ready_l);
        mbar_arrive(&ld_empty[u & 1]);
      }
    }
    mbar_wait(mma_done, 0);
    tc_fence_after();
    const int krow = k0 + t;
    constexpr int kCh = 8 / NQ;
    const int c0 = grp * kCh * 32;
    if (c0 < 128) {
      const float* rc = p.rope_cos ? p.rope_cos + (int64_t)krow * (HD / 2) + c0 / 2 : nullptr;
      const float* rs = p.rope_sin ? p.rope_sin + (int64_t)krow * (HD / 2) + c0 / 2 : nullptr;
      store_row(tmem + lo + cK + c0, p.o0 + ((int64_t)row0 + krow) * p.ld0 + (int64_t)kvh * HD + c0, p.scale, true,
                rc, rs, kCh);
    } else {
      store_row(tmem + lo + cV + (c0 - 128), p.o1 + ((int64_t)row0 + krow) * p.ld1 + (int64_t)kvh * HD + (c0 - 128),
                1.f, true, nullptr, nullptr, kCh);
    }
  }
  tc_fence_before();
  cluster_sync();
  CTA_TRACE(0, 1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, kCols);
  }
}

// =========================================================================== dQ
__global__ void __launch_bounds__(kThreads, 1)
    dq_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  CTA_TRACE(1, 0);
  uint8_t* sQ = smem;
  uint8_t* sG = smem + kTile;
  uint8_t* sK = smem + 2 * kTile;      // [kKSlots]
  uint8_t* sV = sK + kKSlots * kTile;  // [kVSlots]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVSlots * kTile);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [3]
  uint64_t* k_empty = bars + 4;  // [3]
  uint64_t* v_full = bars + 7;   // [2]
  uint64_t* v_empty = bars + 9;  // [2]
  uint64_t* s_full = bars + 11;  // [2]
  uint64_t* dp_full = bars + 13;
  uint64_t* ds_ready = bars + 14;
  uint64_t* mma_done = bars + 15;
  uint64_t* ds_part = bars + 16;  // the first 32 key columns of each half's dS are in TMEM
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.KVH);
  const int nk = (p.T + BT - 1) / BT;
  const int row0 = b * p.T, q0 = qt * BT;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmG);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 8);
    mbar_init(ds_part, 8);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cP = 256, cQ = 384;  // S buffers at (j & 1) * 128

  if (warp == 0) {
    // producer A: Q, dO once, then K_j (3-deep ring; a slot frees after dQ(j))
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kTile);
      tma_load_2d(sQ, &tmQ, q_full, h * HD, row0 + q0);
      tma_load_2d(sQ + kBox, &tmQ, q_full, h * HD + 64, row0 + q0);
      tma_load_2d(sG, &tmG, q_full, h * HD, row0 + q0);
      tma_load_2d(sG + kBox, &tmG, q_full, h * HD + 64, row0 + q0);
      for (int j = 0; j < nk; ++j) {
        const int st = j % kKSlots;
        mbar_wait(&k_empty[st], ((j / kKSlots) & 1) ^ 1);
        BWD_TRACE(16, j);
        mbar_expect_tx(&k_full[st], kTile);
        tma_load_2d(sK + st * kTile, &tmK, &k_full[st], kvh * HD, row0 + j * BT);
        tma_load_2d(sK + st * kTile + kBox, &tmK, &k_full[st], kvh * HD + 64, row0 + j * BT);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // producer B: V_j (a slot frees after dP(j))
    if (lane == 0) {
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        BWD_TRACE(17, j);
        mbar_expect_tx(&v_full[st], kTile);
        tma_load_2d(sV + st * kTile, &tmV, &v_full[st], kvh * HD, row0 + j * BT);
        tma_load_2d(sV + st * kTile + kBox, &tmV, &v_full[st], kvh * HD + 64, row0 + j * BT);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);
    const uint64_t dQ = sw128_desc(smem_u32(sQ), 16, 1024), dG = sw128_desc(smem_u32(sG), 16, 1024);
    auto issue_s = [&](int j) {
      const int ks = j % kKSlots;
      BWD_TRACE(18, j);
      mbar_wait(&k_full[ks], (j / kKSlots) & 1);
      tc_fence_after();
      BWD_TRACE(10, j);
      const uint64_t dKj = sw128_desc(smem_u32(sK + ks * kTile), 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_f16_ss(tmem + (j & 1) * 128u, dQ + koff(kk), dKj + koff(kk), id_s, kk > 0);
        umma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int j) {
      mbar_wait(&v_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      BWD_TRACE(12, j);
      const uint64_t dVj = sw128_desc(smem_u32(sV + (j & 1) * kTile), 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, dG + koff(kk), dVj + koff(kk), id_s, kk > 0);
        umma_commit(dp_full);
        umma_commit(&v_empty[j & 1]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    issue_s(0);
    issue_dp(0);
    for (int j = 0; j < nk; ++j) {
      const int st = j & 1;
      if (j + 1 < nk) issue_s(j + 1);
      // dQ += dS K in two parts: the K-steps over the first 32 keys of each half (k = 0, 1,
      // 4, 5) once those dS columns are stored, the rest after the whole dS pass
      const uint64_t mK = sw128_desc(smem_u32(sK + (j % kKSlots) * kTile), kBox, 1024);
      mbar_wait(ds_part, j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          if ((k & 3) < 2)
            umma_f16_ts(tmem + cQ, tmem + st * 128u + packed_col(k), mK + (uint64_t)(k * 128), id_acc,
                        (j | k) != 0);
      }
      __syncwarp();
      mbar_wait(ds_ready, j & 1);
      tc_fence_after();
      BWD_TRACE(11, j);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          if ((k & 3) >= 2)
            umma_f16_ts(tmem + cQ, tmem + st * 128u + packed_col(k), mK + (uint64_t)(k * 128), id_acc, 1);
        umma_commit(&k_empty[j % kKSlots]);
      }
      __syncwarp();
      if (j + 1 < nk) issue_dp(j + 1);
    }
    if (elect_one()) umma_commit(mma_done);
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int ch = (warp - 4) >> 2;  // key-column half of each tile
    const int t = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float c = p.scale * kLog2e;
    const int qrow = q0 + t;
    const bool ok = qrow < p.T;
    const int64_t li = ((int64_t)b * p.H + h) * p.T + qrow;
    const float L = ok ? p.lse[li] * kLog2e : 0.f;
    const float D = ok ? p.delta[li] : 0.f;
    const float2 c2 = make_float2(c, c), nl2 = make_float2(-L, -L), nd2 = make_float2(-D, -D);
    for (int j = 0; j < nk; ++j) {
      const int st = j & 1;
      const int valid = min(BT, p.T - j * BT) - ch * 64;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(13, j);
      float2 pr[32];
      {
        uint32_t sv[2][32];
        ld64(tmem + lo + st * 128u + ch * 64, sv);
#pragma unroll
        for (int i = 0; i < 32; ++i) pr[i] = exp2_pair(ffma2(col2(sv, i), c2, nl2), i);
        if (valid < 64) {  // key columns past T
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (2 * i >= valid) pr[i].x = 0.f;
            if (2 * i + 1 >= valid) pr[i].y = 0.f;
          }
        }
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(14, j);
      {
        uint32_t dv[2][32];
        ld64(tmem + lo + cP + ch * 64, dv);
        // dS over this half's own S columns, in two 32-column parts (ds_part after the first)
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 d = fmul2(pr[16 * part + i], fadd2(col2(dv, 16 * part + i), nd2));
            pk[i] = pack2(d.x, d.y);
          }
          tmem_st16(tmem + lo + st * 128u + ch * 64 + 16 * part, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (part == 0 && lane == 0) mbar_arrive(ds_part);
        }
      }
      if (warp == 4) BWD_TRACE(15, j);
      if (lane == 0) mbar_arrive(ds_ready);
    }
    mbar_wait(mma_done, 0);
    tc_fence_after();
    const float* rc = p.rope_cos ? p.rope_cos + (int64_t)(ok ? qrow : 0) * (HD / 2) + ch * 32 : nullptr;
    const float* rs = p.rope_sin ? p.rope_sin + (int64_t)(ok ? qrow : 0) * (HD / 2) + ch * 32 : nullptr;
    store_row(tmem + lo + cQ + ch * 64, p.o0 + ((int64_t)row0 + qrow) * p.ld0 + (int64_t)h * HD + ch * 64, p.scale,
              ok, rc, rs, 2);
  }
  tc_fence_before();
  __syncthreads();
  CTA_TRACE(1, 1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// 1 (default): the dQ sweep on CTA pairs (dq_pair_k) when T % 256 == 0 (cb_attention_set_dq_pair)
int g_dq_pair = 1;
// 1: the dK/dV sweep on CTA pairs (dkdv_pair_k) when T % 256 == 0 (cb_attention_set_dkdv_pair)
int g_dkdv_pair = 0;

// ============================================================ dQ sweep on CTA pairs
// The dQ sweep with cta_group::2 MMAs: a cluster of two CTAs owns 256 query rows (128 each);
// every MMA is one pair instruction (M = 256) issued by the leader, each CTA supplying its own
// 128 rows of A (Q, dO, or dS from its TMEM) and half of B:
//   S  = Q K_j^T  : B = its 64 keys of K_j (all 128 head dims)     [64 x 128, K-major]
//   dP = dO V_j^T : B = its 64 keys of V_j                          [64 x 128, K-major]
//   dQ += dS K_j  : B = all 128 keys of K_j, its 64 head-dim columns [128 x 64, MN-major]
// so each SM reads 160 KB of shared memory per key tile instead of the single-CTA sweep's
// 224 KB (which bounds that kernel above its 1536-cycle MMA time).  The pair instruction runs
// at the single-CTA per-SM rate at N = 128 (profiles/r02_ubench_mma_pair.txt).  TMA loads of
// both CTAs complete on the leader's barriers; MMA completions are multicast to both CTAs; the
// compute warps of both CTAs signal dP-consumed / dS-ready on the leader's barriers with
// relaxed cluster arrives (the tcgen05 fences order the TMEM accesses; a release at cluster
// scope cost ~1300 cycles per signal on the critical chain).  Same arithmetic and order as
// dq_k.  Requires T % 256 == 0 (else dq_k runs).
constexpr int kSmemDqPair = 2 * kTile + kKSlots * (2 * kBoxH + kBox) + kVSlots * (2 * kBoxH) + 1024 + 256;


__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    dq_pair_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmK64, const __grid_constant__ CUtensorMap tmV64,
              const __grid_constant__ CUtensorMap tmG, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  CTA_TRACE(1, 0);
  uint8_t* sQ = smem;
  uint8_t* sG = smem + kTile;
  uint8_t* sKs = smem + 2 * kTile;                 // [kKSlots] this CTA's 64 keys of K_j (S operand)
  uint8_t* sKq = sKs + kKSlots * 2 * kBoxH;        // [kKSlots] K_j's 128 keys x this CTA's 64 dims
  uint8_t* sV = sKq + kKSlots * kBox;              // [kVSlots] this CTA's 64 keys of V_j
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVSlots * 2 * kBoxH);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [3]  (leader's copy counts both CTAs' loads)
  uint64_t* k_empty = bars + 4;  // [3]  (multicast by the leader's MMA commits)
  uint64_t* v_full = bars + 7;   // [2]
  uint64_t* v_empty = bars + 9;  // [2]
  uint64_t* s_full = bars + 11;  // [2]
  uint64_t* dp_full = bars + 13;
  // leader's copies, 16 arrivals each (8 compute warps x 2 CTAs).  ds_ready / ds_part are
  // double-buffered by tile parity: dP(j+1) is issued on dp_free(j), so a fast warp can reach
  // tile j+1's dS signals before a slow one has given tile j's (never two tiles ahead: dP(j+2)
  // needs every warp's dp_free(j+1)); one barrier per parity keeps the phases apart
  uint64_t* ds_ready = bars + 14;  // [2]
  uint64_t* mma_done = bars + 16;
  uint64_t* ds_part = bars + 17;  // [2]
  uint64_t* dp_free = bars + 19;  // dP(j) is in the compute warps' registers
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.KVH);
  const int nk = p.T / BT;
  const int row0 = b * p.T, q0 = (blockIdx.x >> 1) * 2 * BT + (int)rank * BT;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmK64);
    tma_prefetch_desc(&tmV64);
    tma_prefetch_desc(&tmG);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(dp_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ds_ready[s], 16);
      mbar_init(&ds_part[s], 16);
    }
    mbar_init(dp_free, 16);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(slot, kCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cP = 256, cQ = 384;  // S buffers at (j & 1) * 128

  if (warp == 0) {
    // producer A (both CTAs): own Q, dO rows once, then per key tile its 64 keys of K_j (two
    // [64][64] boxes) and K_j's 128 keys x its 64 head dims; completions on the leader's barriers
    if (elect_one()) {
      const uint32_t fq = leader_addr(q_full);
      if (leader) mbar_expect_tx(q_full, 2 * 2 * kTile);
      tma_load_2d_pair(sQ, &tmQ, fq, h * HD, row0 + q0);
      tma_load_2d_pair(sQ + kBox, &tmQ, fq, h * HD + 64, row0 + q0);
      tma_load_2d_pair(sG, &tmG, fq, h * HD, row0 + q0);
      tma_load_2d_pair(sG + kBox, &tmG, fq, h * HD + 64, row0 + q0);
      for (int j = 0; j < nk; ++j) {
        const int st = j % kKSlots;
        mbar_wait(&k_empty[st], ((j / kKSlots) & 1) ^ 1);
        BWD_TRACE(16, j);
        const uint32_t fk = leader_addr(&k_full[st]);
        if (leader) mbar_expect_tx(&k_full[st], 2 * (2 * kBoxH + kBox));
        const int krow = row0 + j * BT;
        tma_load_2d_pair(sKs + st * 2 * kBoxH, &tmK64, fk, kvh * HD, krow + (int)rank * 64);
        tma_load_2d_pair(sKs + st * 2 * kBoxH + kBoxH, &tmK64, fk, kvh * HD + 64, krow + (int)rank * 64);
        tma_load_2d_pair(sKq + st * kBox, &tmK, fk, kvh * HD + (int)rank * 64, krow);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // producer B (both CTAs): its 64 keys of V_j
    if (elect_one()) {
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        BWD_TRACE(17, j);
        const uint32_t fv = leader_addr(&v_full[st]);
        if (leader) mbar_expect_tx(&v_full[st], 2 * 2 * kBoxH);
        const int krow = row0 + j * BT + (int)rank * 64;
        tma_load_2d_pair(sV + st * 2 * kBoxH, &tmV64, fv, kvh * HD, krow);
        tma_load_2d_pair(sV + st * 2 * kBoxH + kBoxH, &tmV64, fv, kvh * HD + 64, krow);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      const uint32_t id_s = idesc_bf16_f32(256, 128, 0, 0);
      const uint32_t id_acc = idesc_bf16_f32(256, 128, 0, 1);
      const uint64_t dQd = sw128_desc(smem_u32(sQ), 16, 1024), dGd = sw128_desc(smem_u32(sG), 16, 1024);
      auto issue_s = [&](int j) {
        const int ks = j % kKSlots;
        BWD_TRACE(18, j);
        mbar_wait(&k_full[ks], (j / kKSlots) & 1);
        tc_fence_after();
        BWD_TRACE(10, j);
        const uint64_t dKj = sw128_desc(smem_u32(sKs + ks * 2 * kBoxH), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            umma_f16_ss_pair(tmem + (j & 1) * 128u, dQd + koff(kk), dKj + koff64(kk), id_s, kk > 0);
          umma_commit_pair_mc(&s_full[j & 1], 0x3);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int j) {
        mbar_wait(&v_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        BWD_TRACE(12, j);
        const uint64_t dVj = sw128_desc(smem_u32(sV + (j & 1) * 2 * kBoxH), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            umma_f16_ss_pair(tmem + cP, dGd + koff(kk), dVj + koff64(kk), id_s, kk > 0);
          umma_commit_pair_mc(dp_full, 0x3);
          umma_commit_pair_mc(&v_empty[j & 1], 0x3);
        }
        __syncwarp();
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        if (j + 1 < nk) issue_s(j + 1);
        // dP(j+1) as soon as both CTAs' compute warps hold dP(j) in registers (the cross-SM
        // signal latency then overlaps tile j's dS pass instead of following it)
        if (j + 1 < nk) {
          mbar_wait(dp_free, j & 1);
          tc_fence_after();
          issue_dp(j + 1);
        }
        // B: K_j's 128 keys x this CTA's 64 head dims, MN-major (one 64-column atom)
        const uint64_t mK = sw128_desc(smem_u32(sKq + (j % kKSlots) * kBox), kBox, 1024);
        mbar_wait(&ds_part[j & 1], (j >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)
            if ((k & 3) < 2)
              umma_f16_ts_pair(tmem + cQ, tmem + st * 128u + packed_col(k), mK + (uint64_t)(k * 128), id_acc,
                               (j | k) != 0);
        }
        __syncwarp();
        mbar_wait(&ds_ready[j & 1], (j >> 1) & 1);
        tc_fence_after();
        BWD_TRACE(11, j);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)
            if ((k & 3) >= 2)
              umma_f16_ts_pair(tmem + cQ, tmem + st * 128u + packed_col(k), mK + (uint64_t)(k * 128), id_acc, 1);
          umma_commit_pair_mc(&k_empty[j % kKSlots], 0x3);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit_pair_mc(mma_done, 0x3);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int ch = (warp - 4) >> 2;  // key-column half of each tile
    const int t = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float c = p.scale * kLog2e;
    const int qrow = q0 + t;
    const int64_t li = ((int64_t)b * p.H + h) * p.T + qrow;
    const float L = p.lse[li] * kLog2e;
    const float D = p.delta[li];
    const float2 c2 = make_float2(c, c), nl2 = make_float2(-L, -L), nd2 = make_float2(-D, -D);
    const uint32_t ds_part_l[2] = {leader_addr(&ds_part[0]), leader_addr(&ds_part[1])};
    const uint32_t ds_ready_l[2] = {leader_addr(&ds_ready[0]), leader_addr(&ds_ready[1])};
    const uint32_t dp_free_l = leader_addr(dp_free);
    for (int j = 0; j < nk; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(13, j);
      float2 pr[32];
      {
        uint32_t sv[2][32];
        ld64(tmem + lo + st * 128u + ch * 64, sv);
#pragma unroll
        for (int i = 0; i < 32; ++i) pr[i] = exp2_pair(ffma2(col2(sv, i), c2, nl2), i);
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      if (warp == 4) BWD_TRACE(14, j);
      {
        uint32_t dv[2][32];
        ld64(tmem + lo + cP + ch * 64, dv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(dp_free_l);
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 d = fmul2(pr[16 * part + i], fadd2(col2(dv, 16 * part + i), nd2));
            pk[i] = pack2(d.x, d.y);
          }
          tmem_st16(tmem + lo + st * 128u + ch * 64 + 16 * part, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (part == 0 && lane == 0) mbar_arrive_cluster_relaxed(ds_part_l[st]);
        }
      }
      if (warp == 4) BWD_TRACE(15, j);
      if (lane == 0) mbar_arrive_cluster_relaxed(ds_ready_l[st]);
    }
    mbar_wait(mma_done, 0);
    tc_fence_after();
    const float* rc = p.rope_cos ? p.rope_cos + (int64_t)qrow * (HD / 2) + ch * 32 : nullptr;
    const float* rs = p.rope_sin ? p.rope_sin + (int64_t)qrow * (HD / 2) + ch * 32 : nullptr;
    store_row(tmem + lo + cQ + ch * 64, p.o0 + ((int64_t)row0 + qrow) * p.ld0 + (int64_t)h * HD + ch * 64, p.scale,
              true, rc, rs, 2);
  }
  tc_fence_before();
  cluster_sync();
  CTA_TRACE(1, 1);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, kCols);
  }
}

// ============================================================ dQ as a GEMM over stored dS
// dQ[q, :] = scale * sum_key dS[q, key] K[key, :] for one (128-query tile, head, batch) per
// CTA, reading the dS^T the DS variant of dkdv_k stored (row (b*H + h)*T + key, column query:
// an MN-major A operand) and K (MN-major B), 64 keys per stage through a 6-deep TMA ring;
// tcgen05 accumulator in TMEM; inverse RoPE + bf16 store in the epilogue.  Deterministic
// (one CTA per dQ tile, keys in order).  Requires T % 128 == 0.
constexpr int kGStages = 6;
constexpr int kGThreads = 256;
constexpr int kSmemDqGemm = kGStages * 2 * kBox + 1024 + 256;

__global__ void __launch_bounds__(kGThreads, 1)
    dq_gemm_k(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmK, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                    // [kGStages] dS^T box pairs: 64 keys x 128 queries
  uint8_t* sB = smem + kGStages * kBox;  // [kGStages] K box pairs: 64 keys x 128 head dims
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGStages * 2 * kBox);
  uint64_t* empty = full + kGStages;
  uint64_t* done = empty + kGStages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.KVH);
  const int q0 = qt * BT, nkb = p.T / 64;
  const int srow = (b * p.H + h) * p.T, krow = b * p.T;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmS);
    tma_prefetch_desc(&tmK);
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % kGStages;
        mbar_wait(&empty[st], ((kb / kGStages) & 1) ^ 1);
        mbar_expect_tx(&full[st], 4 * (kBox / 2));
        uint8_t* a = sA + st * kBox;
        uint8_t* bb = sB + st * kBox;
        // [64 keys][64 cols] boxes: two query halves of dS^T, two head-dim halves of K
        tma_load_2d(a, &tmS, &full[st], q0, srow + kb * 64);
        tma_load_2d(a + kBox / 2, &tmS, &full[st], q0 + 64, srow + kb * 64);
        tma_load_2d(bb, &tmK, &full[st], kvh * HD, krow + kb * 64);
        tma_load_2d(bb + kBox / 2, &tmK, &full[st], kvh * HD + 64, krow + kb * 64);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, 1, 1);  // MN-major A and B
    for (int kb = 0; kb < nkb; ++kb) {
      const int st = kb % kGStages;
      mbar_wait(&full[st], (kb / kGStages) & 1);
      tc_fence_after();
      const uint64_t ad = sw128_desc(smem_u32(sA + st * kBox), kBox / 2, 1024);
      const uint64_t bd = sw128_desc(smem_u32(sB + st * kBox), kBox / 2, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // K = 16 keys per MMA: +2048 bytes of the MN-major boxes
          umma_f16_ss(tmem, ad + (uint64_t)(kk * 128), bd + (uint64_t)(kk * 128), idesc, (kb | kk) != 0);
        umma_commit(&empty[st]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  } else if (warp >= 4) {
    const int qd = warp & 3;
    const int qrow = q0 + qd * 32 + lane;
    mbar_wait(done, 0);
    tc_fence_after();
    const float* rc = p.rope_cos ? p.rope_cos + (int64_t)qrow * (HD / 2) : nullptr;
    const float* rs = p.rope_sin ? p.rope_sin + (int64_t)qrow * (HD / 2) : nullptr;
    store_row(tmem + ((uint32_t)(qd * 32) << 16), p.o0 + ((int64_t)krow + qrow) * p.ld0 + (int64_t)h * HD, p.scale,
              qrow < p.T, rc, rs, HD / 32);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

}  // namespace tcb

int attn_bwd_tc(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, int64_t lddo,
                const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                int64_t lddv, cudaStream_t st, const float* rope_cos, const float* rope_sin, void* ds_ws) {
  using namespace tcb;
  if ((lddo | lddq | lddk | lddv) & 7) return fail(CB_ERR_ARG, "tc attention bwd: strides must be 16-byte aligned");
  CUtensorMap mq, mk, mv, mg, ms, mk64;
  const uint64_t rows = (uint64_t)g.B * g.T;
  int s;
  if ((s = make_tmap_2d_bf16(&mq, q, rows, (uint64_t)g.H * HD, g.ldq, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mk, k, rows, (uint64_t)g.KVH * HD, g.ldk, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mv, v, rows, (uint64_t)g.KVH * HD, g.ldv, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mg, dout, rows, (uint64_t)g.H * HD, lddo, 128, 64))) return s;
  // dS path (a caller-provided dS^T workspace, T a multiple of 128): dK/dV sweep storing dS^T,
  // then dQ as a GEMM over it instead of the dQ sweep's S / dP recomputation
  const bool use_ds = ds_ws != nullptr && g.T % 128 == 0;
  if (use_ds) {
    if ((s = make_tmap_2d_bf16(&ms, ds_ws, (uint64_t)g.B * g.H * g.T, (uint64_t)g.T, (uint64_t)g.T, 32, 64))) return s;
    CUtensorMap ms64;
    if ((s = make_tmap_2d_bf16(&ms64, ds_ws, (uint64_t)g.B * g.H * g.T, (uint64_t)g.T, (uint64_t)g.T, 64, 64)))
      return s;
    if ((s = make_tmap_2d_bf16(&mk64, k, rows, (uint64_t)g.KVH * HD, g.ldk, 64, 64))) return s;
    static bool attr_ds = false;
    if (!attr_ds) {
      cudaFuncSetAttribute(dkdv_k<kDkdvGroups, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDkdv);
      cudaFuncSetAttribute(dq_gemm_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDqGemm);
      attr_ds = true;
    }
    Params pk{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dk, lddk, (__nv_bfloat16*)dv, lddv,
              rope_cos, rope_sin};
    dkdv_k<kDkdvGroups, true><<<dim3(g.T / BT, g.KVH, g.B), 128 + 128 * kDkdvGroups, kSmemDkdv, st>>>(mq, mk, mv,
                                                                                                   mg, ms, pk);
    if (int e = check_launch("flash_bwd_dkdv_ds_tc")) return e;
    Params pq{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dq, lddq, nullptr, 0, rope_cos, rope_sin};
    dq_gemm_k<<<dim3(g.T / BT, g.H, g.B), kGThreads, kSmemDqGemm, st>>>(ms64, mk64, pq);
    return check_launch("flash_bwd_dq_gemm_tc");
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dkdv_k<kDkdvGroups, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDkdv);
    cudaFuncSetAttribute(dkdv_pair_k<kDkdvGroups>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDkdv);
    cudaFuncSetAttribute(dq_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDq);
    attr = true;
  }
  Params pk{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dk, lddk, (__nv_bfloat16*)dv, lddv,
            rope_cos, rope_sin};
  if (g_dkdv_pair && g.T % (2 * BT) == 0) {
    CUtensorMap mq64, mg64;
    if ((s = make_tmap_2d_bf16(&mq64, q, rows, (uint64_t)g.H * HD, g.ldq, 64, 64))) return s;
    if ((s = make_tmap_2d_bf16(&mg64, dout, rows, (uint64_t)g.H * HD, lddo, 64, 64))) return s;
    dkdv_pair_k<kDkdvGroups><<<dim3(g.T / BT, g.KVH, g.B), 128 + 128 * kDkdvGroups, kSmemDkdv, st>>>(
        mq, mq64, mk, mv, mg, mg64, pk);
    if (int e = check_launch("flash_bwd_dkdv_pair_tc")) return e;
  } else {
    dkdv_k<kDkdvGroups, false><<<dim3((g.T + BT - 1) / BT, g.KVH, g.B), 128 + 128 * kDkdvGroups, kSmemDkdv, st>>>(
        mq, mk, mv, mg, mg, pk);
    if (int e = check_launch("flash_bwd_dkdv_tc")) return e;
  }
  Params pq{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dq, lddq, nullptr, 0, rope_cos, rope_sin};
  if (g_dq_pair && g.T % (2 * BT) == 0) {
    CUtensorMap mk64p, mv64;
    if ((s = make_tmap_2d_bf16(&mk64p, k, rows, (uint64_t)g.KVH * HD, g.ldk, 64, 64))) return s;
    if ((s = make_tmap_2d_bf16(&mv64, v, rows, (uint64_t)g.KVH * HD, g.ldv, 64, 64))) return s;
    static bool attr_pair = false;
    if (!attr_pair) {
      cudaFuncSetAttribute(dq_pair_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDqPair);
      attr_pair = true;
    }
    dq_pair_k<<<dim3(g.T / BT, g.H, g.B), kThreads, kSmemDqPair, st>>>(mq, mk, mk64p, mv64, mg, pq);
    return check_launch("flash_bwd_dq_pair_tc");
  }
  dq_k<<<dim3((g.T + BT - 1) / BT, g.H, g.B), kThreads, kSmemDq, st>>>(mq, mk, mv, mg, pq);
  return check_launch("flash_bwd_dq_tc");
}

}  // namespace cb
