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
//         MMA issue order  dV(u) S(u+1) | dK(u) dP(u+1)  lets the exp pass of tile u+1
//         overlap dK(u)/dP(u+1) and the dS pass overlap dV(u+1)/S(u+2) with single-buffered
//         TMEM (S^T | dP^T | dV | dK = 512 columns).
//   dq:   one CTA per (128-query tile, head, batch); sweeps every 128-key tile j:
//           S_j = Q K_j^T (double-buffered), dP_j = dO V_j^T, dS = P (dP - delta),
//           dQ += dS K_j (B = K_j MN-major); S_{j+1} is issued before dQ_j.
//           TMEM: S[2] | dP | dQ.
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
constexpr int kSmem = 6 * kTile + 1024 + 4096;
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

// K-major operand descriptor for the kk-th K=16 step of a tile whose rows start at `base`
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  return sw128_desc(base + (kk >> 2) * kBox + (kk & 3) * 32, 16, 1024);
}
// MN-major operand descriptor (rows = K dim, 128 columns = N) for the k-th K=16 step
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k) { return sw128_desc(base + k * 2048, kBox, 1024); }

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

// Packs 64 f32 values (two 32-column TMEM loads at src) through `f` into 32 bf16 pairs.
template <typename F>
__device__ __forceinline__ void load64(uint32_t src, float (&out)[64], F f) {
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    uint32_t v[32];
    tmem_ld32(src + cc * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) out[cc * 32 + i] = f(cc * 32 + i, __uint_as_float(v[i]));
  }
}

// ====================================================================== dK / dV
__global__ void __launch_bounds__(kThreads, 1)
    dkdv_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* ring = smem + 2 * kTile;                        // [2] x {Q tile, dO tile}
  float* sL = reinterpret_cast<float*>(smem + 6 * kTile);  // [2][128] lse * log2e
  float* sD = sL + 256;                                    // [2][128] delta
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 256);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;   // [2]
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* dp_full = bars + 6;
  uint64_t* p_ready = bars + 7;
  uint64_t* ds_ready = bars + 8;
  uint64_t* mma_done = bars + 9;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 10);

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
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&qd_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, 8);
    mbar_init(ds_ready, 8);
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
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * kTile);
      tma_load_2d(sK, &tmK, kv_full, kvh * HD, row0 + k0);
      tma_load_2d(sK + kBox, &tmK, kv_full, kvh * HD + 64, row0 + k0);
      tma_load_2d(sV, &tmV, kv_full, kvh * HD, row0 + k0);
      tma_load_2d(sV + kBox, &tmV, kv_full, kvh * HD + 64, row0 + k0);
      for (int it = 0; it < total; ++it) {
        const int st = it & 1;
        const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
        mbar_wait(&qd_empty[st], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&qd_full[st], 2 * kTile);
        uint8_t* base = ring + st * 2 * kTile;
        tma_load_2d(base, &tmQ, &qd_full[st], h * HD, row0 + q0);
        tma_load_2d(base + kBox, &tmQ, &qd_full[st], h * HD + 64, row0 + q0);
        tma_load_2d(base + kTile, &tmG, &qd_full[st], h * HD, row0 + q0);
        tma_load_2d(base + kTile + kBox, &tmG, &qd_full[st], h * HD + 64, row0 + q0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);    // K-major x K-major
      const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);  // TMEM A x MN-major B
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
      auto tileQ = [&](int u) { return smem_u32(ring + (u & 1) * 2 * kTile); };
      auto issue_s = [&](int u) {
        mbar_wait(&qd_full[u & 1], (u >> 1) & 1);
        tc_fence_after();
        const uint32_t aQ = tileQ(u);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cS, kdesc(aK, kk), kdesc(aQ, kk), id_s, kk > 0);
        umma_commit(s_full);
      };
      auto issue_dp = [&](int u) {
        const uint32_t aG = tileQ(u) + kTile;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, kdesc(aV, kk), kdesc(aG, kk), id_s, kk > 0);
        umma_commit(dp_full);
      };
      mbar_wait(kv_full, 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int u = 0; u < total; ++u) {
        const uint32_t aQ = tileQ(u), aG = aQ + kTile;
        mbar_wait(p_ready, u & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BT / 16; ++k) umma_f16_ts(tmem + cV, tmem + cS + k * 8, mndesc(aG, k), id_acc, (u | k) != 0);
        if (u + 1 < total) issue_s(u + 1);  // S^T region: P^T(u) already consumed (in-order)
        mbar_wait(ds_ready, u & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BT / 16; ++k) umma_f16_ts(tmem + cK, tmem + cP + k * 8, mndesc(aQ, k), id_acc, (u | k) != 0);
        umma_commit(&qd_empty[u & 1]);
        if (u + 1 < total) issue_dp(u + 1);  // dP^T region: dS^T(u) already consumed
      }
      umma_commit(mma_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int ch = (warp - 4) >> 2;    // query-column half of each tile
    const int t = q * 32 + lane;       // key row inside the tile
    const int tt = threadIdx.x - 128;  // 0..255
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float c = p.scale * kLog2e;
    for (int u = 0; u < total; ++u) {
      const int h = kvh * group + u / nq, q0 = (u % nq) * BT;
      if (tt < 128) {
        const int qi = q0 + tt;
        const int64_t li = ((int64_t)b * p.H + h) * p.T + qi;
        sL[(u & 1) * 128 + tt] = qi < p.T ? p.lse[li] * kLog2e : 0.f;
        sD[(u & 1) * 128 + tt] = qi < p.T ? p.delta[li] : 0.f;
      }
      named_sync(1, 256);
      const float* L = sL + (u & 1) * 128 + ch * 64;
      const float* D = sD + (u & 1) * 128 + ch * 64;
      const int valid = min(BT, p.T - q0) - ch * 64;
      mbar_wait(s_full, u & 1);
      tc_fence_after();
      float pr[64];
      if (valid >= 64)
        load64(tmem + lo + cS + ch * 64, pr, [&](int i, float s) { return fast_exp2(fmaf(s, c, -L[i])); });
      else
        load64(tmem + lo + cS + ch * 64, pr,
               [&](int i, float s) { return i < valid ? fast_exp2(fmaf(s, c, -L[i])) : 0.f; });
      {
        uint32_t pk[2][16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          pk[0][i] = pack2(pr[2 * i], pr[2 * i + 1]);
          pk[1][i] = pack2(pr[32 + 2 * i], pr[33 + 2 * i]);
        }
        named_sync(2 + q, 64);  // the partner warp has read its raw S^T columns
        tmem_st16(tmem + lo + cS + ch * 32, pk[0]);
        tmem_st16(tmem + lo + cS + ch * 32 + 16, pk[1]);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      mbar_wait(dp_full, u & 1);
      tc_fence_after();
      {
        float ds[64];
        load64(tmem + lo + cP + ch * 64, ds, [&](int i, float dp) { return pr[i] * (dp - D[i]); });
        uint32_t pk[2][16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          pk[0][i] = pack2(ds[2 * i], ds[2 * i + 1]);
          pk[1][i] = pack2(ds[32 + 2 * i], ds[33 + 2 * i]);
        }
        named_sync(2 + q, 64);
        tmem_st16(tmem + lo + cP + ch * 32, pk[0]);
        tmem_st16(tmem + lo + cP + ch * 32 + 16, pk[1]);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
    }
    mbar_wait(mma_done, 0);
    tc_fence_after();
    const int krow = k0 + t;
    const bool ok = krow < p.T;
    if (ch == 0) {
      const float* rc = p.rope_cos ? p.rope_cos + (int64_t)(ok ? krow : 0) * (HD / 2) : nullptr;
      const float* rs = p.rope_sin ? p.rope_sin + (int64_t)(ok ? krow : 0) * (HD / 2) : nullptr;
      store_row(tmem + lo + cK, p.o0 + ((int64_t)row0 + krow) * p.ld0 + (int64_t)kvh * HD, p.scale, ok, rc, rs, 4);
    } else {
      store_row(tmem + lo + cV, p.o1 + ((int64_t)row0 + krow) * p.ld1 + (int64_t)kvh * HD, 1.f, ok, nullptr,
                nullptr, 4);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// =========================================================================== dQ
__global__ void __launch_bounds__(kThreads, 1)
    dq_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sG = smem + kTile;
  uint8_t* ring = smem + 2 * kTile;  // [2] x {K tile, V tile}
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTile + 2048);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* dp_full = bars + 7;
  uint64_t* ds_ready = bars + 8;
  uint64_t* mma_done = bars + 9;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 10);

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
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 8);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cP = 256, cQ = 384;  // S buffers at st * 128

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kTile);
      tma_load_2d(sQ, &tmQ, q_full, h * HD, row0 + q0);
      tma_load_2d(sQ + kBox, &tmQ, q_full, h * HD + 64, row0 + q0);
      tma_load_2d(sG, &tmG, q_full, h * HD, row0 + q0);
      tma_load_2d(sG + kBox, &tmG, q_full, h * HD + 64, row0 + q0);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * kTile);
        uint8_t* base = ring + st * 2 * kTile;
        const int kr = row0 + j * BT;
        tma_load_2d(base, &tmK, &kv_full[st], kvh * HD, kr);
        tma_load_2d(base + kBox, &tmK, &kv_full[st], kvh * HD + 64, kr);
        tma_load_2d(base + kTile, &tmV, &kv_full[st], kvh * HD, kr);
        tma_load_2d(base + kTile + kBox, &tmV, &kv_full[st], kvh * HD + 64, kr);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);
      const uint32_t aQ = smem_u32(sQ), aG = smem_u32(sG);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t aK = smem_u32(ring + st * 2 * kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + st * 128u, kdesc(aQ, kk), kdesc(aK, kk), id_s, kk > 0);
        umma_commit(&s_full[st]);
      };
      auto issue_dp = [&](int j) {
        const uint32_t aV = smem_u32(ring + (j & 1) * 2 * kTile) + kTile;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, kdesc(aG, kk), kdesc(aV, kk), id_s, kk > 0);
        umma_commit(dp_full);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        if (j + 1 < nk) issue_s(j + 1);
        mbar_wait(ds_ready, j & 1);
        tc_fence_after();
        const uint32_t aK = smem_u32(ring + st * 2 * kTile);
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)
          umma_f16_ts(tmem + cQ, tmem + st * 128u + k * 8, mndesc(aK, k), id_acc, (j | k) != 0);
        umma_commit(&kv_empty[st]);
        if (j + 1 < nk) issue_dp(j + 1);
      }
      umma_commit(mma_done);
    }
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
    for (int j = 0; j < nk; ++j) {
      const int st = j & 1;
      const int valid = min(BT, p.T - j * BT) - ch * 64;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float pr[64];
      if (valid >= 64)
        load64(tmem + lo + st * 128u + ch * 64, pr, [&](int, float s) { return fast_exp2(fmaf(s, c, -L)); });
      else
        load64(tmem + lo + st * 128u + ch * 64, pr,
               [&](int i, float s) { return i < valid ? fast_exp2(fmaf(s, c, -L)) : 0.f; });
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      {
        float ds[64];
        load64(tmem + lo + cP + ch * 64, ds, [&](int i, float dp) { return pr[i] * (dp - D); });
        uint32_t pk[2][16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          pk[0][i] = pack2(ds[2 * i], ds[2 * i + 1]);
          pk[1][i] = pack2(ds[32 + 2 * i], ds[33 + 2 * i]);
        }
        named_sync(2 + q, 64);  // both halves have read their raw S columns
        tmem_st16(tmem + lo + st * 128u + ch * 32, pk[0]);
        tmem_st16(tmem + lo + st * 128u + ch * 32 + 16, pk[1]);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
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
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

}  // namespace tcb

int attn_bwd_tc(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, int64_t lddo,
                const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                int64_t lddv, cudaStream_t st, const float* rope_cos, const float* rope_sin) {
  using namespace tcb;
  if ((lddo | lddq | lddk | lddv) & 7) return fail(CB_ERR_ARG, "tc attention bwd: strides must be 16-byte aligned");
  CUtensorMap mq, mk, mv, mg;
  const uint64_t rows = (uint64_t)g.B * g.T;
  int s;
  if ((s = make_tmap_2d_bf16(&mq, q, rows, (uint64_t)g.H * HD, g.ldq, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mk, k, rows, (uint64_t)g.KVH * HD, g.ldk, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mv, v, rows, (uint64_t)g.KVH * HD, g.ldv, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mg, dout, rows, (uint64_t)g.H * HD, lddo, 128, 64))) return s;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dkdv_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(dq_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  Params pk{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dk, lddk, (__nv_bfloat16*)dv, lddv,
            rope_cos, rope_sin};
  dkdv_k<<<dim3((g.T + BT - 1) / BT, g.KVH, g.B), kThreads, kSmem, st>>>(mq, mk, mv, mg, pk);
  if (int e = check_launch("flash_bwd_dkdv_tc")) return e;
  Params pq{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dq, lddq, nullptr, 0, rope_cos, rope_sin};
  dq_k<<<dim3((g.T + BT - 1) / BT, g.H, g.B), kThreads, kSmem, st>>>(mq, mk, mv, mg, pq);
  return check_launch("flash_bwd_dq_tc");
}

}  // namespace cb
