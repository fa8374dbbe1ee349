// tcgen05 flash attention backward (bf16, head_dim 128), unmasked, GQA-aware.
//
// Deterministic two-kernel split (no atomics), both recomputing P = exp(S - LSE):
//   dkdv: one CTA per (128-key tile, kv head, batch); sweeps every 128-query tile of every
//         query head in the kv group:
//           S^T  = K Q^T          (A = K   smem K-major, B = Q  smem K-major)  -> TMEM
//           dP^T = V dO^T         (A = V   smem K-major, B = dO smem K-major)  -> TMEM
//           P^T  = exp2(S^T c - lse2), dS^T = P^T (dP^T - delta)   [1 thread = 1 key row]
//           dV  += P^T dO         (A = P^T from TMEM, B = dO smem MN-major)
//           dK  += dS^T Q         (A = dS^T from TMEM, B = Q  smem MN-major)
//   dq:   one CTA per (128-query tile, head, batch); sweeps every 128-key tile:
//           S = Q K^T, dP = dO V^T, dS = P (dP - delta), dQ += dS K (B = K MN-major)
// TMEM (512 columns): dkdv = S^T | dP^T | dV | dK;  dq = S | dP | dQ.
// Warp roles as in the forward: 0 TMA, 1 MMA (single thread), 2 TMEM alloc, 4-7 compute.
#include "attn.cuh"
#include "composer_b200.h"

namespace cb {
namespace tcb {

constexpr int HD = 128;
constexpr int BT = 128;  // tile rows (keys or queries)
constexpr int kThreads = 256;
constexpr int kBox = 128 * 64 * 2;    // one [128][64] bf16 TMA box (16 KB)
constexpr int kTile = 2 * kBox;       // one [128][128] tile (two 64-column atoms)
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
};

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// K-major operand descriptor of a [128][128] tile for the kk-th K=16 step
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  return sw128_desc(base + (kk >> 2) * kBox + (kk & 3) * 32, 16, 1024);
}
// MN-major operand descriptor (rows = K dim, 128 columns = N) for the k-th K=16 step
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k) { return sw128_desc(base + k * 2048, kBox, 1024); }

// store one thread's 128-column f32 TMEM row as bf16 (times `mul`) to global
__device__ __forceinline__ void store_row(uint32_t taddr, __nv_bfloat16* dst, float mul, bool ok) {
#pragma unroll 1
  for (int cc = 0; cc < HD / 32; ++cc) {
    uint32_t o[32];
    tmem_ld32(taddr + cc * 32, o);
    tmem_ld_wait();
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

// ====================================================================== dK / dV
__global__ void __launch_bounds__(kThreads, 1)
    dkdv_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* ring = smem + 2 * kTile;  // [2] x {Q tile, dO tile}
  float* sL = reinterpret_cast<float*>(smem + 6 * kTile);  // [2][128] lse * log2e
  float* sD = sL + 256;                                   // [2][128] delta
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
  const int total = group * nq;
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
    mbar_init(p_ready, 4);
    mbar_init(ds_ready, 4);
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
      const uint32_t id_s = idesc_bf16_f32(128, 128, 0, 0);   // K-major x K-major
      const uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1); // TMEM A x MN-major B
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < total; ++it) {
        const int st = it & 1;
        const uint32_t aQ = smem_u32(ring + st * 2 * kTile), aG = aQ + kTile;
        mbar_wait(&qd_full[st], (it >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cS, kdesc(aK, kk), kdesc(aQ, kk), id_s, kk > 0);
        umma_commit(s_full);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, kdesc(aV, kk), kdesc(aG, kk), id_s, kk > 0);
        umma_commit(dp_full);
        mbar_wait(p_ready, it & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BT / 16; ++k) umma_f16_ts(tmem + cV, tmem + cS + k * 8, mndesc(aG, k), id_acc, (it | k) != 0);
        mbar_wait(ds_ready, it & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BT / 16; ++k) umma_f16_ts(tmem + cK, tmem + cP + k * 8, mndesc(aQ, k), id_acc, (it | k) != 0);
        umma_commit(&qd_empty[st]);
        umma_commit(mma_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int t = threadIdx.x - 128;  // 0..127: key row inside the tile
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float c = p.scale * kLog2e;
    for (int it = 0; it < total; ++it) {
      const int h = kvh * group + it / nq, q0 = (it % nq) * BT;
      float* L = sL + (it & 1) * 128;
      float* D = sD + (it & 1) * 128;
      {
        const int qi = q0 + t;
        const int64_t li = ((int64_t)b * p.H + h) * p.T + qi;
        L[t] = qi < p.T ? p.lse[li] * kLog2e : 0.f;
        D[t] = qi < p.T ? p.delta[li] : 0.f;
      }
      named_sync(1, 128);
      const int valid = min(BT, p.T - q0);
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      float pr[128];
      {
        uint32_t v[32];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          tmem_ld32(tmem + lo + cS + cc * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = cc * 32 + i;
            pr[col] = col < valid ? exp2f(__uint_as_float(v[i]) * c - L[col]) : 0.f;
          }
        }
        uint32_t pk[32];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = pack2(pr[hh * 64 + 2 * i], pr[hh * 64 + 2 * i + 1]);
          tmem_st32(tmem + lo + cS + hh * 32, pk);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      {
        uint32_t v[32];
        uint32_t pk[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          tmem_ld32(tmem + lo + cP + cc * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = cc * 32 + 2 * i;
            const float d0 = pr[col] * (__uint_as_float(v[2 * i]) - D[col]);
            const float d1 = pr[col + 1] * (__uint_as_float(v[2 * i + 1]) - D[col + 1]);
            pk[i] = pack2(d0, d1);
          }
          // dS^T chunk cc covers keys' columns [32cc, 32cc+32) -> packed columns [16cc, 16cc+16)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
              "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tmem + lo + cP + cc * 16),
              "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]),
              "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15])
              : "memory");
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
    }
    mbar_wait(mma_done, (total - 1) & 1);
    tc_fence_after();
    const int krow = k0 + t;
    const bool ok = krow < p.T;
    store_row(tmem + lo + cK, p.o0 + ((int64_t)row0 + krow) * p.ld0 + (int64_t)kvh * HD, p.scale, ok);
    store_row(tmem + lo + cV, p.o1 + ((int64_t)row0 + krow) * p.ld1 + (int64_t)kvh * HD, 1.f, ok);
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
  uint64_t* s_full = bars + 5;
  uint64_t* dp_full = bars + 6;
  uint64_t* ds_ready = bars + 7;
  uint64_t* mma_done = bars + 8;
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
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 4);
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t cS = 0, cP = 128, cQ = 256;

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
      mbar_wait(q_full, 0);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        const uint32_t aK = smem_u32(ring + st * 2 * kTile), aV = aK + kTile;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cS, kdesc(aQ, kk), kdesc(aK, kk), id_s, kk > 0);
        umma_commit(s_full);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) umma_f16_ss(tmem + cP, kdesc(aG, kk), kdesc(aV, kk), id_s, kk > 0);
        umma_commit(dp_full);
        mbar_wait(ds_ready, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < BT / 16; ++k) umma_f16_ts(tmem + cQ, tmem + cS + k * 8, mndesc(aK, k), id_acc, (j | k) != 0);
        umma_commit(&kv_empty[st]);
        umma_commit(mma_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int t = threadIdx.x - 128;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float c = p.scale * kLog2e;
    const int qrow = q0 + t;
    const bool ok = qrow < p.T;
    const int64_t li = ((int64_t)b * p.H + h) * p.T + qrow;
    const float L = ok ? p.lse[li] * kLog2e : 0.f;
    const float D = ok ? p.delta[li] : 0.f;
    for (int j = 0; j < nk; ++j) {
      const int valid = min(BT, p.T - j * BT);
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      float pr[128];
      {
        uint32_t v[32];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          tmem_ld32(tmem + lo + cS + cc * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = cc * 32 + i;
            pr[col] = col < valid ? exp2f(__uint_as_float(v[i]) * c - L) : 0.f;
          }
        }
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      {
        uint32_t v[32];
        uint32_t pk[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          tmem_ld32(tmem + lo + cP + cc * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = cc * 32 + 2 * i;
            pk[i] = pack2(pr[col] * (__uint_as_float(v[2 * i]) - D), pr[col + 1] * (__uint_as_float(v[2 * i + 1]) - D));
          }
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
              "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tmem + lo + cS + cc * 16),
              "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]),
              "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15])
              : "memory");
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
    }
    mbar_wait(mma_done, (nk - 1) & 1);
    tc_fence_after();
    store_row(tmem + lo + cQ, p.o0 + ((int64_t)row0 + qrow) * p.ld0 + (int64_t)h * HD, p.scale, ok);
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
                int64_t lddv, cudaStream_t st) {
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
  Params pk{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dk, lddk, (__nv_bfloat16*)dv, lddv};
  dkdv_k<<<dim3((g.T + BT - 1) / BT, g.KVH, g.B), kThreads, kSmem, st>>>(mq, mk, mv, mg, pk);
  if (int e = check_launch("flash_bwd_dkdv_tc")) return e;
  Params pq{g.T, g.H, g.KVH, g.B, g.scale, lse, delta, (__nv_bfloat16*)dq, lddq, nullptr, 0};
  dq_k<<<dim3((g.T + BT - 1) / BT, g.H, g.B), kThreads, kSmem, st>>>(mq, mk, mv, mg, pq);
  return check_launch("flash_bwd_dq_tc");
}

}  // namespace cb
