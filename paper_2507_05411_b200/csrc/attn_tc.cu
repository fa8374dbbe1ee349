// tcgen05 flash attention forward (bf16, head_dim 128), unmasked, GQA-aware.
//
// Reference op: AttentionBehavior.forward (reference layers.py:331-348): softmax over
// all keys (no causal mask) of q k^T / sqrt(hd), then @ v.
//
// One CTA per (256-query block, head, batch) = two 128-row query tiles A and B that share
// every K/V tile (half the K/V shared-memory traffic per FLOP).  384 threads:
//   warp 0       TMA producer: Q_A, Q_B once, then K_j into a 3-slot ring (a slot frees
//                as soon as S_B(j) has read it); warp 3 streams V_j into a 2-slot ring
//   warp 1       MMA issuer (one thread), ping-pong between the tiles so the tensor core
//                always has work while one softmax group runs:
//                  S_A(j) S_B(j) | PV_A(j) S_A(j+1) | PV_B(j) S_B(j+1) | ...
//                S = Q K^T lands in TMEM; P (bf16) is written back over S and consumed as
//                the TMEM A operand of O += P V (V is an MN-major smem operand)
//   warp 2       TMEM allocator (512 columns: S_A | S_B | O_A | O_B)
//   warps 4-7    softmax of tile A, warps 8-11 softmax of tile B: one thread owns one
//                query row (no shuffles), exp2 domain, lazy O rescale (only when the row
//                max grows by more than 2^8), then the epilogue (O / l, natural-log LSE).
#include <type_traits>

#include "attn.cuh"
#include "composer_b200.h"

namespace cb {
namespace tca {

// Optional per-iteration clock64 trace of CTA (0,0,0) for pipeline analysis
// (scripts/attn_trace.cu builds this file with CB_ATTN_TRACE; the library never does).
#ifdef CB_ATTN_TRACE
__device__ unsigned long long g_trace[16][64];
#define ATTN_TRACE(ev, j) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64 && (threadIdx.x & 31) == 0) g_trace[ev][j] = clock64()
#else
#define ATTN_TRACE(ev, j)
#endif

constexpr int HD = 128;
constexpr int BM = 128, BN = 128;
constexpr int kThreads = 384;
constexpr int kTileBytes = 128 * 64 * 2;       // one [128 rows][64 cols] bf16 TMA box
constexpr int kQBytes = 2 * kTileBytes;        // one Q tile: two 64-column K-atoms
constexpr int kKVBytes = 2 * kTileBytes;       // one K or V tile (two 64-column boxes)
constexpr int kKSlots = 3, kVSlots = 2;        // K frees after S_B(j), V after PV_B(j)
// + barriers (256 B) + the row-max exchange buffer of the 2-warps-per-row softmax (2 KB).
// This needs the dynamic shared-memory base to be 1024-aligned already (checked).
constexpr int kSmem = 2 * kQBytes + (kKSlots + kVSlots) * kKVBytes + 256 + 2048;
#ifndef CB_ATTN_FWD_NH
#define CB_ATTN_FWD_NH 1
#endif
constexpr int kFwdNH = CB_ATTN_FWD_NH;  // softmax warps per query row (1 or 2)
constexpr uint32_t kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef CB_ATTN_EMU
#define CB_ATTN_EMU 2
#endif
constexpr int kEmuPairs = CB_ATTN_EMU;  // of every 8 exp2 pairs, this many on the FMA pipe
#ifndef CB_ATTN_SPLIT_P
#define CB_ATTN_SPLIT_P 96
#endif
constexpr int kSplitP = CB_ATTN_SPLIT_P;  // keys of P V issued before the softmax finishes (x 32)

struct Params {
  int T, H, KVH, B;
  float scale;
  __nv_bfloat16* o;
  int64_t ldo;
  float* lse;
  __nv_bfloat16* o_lo;  // optional: o - bf16(o) as bf16 (same layout as o)
};

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// NH softmax warps per query row: warps 4 .. 4 + 8 NH, 128 + 256 NH threads.  With NH = 2
// the two warps of a TMEM lane quadrant split each S row into column halves and exchange
// their row maxima through shared memory (named barrier per warp pair).
template <int NH>
__global__ void __launch_bounds__(128 + 256 * NH, 1)
    fwd_tc_k(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem) & 1023) __trap();  // see kSmem
  uint8_t* sQ = smem;  // [2 tiles][kQBytes]
  uint8_t* sK = smem + 2 * kQBytes;    // [kKSlots]
  uint8_t* sV = sK + kKSlots * kKVBytes;  // [kVSlots]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVSlots * kKVBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [3]
  uint64_t* k_empty = bars + 4;   // [3]
  uint64_t* v_full = bars + 7;    // [2]
  uint64_t* v_empty = bars + 9;   // [2]
  uint64_t* s_full = bars + 11;   // [2] tiles
  uint64_t* p_ready = bars + 13;  // [2] tiles
  uint64_t* o_done = bars + 15;   // [2] tiles
  uint64_t* p_part = bars + 17;   // [2] tiles: the first kSplitP S columns' P is in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);
  float* red = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [2 tiles][2 halves][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.KVH);
  const int q0 = qb * 2 * BM;
  const int nblk = (p.T + BN - 1) / BN;
  const int row0 = b * p.T;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_ready[s], 4 * NH);
      mbar_init(&p_part[s], 4 * NH);
      mbar_init(&o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kQBytes);
      for (int x = 0; x < 2; ++x) {
        tma_load_2d(sQ + x * kQBytes, &tmQ, q_full, h * HD, row0 + q0 + x * BM);
        tma_load_2d(sQ + x * kQBytes + kTileBytes, &tmQ, q_full, h * HD + 64, row0 + q0 + x * BM);
      }
      for (int j = 0; j < nblk; ++j) {
        const int st = j % kKSlots;
        mbar_wait(&k_empty[st], ((j / kKSlots) & 1) ^ 1);
        ATTN_TRACE(12, j);
        mbar_expect_tx(&k_full[st], kKVBytes);
        tma_load_2d(sK + st * kKVBytes, &tmK, &k_full[st], kvh * HD, row0 + j * BN);
        tma_load_2d(sK + st * kKVBytes + kTileBytes, &tmK, &k_full[st], kvh * HD + 64, row0 + j * BN);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // second producer: V_j, independent of the K ring
    if (lane == 0) {
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        ATTN_TRACE(13, j);
        mbar_expect_tx(&v_full[st], kKVBytes);
        tma_load_2d(sV + st * kKVBytes, &tmV, &v_full[st], kvh * HD, row0 + j * BN);
        tma_load_2d(sV + st * kKVBytes + kTileBytes, &tmV, &v_full[st], kvh * HD + 64, row0 + j * BN);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the schedule (so descriptors stay warp-uniform, in
    // uniform registers) and one elected lane issues each group of tcgen05.mma
    const uint32_t idesc_s = idesc_bf16_f32(BM, BN, 0, 0);
    const uint32_t idesc_o = idesc_bf16_f32(BM, HD, 0, 1);
    auto issue_s = [&](int x, int j) {
      ATTN_TRACE(x, j);
      const uint64_t qd = sw128_desc(smem_u32(sQ + x * kQBytes), 16, 1024);
      const uint64_t kd = sw128_desc(smem_u32(sK + (j % kKSlots) * kKVBytes), 16, 1024);
      const uint32_t d = tmem + x * 128u;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * kTileBytes + (kk & 3) * 32) >> 4);
          umma_f16_ss(d, qd + off, kd + off, idesc_s, kk > 0);
        }
        umma_commit(&s_full[x]);
      }
      __syncwarp();
    };
    // O += P V in two parts: the K-steps over the first kSplitP keys as soon as the softmax
    // warps have stored that much of P (p_part), the rest after p_ready, so the PV MMAs start
    // while the softmax finishes its last columns
    auto issue_pv = [&](int x, int j) {
      if (x == 0) ATTN_TRACE(14, j);
      if (x == 0) mbar_wait(&v_full[j & 1], (j >> 1) & 1);
      const uint64_t vd = sw128_desc(smem_u32(sV + (j & 1) * kKVBytes), 16384, 1024);
      const uint32_t o = tmem + 256u + x * 128u, pa = tmem + x * 128u;
      mbar_wait(&p_part[x], j & 1);
      tc_fence_after();
      ATTN_TRACE(2 + x, j);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kSplitP / 16; ++k)
          umma_f16_ts(o, pa + k * 8, vd + (uint64_t)(k * 128), idesc_o, (j | k) != 0);
      }
      __syncwarp();
      mbar_wait(&p_ready[x], j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = kSplitP / 16; k < BN / 16; ++k)
          umma_f16_ts(o, pa + k * 8, vd + (uint64_t)(k * 128), idesc_o, (j | k) != 0);
        umma_commit(&o_done[x]);
      }
      __syncwarp();
      ATTN_TRACE(10 + 5 * x, j);
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    commit(&k_empty[0]);
    for (int j = 0; j < nblk; ++j) {
      issue_pv(0, j);
      if (j + 1 < nblk) {
        mbar_wait(&k_full[(j + 1) % kKSlots], ((j + 1) / kKSlots) & 1);
        tc_fence_after();
        issue_s(0, j + 1);
      }
      issue_pv(1, j);
      commit(&v_empty[j & 1]);
      if (j + 1 < nblk) {
        issue_s(1, j + 1);
        commit(&k_empty[(j + 1) % kKSlots]);
      }
    }
  } else if (warp >= 4) {
    constexpr int W = BN / NH;  // S columns per warp
    const int x = (warp - 4) / (4 * NH);   // query tile
    const int wi = (warp - 4) % (4 * NH);
    const int q = wi & 3;                  // TMEM lane quadrant
    const int hf = wi >> 2;                // column half (NH = 2)
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t scol = tmem + lane_off + x * 128u;
    const uint32_t ocol = tmem + lane_off + 256u + x * 128u + hf * (HD / NH);
    const float c = p.scale * kLog2e;
    float* myred = red + (x * 2 + hf) * 128 + row;
    const float* partred = red + (x * 2 + (hf ^ 1)) * 128 + row;
    const int bar_id = 1 + x * 4 + q;
    float m_used = -INFINITY, l = 0.f;
    // one K/V block of the online softmax; kRagged (the last block when T % 128 != 0) masks
    // the columns past T — a separate instantiation keeps the masking out of the hot loop
    auto block = [&](int j, auto ragged) {
      constexpr bool kRagged = decltype(ragged)::value;
      mbar_wait(&s_full[x], j & 1);
      tc_fence_after();
      if (wi == 0 && lane == 0) ATTN_TRACE(4 + 3 * x, j);
      // this warp's W columns of the S row in registers: loads in flight, one wait
      const int valid = min(BN, p.T - j * BN) - hf * W;
      uint32_t sv[W / 32][32];
#pragma unroll
      for (int cc = 0; cc < W / 32; ++cc) tmem_ld32(scol + hf * W + cc * 32, sv[cc]);
      tmem_ld_wait_regs(sv[0]);
#pragma unroll
      for (int cc = 1; cc < W / 32; ++cc) reg_fence(sv[cc]);
      if (kRagged) {  // columns past T take no part
#pragma unroll
        for (int cc = 0; cc < W / 32; ++cc)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cc * 32 + i >= valid) sv[cc][i] = __float_as_uint(-INFINITY);
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int cc = 0; cc < W / 32; ++cc)
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          mx0 = fmaxf(mx0, fmaxf(__uint_as_float(sv[cc][i]), __uint_as_float(sv[cc][i + 1])));
          mx1 = fmaxf(mx1, fmaxf(__uint_as_float(sv[cc][i + 2]), __uint_as_float(sv[cc][i + 3])));
        }
      float mx = fmaxf(mx0, mx1) * c;
      if (NH == 2) {
        // row max across the two halves; the first barrier keeps this write after the
        // partner's read of the previous block, the second publishes it (and orders both
        // warps' S loads before either overwrites columns with packed P)
        named_bar(bar_id, 64);
        *myred = mx;
        named_bar(bar_id, 64);
        mx = fmaxf(mx, *partred);
      }
      if (wi == 0 && lane == 0) ATTN_TRACE(5 + 3 * x, j);
      const bool need = mx > m_used + kRescaleThreshold;  // same decision in both halves
      const float m_prev = m_used;
      if (need) m_used = mx;
      // P = exp2(S c - m) packed to bf16 pairs: this warp's W columns -> packed columns
      // [hf W/2, (hf+1) W/2) of the S region.  Pair arithmetic (FFMA2/FADD2); kEmuPairs of
      // every 8 pairs take the polynomial exp2 on the FMA pipe.
      const float2 c2 = make_float2(c, c), nm2 = make_float2(-m_used, -m_used);
      float2 rsa = make_float2(0.f, 0.f), rsb = make_float2(0.f, 0.f);
      // a pending O rescale must precede every PV MMA of this block: then p_part is signalled
      // only after the rescale below (with p_ready)
      const bool early = NH == 1 && kSplitP < BN && !__any_sync(0xffffffffu, need);
#pragma unroll
      for (int cc = 0; cc < W / 32; ++cc) {
        if (early && cc == kSplitP / 32) {
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_part[x]);
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 a = ffma2(make_float2(__uint_as_float(sv[cc][2 * i]), __uint_as_float(sv[cc][2 * i + 1])), c2, nm2);
          float2 e;
          if ((i & 7) < kEmuPairs) {
            e = exp2_poly2(a);
          } else {
            e.x = fast_exp2(a.x);
            e.y = fast_exp2(a.y);
          }
          if (i & 1)
            rsb = fadd2(rsb, e);
          else
            rsa = fadd2(rsa, e);
          pk[i] = pack2(e.x, e.y);
        }
        tmem_st16(scol + hf * (W / 2) + cc * 16, pk);
      }
      const float rs = (rsa.x + rsa.y) + (rsb.x + rsb.y);
      // lazy rescale of O (after the exponentials, when the S row is no longer live): only
      // when some row's max grew past the threshold; PV_j has not been issued yet.  Each
      // warp rescales its HD / NH output columns.
      if (__any_sync(0xffffffffu, need)) {
        const float corr = need ? fast_exp2(m_prev - m_used) : 1.f;
        if (j > 0) {
          mbar_wait(&o_done[x], (j - 1) & 1);  // PV_{j-1} has finished writing O
          tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < HD / NH / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(ocol + cc * 32, o);
            tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st32(ocol + cc * 32, o);
          }
        }
        l *= corr;
      }
      l += rs;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (wi == 0 && lane == 0) ATTN_TRACE(6 + 3 * x, j);
      if (lane == 0) {
        if (!early) mbar_arrive(&p_part[x]);
        mbar_arrive(&p_ready[x]);
      }
    };
    const int nfull = p.T / BN;
    for (int j = 0; j < nfull; ++j) block(j, std::false_type{});
    if (nfull < nblk) block(nfull, std::true_type{});
    // epilogue: the row sum is the sum of the halves' partial sums
    if (NH == 2) {
      named_bar(bar_id, 64);
      *myred = l;
      named_bar(bar_id, 64);
      l += *partred;
    }
    mbar_wait(&o_done[x], (nblk - 1) & 1);
    tc_fence_after();
    const int qrow = q0 + x * BM + row;
    const float inv = 1.f / l;
    const int64_t oofs = ((int64_t)row0 + qrow) * p.ldo + (int64_t)h * HD + hf * (HD / NH);
    __nv_bfloat16* orow = p.o + oofs;
#pragma unroll 1
    for (int cc = 0; cc < HD / NH / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(ocol + cc * 32, o);
      tmem_ld_wait();
      if (qrow < p.T) {
        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(o[w * 8 + i]) * inv;
          uint4 pkt;
          pkt.x = pack2(f[0], f[1]);
          pkt.y = pack2(f[2], f[3]);
          pkt.z = pack2(f[4], f[5]);
          pkt.w = pack2(f[6], f[7]);
          dst[w] = pkt;
          if (p.o_lo) {  // the rounding residual, for the backward's delta = rowsum(dO * O)
            const uint32_t hv[4] = {pkt.x, pkt.y, pkt.z, pkt.w};
            uint32_t lv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 hf2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hv[i]));
              lv[i] = pack2(f[2 * i] - hf2.x, f[2 * i + 1] - hf2.y);
            }
            reinterpret_cast<uint4*>(p.o_lo + oofs + cc * 32)[w] = make_uint4(lv[0], lv[1], lv[2], lv[3]);
          }
        }
      }
    }
    if (qrow < p.T && hf == 0) p.lse[((int64_t)b * p.H + h) * p.T + qrow] = (m_used + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace tca

static int g_attn_tc = 1;

bool attn_tc_supported(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v) {
  if (!g_attn_tc || dtype != CB_DT_BF16 || g.hd != 128) return false;
  if ((g.ldq | g.ldk | g.ldv | g.ldo) & 7) return false;
  return ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
}

int attn_fwd_tc(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, void* o_lo, float* lse,
                cudaStream_t st) {
  using namespace tca;
  CUtensorMap mq, mk, mv;
  const uint64_t rows = (uint64_t)g.B * g.T;
  int s;
  if ((s = make_tmap_2d_bf16(&mq, q, rows, (uint64_t)g.H * HD, g.ldq, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mk, k, rows, (uint64_t)g.KVH * HD, g.ldk, 128, 64))) return s;
  if ((s = make_tmap_2d_bf16(&mv, v, rows, (uint64_t)g.KVH * HD, g.ldv, 128, 64))) return s;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fwd_tc_k<kFwdNH>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  Params p{g.T, g.H, g.KVH, g.B, g.scale, (__nv_bfloat16*)o, g.ldo, lse, (__nv_bfloat16*)o_lo};
  dim3 grid((g.T + 2 * BM - 1) / (2 * BM), g.H, g.B);
  fwd_tc_k<kFwdNH><<<grid, 128 + 256 * kFwdNH, kSmem, st>>>(mq, mk, mv, p);
  return check_launch("flash_fwd_tc");
}

}  // namespace cb

extern "C" int cb_attention_set_tc(int enable) {
  cb::g_attn_tc = enable ? 1 : 0;
  return CB_OK;
}
