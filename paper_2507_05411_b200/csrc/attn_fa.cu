// Tensor-core flash attention for bf16 (head_dim 64 / 128), unmasked, GQA-aware.
//
// Reference op: AttentionBehavior.forward (reference layers.py:331-348) — softmax over all
// T keys (no causal mask), so every (query block, key block) tile is computed.
//
// Engine: warp-level bf16 MMA (m16n8k16, f32 accumulate) with ldmatrix from XOR-swizzled
// shared memory and cp.async double-buffered K/V (or Q/dO) tiles.  64-row tiles, 4 warps
// per CTA, 16 rows per warp; online softmax in the exp2 domain with f32 statistics.
//   fwd : grid (T/64 query blocks, H, B);  O and the per-row natural-log LSE.
//   bwd : deterministic, no atomics — one kernel owns a 64-key block and sweeps every
//         query block of every query head in its KV group (dK, dV), a second owns a
//         64-query block and sweeps every key block (dQ); both recompute P from the LSE.
#include "attn.cuh"
#include "composer_b200.h"

namespace cb {
namespace fa {

typedef __nv_bfloat16 bf16;
constexpr int BM = 64, BN = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// byte offset of 16-byte chunk `c` of row `r` in a swizzled [rows][HD] bf16 tile
template <int HD>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)(r * HD * 2 + ((c ^ (r & 7)) << 4));
}

// async copy of `rows` x HD tile; rows beyond `valid_rows` are zero-filled
template <int HD>
__device__ __forceinline__ void load_tile(uint32_t sbase, const bf16* g, int64_t ld, int valid_rows) {
  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < 64 * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < valid_rows;
    cp16(sbase + swz<HD>(r, c), ok ? (const void*)(g + (int64_t)r * ld + c * 8) : (const void*)g, ok);
  }
}

// ------------------------------------------------------------------------------ forward
template <int HD>
__global__ void __launch_bounds__(128) fwd_k(AttnGeom g, const bf16* __restrict__ q, const bf16* __restrict__ k,
                                             const bf16* __restrict__ v, bf16* __restrict__ o, float* __restrict__ lse) {
  constexpr int TILE = 64 * HD * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem), sK = sQ + TILE, sV = sQ + 3 * TILE;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (g.H / g.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int q0 = qb * BM;
  const bf16* qg = q + ((int64_t)b * g.T + q0) * g.ldq + (int64_t)h * HD;
  const bf16* kg = k + (int64_t)b * g.T * g.ldk + (int64_t)kvh * HD;
  const bf16* vg = v + (int64_t)b * g.T * g.ldv + (int64_t)kvh * HD;
  load_tile<HD>(sQ, qg, g.ldq, g.T - q0);
  load_tile<HD>(sK, kg, g.ldk, g.T);
  load_tile<HD>(sV, vg, g.ldv, g.T);
  cp_commit();
  const float c = g.scale * kLog2e;
  float oacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[HD / 16][4];
  const int nblk = (g.T + BN - 1) / BN;
  for (int j = 0; j < nblk; ++j) {
    const int st = j & 1;
    if (j + 1 < nblk) {
      const int k1 = (j + 1) * BN;
      load_tile<HD>(sK + (st ^ 1) * TILE, kg + (int64_t)k1 * g.ldk, g.ldk, g.T - k1);
      load_tile<HD>(sV + (st ^ 1) * TILE, vg + (int64_t)k1 * g.ldv, g.ldv, g.T - k1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(sQ + swz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    const uint32_t kt = sK + st * TILE, vt = sV + st * TILE;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kt + swz<HD>(np * 16 + (lane & 7) + ((lane >> 4) << 3), kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
        mma(s[2 * np], qf[kk], b0, b1);
        mma(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    const int kbase = j * BN;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int key = kbase + nt * 8 + 2 * tq;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = key + (e & 1) < g.T;
        s[nt][e] = ok ? s[nt][e] * c : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float cr0 = exp2f(m0 - mn0), cr1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mn0), p1 = exp2f(s[nt][1] - mn0);
      const float p2 = exp2f(s[nt][2] - mn1), p3 = exp2f(s[nt][3] - mn1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
    l0 = l0 * cr0 + rs0;
    l1 = l1 * cr1 + rs1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      oacc[i][0] *= cr0;
      oacc[i][1] *= cr0;
      oacc[i][2] *= cr1;
      oacc[i][3] *= cr1;
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      // A fragment order: a0 (row g, k 0-7) a1 (row g+8, k 0-7) a2 (row g, k 8-15) a3 (row g+8, k 8-15)
      const uint32_t a[4] = {pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3]};
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vt + swz<HD>(ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dp * 2 + (lane >> 4)), b0, b1, b2, b3);
        mma(oacc[2 * dp], a, b0, b1);
        mma(oacc[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  const int r0 = q0 + warp * 16 + gq, r1 = r0 + 8;
  bf16* ob = o + (int64_t)b * g.T * g.ldo + (int64_t)h * HD;
#pragma unroll
  for (int dt = 0; dt < HD / 8; ++dt) {
    const int col = dt * 8 + 2 * tq;
    if (r0 < g.T) *reinterpret_cast<uint32_t*>(ob + (int64_t)r0 * g.ldo + col) = pack_bf16(oacc[dt][0] * inv0, oacc[dt][1] * inv0);
    if (r1 < g.T) *reinterpret_cast<uint32_t*>(ob + (int64_t)r1 * g.ldo + col) = pack_bf16(oacc[dt][2] * inv1, oacc[dt][3] * inv1);
  }
  if (tq == 0) {
    float* lb = lse + ((int64_t)b * g.H + h) * g.T;
    if (r0 < g.T) lb[r0] = (m0 + log2f(l0)) * kLn2;
    if (r1 < g.T) lb[r1] = (m1 + log2f(l1)) * kLn2;
  }
}

// ------------------------------------------------------------------ backward: dK, dV
template <int HD>
__global__ void __launch_bounds__(128) bwd_dkdv_k(AttnGeom g, const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                  const bf16* __restrict__ v, const bf16* __restrict__ dout,
                                                  int64_t lddo, const float* __restrict__ lse,
                                                  const float* __restrict__ delta, bf16* __restrict__ dk, int64_t lddk,
                                                  bf16* __restrict__ dv, int64_t lddv) {
  constexpr int TILE = 64 * HD * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = smem_u32(smem), sV = sK + TILE, sQ = sK + 2 * TILE, sG = sK + 4 * TILE;
  float* sL = reinterpret_cast<float*>(smem + 6 * TILE);  // [2][64] lse*log2e
  float* sD = sL + 128;                                   // [2][64] delta
  const int kb = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int group = g.H / g.KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int k0 = kb * BN;
  load_tile<HD>(sK, k + ((int64_t)b * g.T + k0) * g.ldk + (int64_t)kvh * HD, g.ldk, g.T - k0);
  load_tile<HD>(sV, v + ((int64_t)b * g.T + k0) * g.ldv + (int64_t)kvh * HD, g.ldv, g.T - k0);
  cp_commit();
  const float c = g.scale * kLog2e;
  float dka[HD / 8][4], dva[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dka[i][e] = dva[i][e] = 0.f;
  const int nq = (g.T + BM - 1) / BM;
  const int total = nq * group;
  auto issue = [&](int it, int st) {
    const int hh = it / nq, qbk = it % nq;
    const int h = kvh * group + hh;
    const int q0 = qbk * BM;
    load_tile<HD>(sQ + st * TILE, q + ((int64_t)b * g.T + q0) * g.ldq + (int64_t)h * HD, g.ldq, g.T - q0);
    load_tile<HD>(sG + st * TILE, dout + ((int64_t)b * g.T + q0) * lddo + (int64_t)h * HD, lddo, g.T - q0);
    for (int i = threadIdx.x; i < BM; i += blockDim.x) {
      const int r = q0 + i;
      const int64_t li = ((int64_t)b * g.H + h) * g.T + r;
      sL[st * 64 + i] = r < g.T ? lse[li] * kLog2e : 0.f;
      sD[st * 64 + i] = r < g.T ? delta[li] : 0.f;
    }
  };
  issue(0, 0);
  cp_commit();
  for (int it = 0; it < total; ++it) {
    const int st = it & 1;
    if (it + 1 < total) {
      issue(it + 1, st ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int q0 = (it % nq) * BM;
    const uint32_t qt = sQ + st * TILE, gt = sG + st * TILE;
    const float* Ls = sL + st * 64;
    const float* Ds = sD + st * 64;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float sT[4][4], dpT[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) sT[i][e] = dpT[i][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t ak[4], av[4];
        ldsm_x4(sK + swz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), ak[0], ak[1], ak[2], ak[3]);
        ldsm_x4(sV + swz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), av[0], av[1], av[2], av[3]);
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          const int row = half * 32 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(qt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma(sT[2 * np], ak, b0, b1);
          mma(sT[2 * np + 1], ak, b2, b3);
          ldsm_x4(gt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma(dpT[2 * np], av, b0, b1);
          mma(dpT[2 * np + 1], av, b2, b3);
        }
      }
      // rows: keys (warp*16 + gq, +8); cols: queries half*32 + nt*8 + 2tq + {0,1}
      uint32_t pa[2][4], da[2][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int qi = half * 32 + nt * 8 + 2 * tq;
        float p[4], ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = qi + (e & 1);
          const bool ok = q0 + col < g.T;
          p[e] = ok ? exp2f(sT[nt][e] * c - Ls[col]) : 0.f;
          ds[e] = p[e] * (dpT[nt][e] - Ds[col]);
        }
        pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
        pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
        da[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
        da[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int row = half * 32 + ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(gt + swz<HD>(row, dp * 2 + (lane >> 4)), b0, b1, b2, b3);
          mma(dva[2 * dp], pa[ks], b0, b1);
          mma(dva[2 * dp + 1], pa[ks], b2, b3);
          ldsm_x4_t(qt + swz<HD>(row, dp * 2 + (lane >> 4)), b0, b1, b2, b3);
          mma(dka[2 * dp], da[ks], b0, b1);
          mma(dka[2 * dp + 1], da[ks], b2, b3);
        }
      }
    }
    __syncthreads();
  }
  const int r0 = k0 + warp * 16 + gq, r1 = r0 + 8;
  bf16* dkb = dk + (int64_t)b * g.T * lddk + (int64_t)kvh * HD;
  bf16* dvb = dv + (int64_t)b * g.T * lddv + (int64_t)kvh * HD;
#pragma unroll
  for (int dt = 0; dt < HD / 8; ++dt) {
    const int col = dt * 8 + 2 * tq;
    if (r0 < g.T) {
      *reinterpret_cast<uint32_t*>(dkb + (int64_t)r0 * lddk + col) = pack_bf16(dka[dt][0] * g.scale, dka[dt][1] * g.scale);
      *reinterpret_cast<uint32_t*>(dvb + (int64_t)r0 * lddv + col) = pack_bf16(dva[dt][0], dva[dt][1]);
    }
    if (r1 < g.T) {
      *reinterpret_cast<uint32_t*>(dkb + (int64_t)r1 * lddk + col) = pack_bf16(dka[dt][2] * g.scale, dka[dt][3] * g.scale);
      *reinterpret_cast<uint32_t*>(dvb + (int64_t)r1 * lddv + col) = pack_bf16(dva[dt][2], dva[dt][3]);
    }
  }
}

// ----------------------------------------------------------------------- backward: dQ
template <int HD>
__global__ void __launch_bounds__(128) bwd_dq_k(AttnGeom g, const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                const bf16* __restrict__ v, const bf16* __restrict__ dout, int64_t lddo,
                                                const float* __restrict__ lse, const float* __restrict__ delta,
                                                bf16* __restrict__ dq, int64_t lddq) {
  constexpr int TILE = 64 * HD * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem), sG = sQ + TILE, sK = sQ + 2 * TILE, sV = sQ + 4 * TILE;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (g.H / g.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int q0 = qb * BM;
  const bf16* kg = k + (int64_t)b * g.T * g.ldk + (int64_t)kvh * HD;
  const bf16* vg = v + (int64_t)b * g.T * g.ldv + (int64_t)kvh * HD;
  load_tile<HD>(sQ, q + ((int64_t)b * g.T + q0) * g.ldq + (int64_t)h * HD, g.ldq, g.T - q0);
  load_tile<HD>(sG, dout + ((int64_t)b * g.T + q0) * lddo + (int64_t)h * HD, lddo, g.T - q0);
  load_tile<HD>(sK, kg, g.ldk, g.T);
  load_tile<HD>(sV, vg, g.ldv, g.T);
  cp_commit();
  const float c = g.scale * kLog2e;
  const int r0 = q0 + warp * 16 + gq, r1 = r0 + 8;
  const int64_t lbase = ((int64_t)b * g.H + h) * g.T;
  const float L0 = r0 < g.T ? lse[lbase + r0] * kLog2e : 0.f, L1 = r1 < g.T ? lse[lbase + r1] * kLog2e : 0.f;
  const float D0 = r0 < g.T ? delta[lbase + r0] : 0.f, D1 = r1 < g.T ? delta[lbase + r1] : 0.f;
  float dqa[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dqa[i][0] = dqa[i][1] = dqa[i][2] = dqa[i][3] = 0.f;
  const int nblk = (g.T + BN - 1) / BN;
  for (int j = 0; j < nblk; ++j) {
    const int st = j & 1;
    if (j + 1 < nblk) {
      const int k1 = (j + 1) * BN;
      load_tile<HD>(sK + (st ^ 1) * TILE, kg + (int64_t)k1 * g.ldk, g.ldk, g.T - k1);
      load_tile<HD>(sV + (st ^ 1) * TILE, vg + (int64_t)k1 * g.ldv, g.ldv, g.T - k1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t kt = sK + st * TILE, vt = sV + st * TILE;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float s[4][4], dp[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t aq[4], ag[4];
        ldsm_x4(sQ + swz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), aq[0], aq[1], aq[2], aq[3]);
        ldsm_x4(sG + swz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), ag[0], ag[1], ag[2], ag[3]);
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          const int row = half * 32 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma(s[2 * np], aq, b0, b1);
          mma(s[2 * np + 1], aq, b2, b3);
          ldsm_x4(vt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma(dp[2 * np], ag, b0, b1);
          mma(dp[2 * np + 1], ag, b2, b3);
        }
      }
      uint32_t da[2][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int key = j * BN + half * 32 + nt * 8 + 2 * tq;
        float ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = key + (e & 1) < g.T;
          const float p = ok ? exp2f(s[nt][e] * c - (e < 2 ? L0 : L1)) : 0.f;
          ds[e] = p * (dp[nt][e] - (e < 2 ? D0 : D1));
        }
        da[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
        da[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int row = half * 32 + ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
        for (int dpi = 0; dpi < HD / 16; ++dpi) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(kt + swz<HD>(row, dpi * 2 + (lane >> 4)), b0, b1, b2, b3);
          mma(dqa[2 * dpi], da[ks], b0, b1);
          mma(dqa[2 * dpi + 1], da[ks], b2, b3);
        }
      }
    }
    __syncthreads();
  }
  bf16* qo = dq + (int64_t)b * g.T * lddq + (int64_t)h * HD;
#pragma unroll
  for (int dt = 0; dt < HD / 8; ++dt) {
    const int col = dt * 8 + 2 * tq;
    if (r0 < g.T) *reinterpret_cast<uint32_t*>(qo + (int64_t)r0 * lddq + col) = pack_bf16(dqa[dt][0] * g.scale, dqa[dt][1] * g.scale);
    if (r1 < g.T) *reinterpret_cast<uint32_t*>(qo + (int64_t)r1 * lddq + col) = pack_bf16(dqa[dt][2] * g.scale, dqa[dt][3] * g.scale);
  }
}

template <int HD>
int launch_fwd(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
  const int smem = 5 * 64 * HD * 2;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(fwd_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  dim3 grid((g.T + BM - 1) / BM, g.H, g.B);
  fwd_k<HD><<<grid, 128, smem, st>>>(g, (const bf16*)q, (const bf16*)k, (const bf16*)v, (bf16*)o, lse);
  return check_launch("flash_fwd");
}

template <int HD>
int launch_bwd(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, int64_t lddo,
               const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
               int64_t lddv, cudaStream_t st) {
  const int smem_kv = 6 * 64 * HD * 2 + 4 * 64 * 4;
  const int smem_q = 6 * 64 * HD * 2;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(bwd_dkdv_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
    cudaFuncSetAttribute(bwd_dq_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
    set = true;
  }
  dim3 gkv((g.T + BN - 1) / BN, g.KVH, g.B);
  bwd_dkdv_k<HD><<<gkv, 128, smem_kv, st>>>(g, (const bf16*)q, (const bf16*)k, (const bf16*)v, (const bf16*)dout, lddo,
                                           lse, delta, (bf16*)dk, lddk, (bf16*)dv, lddv);
  if (int s = check_launch("flash_bwd_dkdv")) return s;
  dim3 gq((g.T + BM - 1) / BM, g.H, g.B);
  bwd_dq_k<HD><<<gq, 128, smem_q, st>>>(g, (const bf16*)q, (const bf16*)k, (const bf16*)v, (const bf16*)dout, lddo, lse,
                                       delta, (bf16*)dq, lddq);
  return check_launch("flash_bwd_dq");
}

}  // namespace fa

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool attn_fa_supported(const AttnGeom& g, int dtype, const void* q, const void* k, const void* v) {
  if (dtype != CB_DT_BF16) return false;
  if (g.hd != 64 && g.hd != 128) return false;
  if ((g.ldq | g.ldk | g.ldv | g.ldo) & 7) return false;
  return aligned16(q) && aligned16(k) && aligned16(v);
}

int attn_fwd_fa(const AttnGeom& g, const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
  if (g.hd == 128) return fa::launch_fwd<128>(g, q, k, v, o, lse, st);
  return fa::launch_fwd<64>(g, q, k, v, o, lse, st);
}

int attn_bwd_fa(const AttnGeom& g, const void* q, const void* k, const void* v, const void* dout, int64_t lddo,
                const float* lse, const float* delta, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                int64_t lddv, cudaStream_t st) {
  if ((lddo | lddq | lddk | lddv) & 7) return fail(CB_ERR_ARG, "flash bwd: gradient strides must be 16-byte aligned");
  if (g.hd == 128) return fa::launch_bwd<128>(g, q, k, v, dout, lddo, lse, delta, dq, lddq, dk, lddk, dv, lddv, st);
  return fa::launch_bwd<64>(g, q, k, v, dout, lddo, lse, delta, dq, lddq, dk, lddk, dv, lddv, st);
}

}  // namespace cb
