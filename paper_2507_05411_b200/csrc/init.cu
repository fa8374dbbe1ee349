// Parameter initialisation on the device, bit-identical to the reference's init_state.
//
// Reference: prng.py:61-69 (generator = numpy PCG64(SeedSequence(int(key))),
// uniform(low, high) = low + (high - low) * next_double) and layers.py:114-116
// (U(-1/sqrt(fan_in), 1/sqrt(fan_in)) per parameter, C order).
//
// numpy's PCG64 is the 128-bit LCG state' = state * M + inc followed by the XSL-RR output
// rotr64(hi ^ lo, hi >> 58); next_double = (out >> 11) * 2^-53.  The host derives each
// tensor's (state, inc) from its key with numpy's SeedSequence (a few hundred ns); every
// thread then jumps the LCG to the start of its 64-element chunk (O(log n) 128-bit
// multiply-adds) and steps sequentially, converting in double exactly as numpy does
// (explicit round-to-nearest mul/add, no FMA contraction) before rounding to the stored
// f32 master / bf16 working copies.  7B parameters initialise in well under a second
// instead of generating 53 GB of float64 on the host.
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

struct U128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__device__ __constant__ U128 kMult = {4865540595714422341ull, 2549297995355413924ull};

// state after `delta` LCG steps (PCG's pcg_advance_lcg_128)
__device__ U128 advance(U128 state, U128 inc, uint64_t delta) {
  U128 acc_mult = {1, 0}, acc_plus = {0, 0}, cur_mult = kMult, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1, 0}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}

constexpr int kChunk = 64;

// element i of a [rows][cols] C-order tensor lands at bucket position
// offset + (i / cols) * ld + col0 + (i % cols)  (ld == 0: contiguous, position offset + i)
__global__ void __launch_bounds__(256) init_uniform_k(uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi,
                                                      int64_t n, double low, double high, int64_t cols, int64_t ld,
                                                      int64_t col0, int64_t offset, float* __restrict__ master,
                                                      int64_t m0, int64_t m1, void* __restrict__ work,
                                                      int work_bf16) {
  const int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kChunk;
  if (c0 >= n) return;
  const U128 inc = {i_lo, i_hi};
  U128 st = advance(U128{s_lo, s_hi}, inc, (uint64_t)c0);
  const double scale = __dsub_rn(high, low);
  const int64_t c1 = min(n, c0 + kChunk);
  for (int64_t i = c0; i < c1; ++i) {
    st = add128(mul128(st, kMult), inc);
    const uint64_t x = st.hi ^ st.lo;
    const unsigned rot = (unsigned)(st.hi >> 58);
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    const double u = (double)(out >> 11) * (1.0 / 9007199254740992.0);
    const float v = (float)__dadd_rn(low, __dmul_rn(scale, u));
    const int64_t pos = ld ? offset + (i / cols) * ld + col0 + (i % cols) : offset + i;
    if (master && pos >= m0 && pos < m1) master[pos - m0] = v;
    if (work) {
      if (work_bf16)
        reinterpret_cast<__nv_bfloat16*>(work)[pos] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(work)[pos] = v;
    }
  }
}

__global__ void init_const_k(int64_t n, float value, int64_t cols, int64_t ld, int64_t col0, int64_t offset,
                             float* __restrict__ master, int64_t m0, int64_t m1, void* __restrict__ work,
                             int work_bf16) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t pos = ld ? offset + (i / cols) * ld + col0 + (i % cols) : offset + i;
  if (master && pos >= m0 && pos < m1) master[pos - m0] = value;
  if (work) {
    if (work_bf16)
      reinterpret_cast<__nv_bfloat16*>(work)[pos] = __float2bfloat16_rn(value);
    else
      reinterpret_cast<float*>(work)[pos] = value;
  }
}

}  // namespace cb

using namespace cb;

extern "C" int cb_init_uniform(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int64_t n,
                               double low, double high, int64_t cols, int64_t ld, int64_t col0, int64_t offset,
                               float* master, int64_t master_begin, int64_t master_end, void* work, int work_dtype,
                               void* stream) {
  if (n <= 0) return CB_OK;
  if (ld && cols <= 0) return fail(CB_ERR_SHAPE, "init: strided tensor needs cols > 0");
  const int64_t threads = (n + kChunk - 1) / kChunk;
  init_uniform_k<<<(int)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      state_lo, state_hi, inc_lo, inc_hi, n, low, high, cols, ld, col0, offset, master, master_begin, master_end, work,
      work_dtype == CB_DT_BF16);
  return check_launch("init_uniform");
}

extern "C" int cb_init_const(int64_t n, float value, int64_t cols, int64_t ld, int64_t col0, int64_t offset,
                             float* master, int64_t master_begin, int64_t master_end, void* work, int work_dtype,
                             void* stream) {
  if (n <= 0) return CB_OK;
  init_const_k<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, value, cols, ld, col0, offset, master,
                                                                         master_begin, master_end, work,
                                                                         work_dtype == CB_DT_BF16);
  return check_launch("init_const");
}
