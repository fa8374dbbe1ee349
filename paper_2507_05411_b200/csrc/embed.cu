// Embedding lookup and its deterministic gradient (reference layers.py:199-229: table[ids]).
//
// Forward: one CTA per token row gathers (and converts) its table row.
// Backward: the table gradient is a scatter-add, which with float atomics would depend on
// arrival order.  Instead a single-CTA stable counting sort groups token positions by id
// (cb_sort_ids), and cb_embedding_bwd then sums each id's rows in position order — the
// same answer on every run (SURVEY §7.3 "the scatter must be deterministic").
#include "common.cuh"
#include "composer_b200.h"

namespace cb {

template <typename TT, typename TO>
__global__ void __launch_bounds__(256) embed_fwd_k(int dim, const int64_t* __restrict__ ids, const TT* __restrict__ table,
                                                   int64_t ldt, TO* __restrict__ out, int64_t ldo) {
  const int64_t row = blockIdx.x;
  const int64_t id = ids[row];
  const TT* src = table + id * ldt;
  TO* dst = out + row * ldo;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) dst[i] = from_f32<TO>(to_f32(src[i]));
}

// Single CTA: histogram -> exclusive scan -> warp-ordered stable scatter.
__global__ void __launch_bounds__(1024) sort_ids_k(int n, int vocab, const int64_t* __restrict__ ids,
                                                   int* __restrict__ offsets, int* __restrict__ cursor,
                                                   int* __restrict__ perm) {
  __shared__ int part[1024];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int v = tid; v < vocab; v += blockDim.x) cursor[v] = 0;
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) atomicAdd(&cursor[(int)ids[i]], 1);
  __syncthreads();
  // exclusive scan of counts: each thread owns a contiguous segment
  const int seg = (vocab + blockDim.x - 1) / blockDim.x;
  const int v0 = min(vocab, tid * seg), v1 = min(vocab, v0 + seg);
  int local = 0;
  for (int v = v0; v < v1; ++v) local += cursor[v];
  part[tid] = local;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
    const int t = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += t;
    __syncthreads();
  }
  int run = part[tid] - local;
  for (int v = v0; v < v1; ++v) {
    const int c = cursor[v];
    offsets[v] = run;
    cursor[v] = run;
    run += c;
  }
  if (tid == 0) offsets[vocab] = n;
  __syncthreads();
  // stable scatter, warps strictly in order within each chunk of 1024 positions
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int base = 0; base < n; base += blockDim.x) {
    const int pos = base + tid;
    const bool valid = pos < n;
    const int id = valid ? (int)ids[pos] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, id);
    const int rank = __popc(peers & lt_mask);
    const bool leader = (peers & lt_mask) == 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (warp == w && valid) {
        perm[cursor[id] + rank] = pos;
      }
      __syncwarp();
      if (warp == w && valid && leader) cursor[id] += __popc(peers);
      __syncthreads();
    }
  }
}

// Multi-CTA stable counting sort for few keys (vocab <= kSortSmallVocab: the MoE dispatch's
// expert ids), the single-CTA kernel's warp-serial scatter being the MoE forward's longest
// serial step.  Chunks of 1024 positions, one per CTA:
//   sort_count_k:   cnt[chunk][v] = occurrences of v in the chunk
//   sort_scatter_k: base[v] = (positions of every key < v) + (occurrences of v in earlier
//                   chunks); within the chunk a position's rank among equal ids is its rank
//                   in its warp (__match_any_sync) plus the counts of that id in earlier warps.
// The output (offsets, perm) is identical to sort_ids_k's: positions grouped by id, in
// position order within an id.
constexpr int kSortChunk = 1024;
constexpr int kSortSmallVocab = 64;

__global__ void __launch_bounds__(kSortChunk) sort_count_k(int n, int vocab, const int64_t* __restrict__ ids,
                                                          int* __restrict__ cnt) {
  __shared__ int c[kSortSmallVocab];
  if (threadIdx.x < vocab) c[threadIdx.x] = 0;
  __syncthreads();
  const int pos = blockIdx.x * kSortChunk + threadIdx.x;
  if (pos < n) atomicAdd(&c[(int)ids[pos]], 1);
  __syncthreads();
  if (threadIdx.x < vocab) cnt[blockIdx.x * vocab + threadIdx.x] = c[threadIdx.x];
}

__global__ void __launch_bounds__(kSortChunk) sort_scatter_k(int n, int vocab, const int64_t* __restrict__ ids,
                                                            const int* __restrict__ cnt, int* __restrict__ offsets,
                                                            int* __restrict__ perm) {
  __shared__ int base[kSortSmallVocab];
  __shared__ int wcnt[kSortChunk / 32][kSortSmallVocab];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunks = gridDim.x, me = blockIdx.x;
  for (int i = tid; i < (kSortChunk / 32) * kSortSmallVocab; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  if (warp == 0) {
    // lane v (and v + 32): total and earlier-chunk counts of key v, then an exclusive scan of
    // the totals across keys
    int tot[2] = {0, 0}, pre[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = lane + 32 * h;
      if (v < vocab)
        for (int b = 0; b < chunks; ++b) {
          const int x = cnt[b * vocab + v];
          tot[h] += x;
          pre[h] += b < me ? x : 0;
        }
    }
    int run = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int inc = tot[h];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int v = lane + 32 * h;
      const int excl = run + inc - tot[h];
      if (v < vocab) {
        base[v] = excl + pre[h];
        if (me == 0) offsets[v] = excl;
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (me == 0 && lane == 0) offsets[vocab] = n;
  }
  __syncthreads();
  const int pos = me * kSortChunk + tid;
  const bool valid = pos < n;
  const int id = valid ? (int)ids[pos] : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, id);
  const unsigned lt_mask = (1u << lane) - 1u;
  const int rank = __popc(peers & lt_mask);
  if (valid && (peers & lt_mask) == 0) wcnt[warp][id] = __popc(peers);
  __syncthreads();
  if (tid < vocab) {  // exclusive prefix of this key's per-warp counts
    int run = 0;
    for (int w = 0; w < kSortChunk / 32; ++w) {
      const int c = wcnt[w][tid];
      wcnt[w][tid] = run;
      run += c;
    }
  }
  __syncthreads();
  if (valid) perm[base[id] + wcnt[warp][id] + rank] = pos;
}

template <typename TG>
__global__ void __launch_bounds__(256) embed_bwd_k(int dim, const int* __restrict__ offsets, const int* __restrict__ perm,
                                                   const TG* __restrict__ dout, int64_t ldo, float* __restrict__ dtable,
                                                   int64_t ldt) {
  const int v = blockIdx.x;
  const int j0 = offsets[v], j1 = offsets[v + 1];
  if (j0 == j1) return;
  float* dst = dtable + (int64_t)v * ldt;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    float acc = 0.f;
    for (int j = j0; j < j1; ++j) acc += to_f32(dout[(int64_t)perm[j] * ldo + i]);
    dst[i] += acc;
  }
}

}  // namespace cb

using namespace cb;

extern "C" int cb_embedding_fwd(int64_t n, int dim, const int64_t* ids, const void* table, int64_t ldt, int t_dtype,
                                void* out, int64_t ldo, int o_dtype, void* stream) {
  if (n <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (t_dtype == CB_DT_F32 && o_dtype == CB_DT_F32)
    embed_fwd_k<float, float><<<n, 256, 0, st>>>(dim, ids, (const float*)table, ldt, (float*)out, ldo);
  else if (t_dtype == CB_DT_F32)
    embed_fwd_k<float, __nv_bfloat16><<<n, 256, 0, st>>>(dim, ids, (const float*)table, ldt, (__nv_bfloat16*)out, ldo);
  else if (o_dtype == CB_DT_F32)
    embed_fwd_k<__nv_bfloat16, float><<<n, 256, 0, st>>>(dim, ids, (const __nv_bfloat16*)table, ldt, (float*)out, ldo);
  else
    embed_fwd_k<__nv_bfloat16, __nv_bfloat16><<<n, 256, 0, st>>>(dim, ids, (const __nv_bfloat16*)table, ldt,
                                                                 (__nv_bfloat16*)out, ldo);
  return check_launch("embedding_fwd");
}

// scratch (the `cursor` argument of cb_sort_ids) in int32 elements
extern "C" int64_t cb_sort_ids_scratch(int n, int vocab) {
  if (vocab <= kSortSmallVocab && n > kSortChunk) return (int64_t)((n + kSortChunk - 1) / kSortChunk) * vocab;
  return vocab;
}

// offsets: int32[vocab+1] (out), cursor: int32[cb_sort_ids_scratch(n, vocab)] (scratch), perm: int32[n] (out)
extern "C" int cb_sort_ids(int n, int vocab, const int64_t* ids, int* offsets, int* cursor, int* perm, void* stream) {
  if (n < 0 || vocab <= 0) return fail(CB_ERR_SHAPE, "sort_ids: bad extents");
  cudaStream_t st = (cudaStream_t)stream;
  if (vocab <= kSortSmallVocab && n > kSortChunk) {
    const int chunks = (n + kSortChunk - 1) / kSortChunk;
    sort_count_k<<<chunks, kSortChunk, 0, st>>>(n, vocab, ids, cursor);
    sort_scatter_k<<<chunks, kSortChunk, 0, st>>>(n, vocab, ids, cursor, offsets, perm);
    return check_launch("sort_ids");
  }
  sort_ids_k<<<1, 1024, 0, st>>>(n, vocab, ids, offsets, cursor, perm);
  return check_launch("sort_ids");
}

extern "C" int cb_embedding_bwd(int vocab, int dim, const int* offsets, const int* perm, const void* dout, int64_t ldo,
                                int g_dtype, float* dtable, int64_t ldt, void* stream) {
  if (vocab <= 0) return CB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g_dtype == CB_DT_F32)
    embed_bwd_k<float><<<vocab, 256, 0, st>>>(dim, offsets, perm, (const float*)dout, ldo, dtable, ldt);
  else
    embed_bwd_k<__nv_bfloat16><<<vocab, 256, 0, st>>>(dim, offsets, perm, (const __nv_bfloat16*)dout, ldo, dtable, ldt);
  return check_launch("embedding_bwd");
}
