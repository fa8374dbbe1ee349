// Host-side runtime support: thread-local error reporting and TMA descriptor encoding.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <mutex>

#include "common.cuh"
#include "composer_b200.h"

namespace cb {

static thread_local char g_last_error[1024] = {0};

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

static std::atomic<long long> g_launches{0};

int check_launch(const char* what, int launches) {
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return CB_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static int encoder(PFN_cuTensorMapEncodeTiled_v12000* fn) {
  std::call_once(g_encode_once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!g_encode) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  *fn = g_encode;
  return CB_OK;
}

int make_tmap_2d_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, uint32_t box_cols) {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  if (int s = encoder(&enc)) return s;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 2) & 15))
    return fail(CB_ERR_ARG, "TMA needs 16-byte aligned base and row stride (ld=%llu)", (unsigned long long)ld);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled(2d) failed: %d", (int)r);
  return CB_OK;
}

int make_tmap_3d_bf16(CUtensorMap* out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                      uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2) {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  if (int s = encoder(&enc)) return s;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((s1 * 2) & 15) || ((s2 * 2) & 15))
    return fail(CB_ERR_ARG, "TMA needs 16-byte aligned base and strides");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 2, s2 * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled(3d) failed: %d", (int)r);
  return CB_OK;
}

}  // namespace cb

extern "C" const char* cb_last_error(void) { return cb::g_last_error; }
extern "C" int cb_abi_version(void) { return 1; }
// Number of kernels this library has launched in this process (all threads).
extern "C" long long cb_launch_count(void) { return cb::g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------- stream memory operations
// Cross-GPU ordering without a kernel: the FSDP collectives' barriers as stream memory
// operations executed by the GPU front end (no SM spins while a peer is late).  A rank posts
// an epoch into each peer's signal slot (cuStreamWriteValue32 through the peer mapping of
// symmetric memory, after a memory barrier that makes its earlier writes visible) and waits
// until its own slots reach the epoch (cuStreamWaitValue32, GEQ).
namespace cb {
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_streamValue32 g_write32 = nullptr, g_wait32 = nullptr;
static std::once_flag g_memop_once;

static int memops() {
  std::call_once(g_memop_once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write32 = reinterpret_cast<PFN_streamValue32>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait32 = reinterpret_cast<PFN_streamValue32>(p);
  });
  if (!g_write32 || !g_wait32) return fail(CB_ERR_UNSUPPORTED, "stream memory operations unavailable from the driver");
  return CB_OK;
}
}  // namespace cb

using namespace cb;

extern "C" int cb_stream_signal(void* const* slots, int n, uint32_t epoch, void* stream) {
  if (int s = memops()) return s;
  for (int i = 0; i < n; ++i) {
    // default flags: a memory barrier orders the stream's earlier writes before the value
    CUresult r = g_write32((CUstream)stream, (CUdeviceptr)slots[i], epoch, 0);
    if (r != CUDA_SUCCESS) return fail(CB_ERR_CUDA, "cuStreamWriteValue32 failed: %d", (int)r);
  }
  return CB_OK;
}

extern "C" int cb_stream_wait(void* const* slots, int n, uint32_t epoch, void* stream) {
  if (int s = memops()) return s;
  for (int i = 0; i < n; ++i) {
    CUresult r = g_wait32((CUstream)stream, (CUdeviceptr)slots[i], epoch, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(CB_ERR_CUDA, "cuStreamWaitValue32 failed: %d", (int)r);
  }
  return CB_OK;
}
