"""Times the tcgen05 GEMM on the 1B/7B layer shapes (CUDA events, inputs > L2 rotated)."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_05411_b200 import _lib, ops

shapes = [(32768, 2048, 2048, 0, 0), (32768, 5632, 2048, 0, 0), (32768, 2048, 5632, 0, 0),
          (32768, 2048, 2048, 0, 1), (2048, 2048, 32768, 1, 0), (16384, 4096, 4096, 0, 0), (16384, 32000, 4096, 0, 1)]
dev = torch.device("cuda")
for (M, N, K, ta, tb) in shapes:
    a = torch.randn((K, M) if ta else (M, K), device=dev).bfloat16()
    b = torch.randn((N, K) if tb else (K, N), device=dev).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        ops.gemm(a, b, out, trans_a=bool(ta), trans_b=bool(tb))
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    s.record()
    for _ in range(n):
        ops.gemm(a, b, out, trans_a=bool(ta), trans_b=bool(tb))
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    tf = 2 * M * N * K / ms / 1e9
    _lib.call("cb_gemm_set_multicast", 0)
    for _ in range(3):
        ops.gemm(a, b, out, trans_a=bool(ta), trans_b=bool(tb))
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        ops.gemm(a, b, out, trans_a=bool(ta), trans_b=bool(tb))
    e.record()
    torch.cuda.synchronize()
    tf1 = 2 * M * N * K / (s.elapsed_time(e) / n) / 1e9
    _lib.call("cb_gemm_set_multicast", 1)
    # torch (cuBLAS) for context
    A = a.t() if ta else a
    B = b.t() if tb else b
    for _ in range(3):
        torch.matmul(A, B)
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        torch.matmul(A, B)
    e.record()
    torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / n
    print(json.dumps({"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "ms": round(ms, 4), "tflops": round(tf, 1), "tflops_1cta": round(tf1, 1),
                      "cublas_tflops": round(2 * M * N * K / ms2 / 1e9, 1)}), flush=True)
