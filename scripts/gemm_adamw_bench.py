"""Weight-gradient GEMM (accumulate into f32) vs the same GEMM with AdamW in its epilogue
(cb_gemm_adamw) vs GEMM + the separate cb_adamw, on the 7B step's wgrad shapes (K = tokens)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import _lib, ops  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 12288
SHAPES = {"qkv": (4096, 12288), "o": (4096, 4096), "up": (4096, 22016), "down": (11008, 4096)}
dev = torch.device("cuda")


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for name, (M, N) in SHAPES.items():
    x = torch.randn(T, M, device=dev).bfloat16()
    dy = torch.randn(T, N, device=dev).bfloat16()
    grad = torch.zeros(M, N, device=dev)
    p, m, v = torch.randn(M * N, device=dev), torch.zeros(M * N, device=dev), torch.zeros(M * N, device=dev)
    bf = torch.empty(M * N, device=dev, dtype=torch.bfloat16)

    def plain():
        ops.gemm(x, dy, grad, trans_a=True, accumulate=True)

    def fused():
        _lib.call("cb_gemm_adamw", M, N, T, ops.dt(x), x.data_ptr(), M, 1, dy.data_ptr(), N, 0, grad.data_ptr(), N,
                  1.0, p.data_ptr(), m.data_ptr(), v.data_ptr(), None, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1, ops.stream_ptr())

    def adam():
        ops.adamw(p, grad.view(-1), m, v, bf, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1)

    tp, tf, ta = timeit(plain), timeit(fused), timeit(adam)
    fl = 2 * M * N * T
    print(f"{name:5s} M={M} N={N} K={T}: gemm {tp:.3f} ms ({fl / tp / 1e9:.0f} TF/s), gemm+adamw epilogue {tf:.3f} ms, "
          f"adamw kernel {ta:.3f} ms -> fused saves {tp + ta - tf:+.3f} ms", flush=True)
