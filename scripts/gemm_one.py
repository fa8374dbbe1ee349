"""One step-shaped CTA-pair GEMM launch (after a warm-up launch), for ncu --set full captures.

    python scripts/gemm_one.py [qkv7b|qkv7b3|o7b|up7b|down7b|qkv1b]   (qkv7b3: 3 sequences per GPU)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import _lib, ops  # noqa: E402

if "CB_GEMM_RASTER" in os.environ:
    _lib.call("cb_gemm_set_raster", int(os.environ["CB_GEMM_RASTER"]))

# (M, N, K, out dtype): x[tokens, d] @ W[d, n] as the 7B / 1B steps issue them
SHAPES = {"qkv7b": (8192, 12288, 4096, torch.bfloat16), "qkv7b3": (12288, 12288, 4096, torch.bfloat16), "o7b": (8192, 4096, 4096, torch.float32),
          "up7b": (8192, 22016, 4096, torch.bfloat16), "down7b": (8192, 4096, 11008, torch.float32),
          "qkv1b": (32768, 6144, 2048, torch.bfloat16)}
M, N, K, odt = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "qkv7b"]
dev = torch.device("cuda")
a = torch.randn(M, K, device=dev).bfloat16()
b = (0.02 * torch.randn(K, N, device=dev)).bfloat16()
c = torch.empty(M, N, device=dev, dtype=odt)
for _ in range(2):
    ops.gemm(a, b, c)
torch.cuda.synchronize()
print("algorithmic bytes", 2 * M * K + 2 * K * N + c.element_size() * M * N, "flops", 2 * M * N * K)
