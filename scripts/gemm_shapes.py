"""Times every GEMM shape of one 1B (default) or 7B decoder layer (forward, dgrad, wgrad) on the
default engine: TFLOP/s per shape, with and without the split-K workspace (interleaved, same
box).   python scripts/gemm_shapes.py [--7b] [shape names...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import _lib, ops

dev = torch.device("cuda")
T, d, qkv, ffn = (12288, 4096, 12288, 11008) if "--7b" in sys.argv else (32768, 2048, 6144, 5632)
# (name, M, N, K, trans_a, trans_b, out f32, accumulate)
shapes = [
    ("fwd_qkv", T, qkv, d, 0, 0, 0, 0), ("fwd_o", T, d, d, 0, 0, 1, 0), ("fwd_up", T, 2 * ffn, d, 0, 0, 0, 0),
    ("fwd_down", T, d, ffn, 0, 0, 1, 0), ("head", T, 32000, d, 0, 1, 1, 0),
    ("dgrad_qkv", T, d, qkv, 0, 1, 1, 0), ("dgrad_o", T, d, d, 0, 1, 0, 0), ("dgrad_up", T, d, 2 * ffn, 0, 1, 1, 0),
    ("dgrad_down", T, ffn, d, 0, 1, 0, 0),
    ("wgrad_qkv", d, qkv, T, 1, 0, 1, 1), ("wgrad_o", d, d, T, 1, 0, 1, 1), ("wgrad_up", d, 2 * ffn, T, 1, 0, 1, 1),
    ("wgrad_down", ffn, d, T, 1, 0, 1, 1), ("head_wgrad", 32000, d, T, 1, 0, 1, 1), ("head_dgrad", T, d, 32000, 0, 0, 1, 0),
]
only = [a for a in sys.argv[1:] if not a.startswith("--")]
ws = torch.empty((256 << 20) // 4, device=dev)


def timed(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


for name, M, N, K, ta, tb, f32, acc in shapes:
    if only and name not in only:
        continue
    a = torch.randn((K, M) if ta else (M, K), device=dev).bfloat16()
    b = torch.randn((N, K) if tb else (K, N), device=dev).bfloat16()
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    fn = lambda: ops.gemm(a, b, out, trans_a=bool(ta), trans_b=bool(tb), accumulate=bool(acc))  # noqa: E731
    res = {"gemm": name, "M": M, "N": N, "K": K, "units": ((M + 255) // 256) * ((N + 255) // 256)}
    for rep in range(2):
        for mode in ("plain", "splitk"):
            _lib.call("cb_gemm_set_workspace", ws.data_ptr() if mode == "splitk" else None, ws.numel() * 4 if mode == "splitk" else 0)
            ms = timed(fn)
            res[f"{mode}_tflops_{rep}"] = round(2 * M * N * K / ms / 1e9, 1)
    print(json.dumps(res), flush=True)
    del a, b, out
