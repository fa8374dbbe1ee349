"""Times the attention kernels at the 1B / 7B step shapes (CUDA events)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import _lib, ops

dev = torch.device("cuda")
for (B, T, H, KVH, hd) in [(8, 4096, 16, 16, 128), (2, 4096, 32, 32, 128), (1, 4096, 64, 8, 128)]:
    d, kvd = H * hd, KVH * hd
    qkv = torch.randn(B * T, d + 2 * kvd, device=dev).bfloat16()
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    do = torch.randn(B * T, d, device=dev).bfloat16()
    dqkv = torch.empty_like(qkv)
    scale = 1 / math.sqrt(hd)
    flops = 4 * B * T * T * H * hd
    res = {"B": B, "T": T, "H": H, "KVH": KVH}
    for tc in (1, 0):
        _lib.call("cb_attention_set_tc", tc)
        for _ in range(2):
            o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        res[f"fwd_{'tc' if tc else 'mma'}_ms"] = round(ms, 3)
        res[f"fwd_{'tc' if tc else 'mma'}_tflops"] = round(flops / ms / 1e9, 1)
    _lib.call("cb_attention_set_tc", 1)
    o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
    for _ in range(2):
        ops.attention_bwd(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        ops.attention_bwd(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    res["bwd_ms"] = round(ms, 3)
    res["bwd_tflops_alg"] = round(2 * flops / ms / 1e9, 1)
    print(json.dumps(res), flush=True)
