"""Runs the attention kernels twice at a step shape (1b | 7b | 70b; for ncu captures)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import ops

SHAPES = {"1b": (8, 4096, 16, 16, 128), "7b": (2, 4096, 32, 32, 128), "70b": (1, 4096, 64, 8, 128)}
B, T, H, KVH, hd = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "1b"]
d, kvd = H * hd, KVH * hd
dev = torch.device("cuda")
qkv = torch.randn(B * T, d + 2 * kvd, device=dev).bfloat16()
q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
do = torch.randn(B * T, d, device=dev).bfloat16()
dqkv = torch.empty_like(qkv)
scale = 1 / math.sqrt(hd)
for _ in range(2):
    o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
    ops.attention_bwd(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
torch.cuda.synchronize()
print("ok")
