"""Stress test of the attention backward sweeps (CTA-pair variants): thousands of back-to-back
backward passes per shape, every result compared bit for bit with the first (a race between
cluster barrier phases shows up as a mismatch or a hang — run under `timeout`).

    timeout 600 python scripts/attn_stress.py [iterations] [dkdv_pair 0/1]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import ops  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ops.set_dq_pair(True)
ops.set_dkdv_pair(len(sys.argv) > 2 and sys.argv[2] == "1")
dev = torch.device("cuda")
for (B, T, H, KVH) in [(1, 512, 4, 4), (2, 1024, 8, 2), (3, 4096, 32, 32)]:
    hd = 128
    d, kvd = H * hd, KVH * hd
    g = torch.Generator().manual_seed(T + H)
    qkv = torch.randn(B * T, d + 2 * kvd, generator=g).to(dev, torch.bfloat16)
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    do = torch.randn(B * T, d, generator=g).to(dev, torch.bfloat16)
    scale = 1 / math.sqrt(hd)
    o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
    ref = torch.empty_like(qkv)
    out = torch.empty_like(qkv)

    def bwd(dst):
        ops.attention_bwd(q, k, v, o, lse, do, dst[:, :d], dst[:, d:d + kvd], dst[:, d + kvd:], B, T, H, KVH, hd,
                          scale, o_lo=o_lo)

    bwd(ref)
    n = iters if T <= 1024 else max(20, iters // 20)
    bad = 0
    for i in range(n):
        bwd(out)
        if i % 25 == 24 or i == n - 1:
            torch.cuda.synchronize()
            bad += int(not torch.equal(out, ref))
    torch.cuda.synchronize()
    print(f"B={B} T={T} H={H} KVH={KVH}: {n} backward passes, {bad} mismatching checks", flush=True)
print("done", flush=True)
