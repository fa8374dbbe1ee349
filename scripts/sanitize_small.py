"""One launch of each hot kernel at a tiny shape, for compute-sanitizer (racecheck / synccheck /
memcheck): the CTA-pair tcgen05 GEMM (plain, RoPE and gated epilogues, f32 accumulate), the
tcgen05 flash attention forward / backward, RMSNorm, cross-entropy and AdamW.

    compute-sanitizer --tool racecheck python scripts/sanitize_small.py
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import ops  # noqa: E402
from paper_2507_05411_b200.layers import rope_tables  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device="cpu").manual_seed(0)


def rnd(*shape, dt=torch.bfloat16, s=1.0):
    return (s * torch.randn(*shape, generator=g)).to(dev, dt)


M, N, K = 512, 512, 256
a, b = rnd(M, K), rnd(K, N, s=0.05)
c = torch.empty(M, N, device=dev, dtype=torch.float32)
ops.gemm(a, b, c)                                   # CTA-pair GEMM, f32 out
cb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
ops.gemm(a, b, cb)                                  # bf16 out (staged epilogue)
ops.gemm(a, rnd(M, N), torch.zeros(K, N, device=dev), trans_a=True, accumulate=True)  # wgrad form
B, T, H, hd = 2, 256, 2, 128
d = H * hd
x = rnd(B * T, d)
w = rnd(d, 3 * d, s=0.05)
qkv = torch.empty(B * T, 3 * d, device=dev, dtype=torch.bfloat16)
cs, sn = rope_tables(T, hd, 10000.0, dev)
ops.gemm_rope(x, w, qkv, T, hd, 2 * d, cs, sn)      # RoPE epilogue
wg = rnd(d, 2 * 768, s=0.05)
ops.gemm_gated_fwd(x, wg, "linear", "silu")          # gated epilogue
q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
o, lse = ops.attention_fwd(q, k, v, B, T, H, H, hd, 1 / math.sqrt(hd))
do = rnd(B * T, d)
dqkv = torch.empty_like(qkv)
ops.attention_bwd_rope(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:2 * d], dqkv[:, 2 * d:], B, T, H, H, hd,
                       1 / math.sqrt(hd), cs, sn)
xs = rnd(B * T, d, dt=torch.float32)
sc = torch.ones(d, device=dev)
y, rstd = ops.rmsnorm_fwd(xs, sc, 1e-6, torch.bfloat16)
ops.rmsnorm_bwd(xs, sc, rstd, rnd(B * T, d), dscale=torch.zeros(d, device=dev))
logits = rnd(B * T, 512, dt=torch.float32)
toks = torch.randint(0, 512, (B, T), device=dev)
ops.xent(logits, toks, torch.empty_like(logits), 1.0 / (B * T))
p = rnd(4096, dt=torch.float32)
ops.adamw(p, rnd(4096, dt=torch.float32), torch.zeros_like(p), torch.zeros_like(p), None, 1e-3, 0.9, 0.999, 1e-8,
          0.0, 1)
torch.cuda.synchronize()
print("sanitize_small ok")
