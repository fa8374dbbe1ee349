"""Times the fused softmax cross-entropy (loss + dlogits in one pass) on the 1B head shape:
f32 logits [8*4096, 32000] in, bf16 dlogits out; reports achieved HBM GB/s (6 B/element)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import ops

dev = torch.device("cuda")
B, T, V = 8, 4096, 32000
logits = torch.randn(B * T, V, device=dev) * 3
tokens = torch.randint(0, V, (B, T), device=dev)
dl = torch.empty(B * T, V, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    ops.xent(logits, tokens, dl, 1.0 / (B * (T - 1)))
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
s.record()
for _ in range(n):
    ops.xent(logits, tokens, dl, 1.0 / (B * (T - 1)))
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"xent {ms:.3f} ms  {B * T * V * 6 / ms / 1e6:.0f} GB/s")
