"""Attention backward at a step shape under steady-state (power-capped) clocks: a GEMM loop
heats the GPU first, then N backward calls (the RoPE variant the step uses) run back to back;
kernel durations from CUPTI, SM clock sampled by nvidia-smi during the run.

    python scripts/attn_steady.py [1b|7b|70b] [iters]
"""
import json
import math
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import ops  # noqa: E402
from paper_2507_05411_b200.layers import rope_tables  # noqa: E402

SHAPES = {"1b": (8, 4096, 16, 16, 128), "7b": (2, 4096, 32, 32, 128), "70b": (2, 4096, 64, 8, 128)}
name = sys.argv[1] if len(sys.argv) > 1 else "7b"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
B, T, H, KVH, hd = SHAPES[name]
dev = torch.device("cuda")
d, kvd = H * hd, KVH * hd
qkv = (0.5 * torch.randn(B * T, d + 2 * kvd, device=dev)).bfloat16()
q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
do = torch.randn(B * T, d, device=dev).bfloat16()
dqkv = torch.empty_like(qkv)
cs, sn = rope_tables(T, hd, 10000.0, dev)
scale = 1 / math.sqrt(hd)
o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
a = torch.randn(8192, 8192, device=dev).bfloat16()
c = torch.empty(8192, 8192, device=dev)
for _ in range(200):  # ~3 s of GEMMs: clocks settle under the power cap
    ops.gemm(a, a, c)
torch.cuda.synchronize()
fd, path = tempfile.mkstemp()
os.close(fd)
smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "100"], stdout=open(path, "w"))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(iters):
        ops.attention_bwd_rope(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H,
                               KVH, hd, scale, cs, sn, o_lo=o_lo)
    torch.cuda.synchronize()
smi.terminate()
smi.wait()
clk = [float(x.split(",")[0]) for x in open(path) if x.strip()]
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        kname = e.name.split("(")[0].split("<")[0].split("::")[-1]
        t = tot.setdefault(kname, [0, 0.0])
        t[0] += 1
        t[1] += e.time_range.elapsed_us()
flops = 8 * B * T * T * H * hd
per = {k: round(v[1] / v[0], 1) for k, v in tot.items()}
total_us = sum(v[1] for v in tot.values()) / iters
print(json.dumps({"shape": name, "iters": iters, "us_per_call": per, "bwd_us": round(total_us, 1),
                  "tflops_alg": round(flops / total_us / 1e6, 1),
                  "sm_mhz_median": sorted(clk)[len(clk) // 2] if clk else None}))
