"""dQ sweep: single-CTA (dq_k) vs CTA pairs (dq_pair_k) at the 1B / 7B / 70B-layer attention
shapes, whole attention backward timed with CUDA events (the dK/dV sweep is the same)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import ops  # noqa: E402

dev = torch.device("cuda")
for (B, T, H, KVH) in [(8, 4096, 16, 16), (3, 4096, 32, 32), (2, 4096, 64, 8)]:
    hd = 128
    d, kvd = H * hd, KVH * hd
    qkv = torch.randn(B * T, d + 2 * kvd, device=dev).bfloat16()
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    do = torch.randn(B * T, d, device=dev).bfloat16()
    scale = 1 / math.sqrt(hd)
    o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
    dqkv = torch.empty_like(qkv)
    args = (q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
    flops = 8 * B * T * T * H * hd
    res = {}
    for rep in range(6):
        for pair in ((0, 1, 2) if rep % 2 == 0 else (2, 1, 0)):  # 0 single, 1 pair dQ, 2 pair dQ + dK/dV
            ops.set_dq_pair(pair >= 1)
            ops.set_dkdv_pair(pair >= 2)
            for _ in range(2):
                ops.attention_bwd(*args, o_lo=o_lo)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                ops.attention_bwd(*args, o_lo=o_lo)
            e.record()
            torch.cuda.synchronize()
            res.setdefault(pair, []).append(s.elapsed_time(e) / 10)
    ops.set_dq_pair(True)
    ops.set_dkdv_pair(False)
    import statistics

    t0, t1, t2 = statistics.median(res[0]), statistics.median(res[1]), statistics.median(res[2])
    print(f"B={B} T={T} H={H} KVH={KVH}: backward single {t0:.3f} ms ({flops / t0 / 1e9:.0f} TF/s), "
          f"pair dQ {t1:.3f} ms ({flops / t1 / 1e9:.0f} TF/s), {100 * (t0 - t1) / t0:+.1f}% (medians of 6, "
          f"alternating order; min {min(res[0]):.3f} / {min(res[1]):.3f}); pair dQ + dK/dV {t2:.3f} ms "
          f"({flops / t2 / 1e9:.0f} TF/s), {100 * (t0 - t2) / t0:+.1f}%", flush=True)
