"""Diagnostic only (never a bench number): the in-step cost of AdamW on one GPU — the 7B step
timed as is, then with ops.adamw replaced by a no-op (the update skipped), interleaved."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, ops, synthetic_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = TrainEngine(BENCH_CONFIGS["7b"](batch=B, dtype="bf16"), device="cuda:0")
toks = [eng.upload_tokens(synthetic_batch(0, s, B, 4096, 32000)["tokens"]) for s in range(4)]
real = ops.adamw


def timed(k=6):
    for s in range(2):
        eng.step(toks[s % 4])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(k):
        eng.step(toks[s % 4])
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


for rep in range(2):
    ops.adamw = real
    t1 = timed()
    ops.adamw = lambda *a, **k: None
    t0 = timed()
    print(f"B={B} rep {rep}: step {t1:.1f} ms, without AdamW {t0:.1f} ms, AdamW costs {t1 - t0:.1f} ms "
          f"({100 * (t1 - t0) / t1:.1f}%)", flush=True)
ops.adamw = real
