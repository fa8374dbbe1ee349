"""Loss trajectory of the 7B-shaped step (diagnostic): full depth at 2 and 3 sequences, and at
8 layers with the one-GPU gradient ring forced on and off (must be bit-identical)."""
import gc
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, synthetic_batch  # noqa: E402


def run(B, layers, ring, steps=5, same_batch=True):
    os.environ["CB_GRAD_RING"] = ring
    gc.collect()
    torch.cuda.empty_cache()
    eng = TrainEngine(BENCH_CONFIGS["7b"](batch=B, layers=layers, dtype="bf16"), device="cuda:0")
    out = []
    for s in range(steps):
        toks = synthetic_batch(0, 0 if same_batch else s, B, 4096, 32000)["tokens"]
        out.append(float(eng.step(toks)[0].item()))
    r = eng._grad_ring
    del eng
    torch.cuda.empty_cache()
    return out, r


for B, layers, ring in [(3, 8, "0"), (3, 8, "1"), (2, 32, "auto"), (3, 32, "auto")]:
    losses, r = run(B, layers, ring)
    print(json.dumps({"B": B, "layers": layers, "ring": r, "losses": losses}), flush=True)
losses, r = run(3, 32, "auto", steps=5, same_batch=False)
print(json.dumps({"B": 3, "layers": 32, "ring": r, "fresh_batches": True, "losses": losses}), flush=True)
