"""Runs warm-up steps, then exactly one training step inside cudaProfilerStart/Stop, so
`ncu --profile-from-start off` captures the launches of one step.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python scripts/step_once.py --config 1b
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, synthetic_batch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1b")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--seq", type=int, default=None)
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
kw = {k: v for k, v in (("batch", args.batch), ("seq", args.seq)) if v is not None}
cfg = BENCH_CONFIGS[args.config](dtype="bf16", **kw)
eng = TrainEngine(cfg, device=dev)
V = eng.cfg.get("model.vocab_size")
B = args.batch or BENCH_CONFIGS[args.config].__defaults__[0]
T = args.seq or BENCH_CONFIGS[args.config].__defaults__[1]
toks = [eng.upload_tokens(synthetic_batch(0, s, B, T, V)["tokens"]) for s in range(args.warmup + 1)]
for s in range(args.warmup):
    eng.step(toks[s])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
loss, _ = eng.step(toks[args.warmup])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("loss", float(loss.item()))
