"""GPU idle gaps inside training steps: runs warm-up steps, then N steps under torch.profiler
(CUPTI kernel activity) and reports busy time vs span and the largest gaps between
consecutive kernels on the compute stream (with the kernel before each gap).

    python scripts/gap_profile.py --config moe --steps 2
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/gap_profile.py --config 1b
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, synthetic_batch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1b")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--batch", type=int, default=None)
args = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:  # under torchrun: FSDP over the ranks, rank 0 reports
    import torch.distributed as dist

    dist.init_process_group("nccl", device_id=dev)
B, T = args.batch or BENCH_CONFIGS[args.config].__defaults__[0], BENCH_CONFIGS[args.config].__defaults__[1]
cfg = BENCH_CONFIGS[args.config](batch=B, dtype="bf16")
eng = TrainEngine(cfg, device=dev)
V = eng.cfg.get("model.vocab_size")
toks = [eng.upload_tokens(synthetic_batch(0, s, B, T, V)["tokens"]) for s in range(3 + args.steps)]
for s in range(3):
    eng.step(toks[s])
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for s in range(args.steps):
        eng.step(toks[3 + s])
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
       and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
by_stream = {}
for e in evs:
    by_stream.setdefault(getattr(e, "device_index", 0), []).append(e)
evs.sort(key=lambda e: e.time_range.start)
t0, t1 = evs[0].time_range.start, max(e.time_range.end for e in evs)
# union of busy intervals over all streams
busy, cur_s, cur_e = 0.0, None, None
for e in evs:
    s, en = e.time_range.start, e.time_range.end
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, en
    else:
        cur_e = max(cur_e, en)
busy += cur_e - cur_s
print(f"rank {rank} {args.config}: {args.steps} steps, span {(t1 - t0) / 1e3:.2f} ms, GPU busy {busy / 1e3:.2f} ms "
      f"({100 * busy / (t1 - t0):.1f}%), {len(evs)} kernels")
gaps = []
end = evs[0].time_range.end
prev = evs[0]
for e in evs[1:]:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, prev.name[:60], e.name[:60]))
    if e.time_range.end > end:
        end, prev = e.time_range.end, e
gaps.sort(reverse=True)
print(f"rank {rank} idle total {sum(g[0] for g in gaps) / 1e3:.2f} ms in {len(gaps)} gaps; largest:")
for g, a, b in gaps[:15 if rank == 0 else 5]:
    print(f"  {g:8.1f} us  after {a}  before {b}")
