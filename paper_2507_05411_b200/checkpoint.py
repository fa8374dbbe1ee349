"""Sharded checkpoint save / restore of a TrainEngine.

The reference only *simulates* checkpointing (reference runtime_sim.py:22-157): a manifest
of shards, a plan that assigns every shard to exactly one saving replica (replicated shards
round-robin, owned shards by their owner), a bounded-concurrency save, and a retention
policy.  This module runs that plan for real on the engine's state:

* shards are the engine's flat parameter buckets: for an FSDP-sharded bucket, each rank
  owns its slice of the f32 master copy and of the AdamW m / v (non-replicated shards);
  replicated buckets (norm scales, MoE router) are replicated shards spread round-robin;
* every rank writes the shards the plan gives it, with at most ``concurrency_bound`` shards
  staged in pinned host memory at once (device->host copy on a side stream, file write on a
  worker thread);
* rank 0 writes ``manifest.json`` (layout, world size, optimizer step) last, so a directory
  without it is an incomplete checkpoint;
* restore reads the same layout at any world size (a bucket saved by N ranks is
  reassembled and re-sliced for M ranks), rebuilds the bf16 working copy and the step count;
* ``GcPolicy`` / ``gc_retained`` decide which step directories survive.

The planning / retention functions restate reference runtime_sim.py:22-79 and :134-157.
"""

from __future__ import annotations

import json
import os
import shutil
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

FORMAT = "composer_b200.ckpt.v1"


# --------------------------------------------------------------------- planning
@dataclass(frozen=True)
class Shard:
    """One saveable piece of state (reference runtime_sim.py:25-36): replicated shards exist
    on every rank; the others only on ``owner``."""

    name: str
    nbytes: int
    replicated: bool = True
    owner: int = 0


@dataclass(frozen=True)
class ShardManifest:
    """reference runtime_sim.py:39-62 (same validation)."""

    shards: tuple[Shard, ...]
    replicas: int = 1

    def __post_init__(self):
        if self.replicas < 1:
            raise ValueError(f"replicas must be >= 1, got {self.replicas}")
        names = set()
        for sh in self.shards:
            if sh.nbytes <= 0:
                raise ValueError(f"shard {sh.name!r} has non-positive bytes")
            if sh.name in names:
                raise ValueError(f"duplicate shard name {sh.name!r}")
            names.add(sh.name)
            if not 0 <= sh.owner < self.replicas:
                raise ValueError(f"shard {sh.name!r} owner {sh.owner} outside [0, {self.replicas})")

    @property
    def total_bytes(self) -> int:
        return sum(sh.nbytes for sh in self.shards)


def plan_checkpoint(manifest: ShardManifest) -> dict[int, list[Shard]]:
    """Exact partition of the shards over the saving ranks (reference runtime_sim.py:65-79):
    replicated shards round-robin over the replicas in manifest order, owned shards to their
    owner."""
    plan: dict[int, list[Shard]] = {r: [] for r in range(manifest.replicas)}
    rr = 0
    for sh in manifest.shards:
        if sh.replicated and manifest.replicas > 1:
            plan[rr % manifest.replicas].append(sh)
            rr += 1
        else:
            plan[sh.owner].append(sh)
    return plan


@dataclass(frozen=True)
class GcPolicy:
    """Which checkpoint steps survive (reference runtime_sim.py:134-144)."""

    keep_last_n: int = 0
    keep_every_k: int = 0

    def __post_init__(self):
        if self.keep_last_n < 0 or self.keep_every_k < 0:
            raise ValueError("retention counts must be >= 0")
        if self.keep_last_n == 0 and self.keep_every_k == 0:
            raise ValueError("at least one retention criterion must be enabled")


def gc_retained(checkpoint_steps: Sequence[int], policy: GcPolicy) -> set[int]:
    """The newest keep_last_n steps plus every multiple of keep_every_k
    (reference runtime_sim.py:147-157)."""
    steps = list(checkpoint_steps)
    if steps != sorted(steps):
        raise ValueError("checkpoint steps must be sorted ascending")
    keep: set[int] = set()
    if policy.keep_last_n:
        keep.update(steps[-policy.keep_last_n:])
    if policy.keep_every_k:
        keep.update(s for s in steps if s % policy.keep_every_k == 0)
    return keep


# ---------------------------------------------------------------- engine state
_PARTS = ("master", "m", "v")


def _shard_name(bucket: int, part: str, rank: int | None) -> str:
    return f"b{bucket:03d}.{part}" if rank is None else f"b{bucket:03d}.{part}.r{rank}"


def engine_manifest(eng) -> ShardManifest:
    """The engine's state as a shard manifest: per bucket and per optimizer part, one
    replicated shard (replicated buckets) or one shard per rank (FSDP-sharded buckets)."""
    shards = []
    for i, (b, rec) in enumerate(zip(eng.buckets, eng.bufs)):
        for part in _PARTS:
            if b.replicated or eng.d.world == 1:
                shards.append(Shard(_shard_name(i, part, None), 4 * rec["total"], replicated=True))
            else:
                for r in range(eng.d.world):
                    shards.append(Shard(_shard_name(i, part, r), 4 * rec["shard"], replicated=False, owner=r))
    return ShardManifest(tuple(shards), replicas=eng.d.world)


def _layout(eng) -> list[dict]:
    return [{"numel": int(b.numel), "total": int(rec["total"]), "shard": int(rec["shard"]),
             "replicated": bool(b.replicated),
             "entries": [[e.path, e.name, list(e.shape)] for e in b.entries]}
            for b, rec in zip(eng.buckets, eng.bufs)]


def _barrier(eng):
    if eng.d.world > 1:
        eng.d.dist.barrier(group=eng.d.group)


def step_dir(root: str, step: int) -> str:
    return os.path.join(root, f"step_{step:08d}")


def list_steps(root: str) -> list[int]:
    """Complete checkpoints under root (those whose manifest was written), ascending."""
    out = []
    if os.path.isdir(root):
        for name in os.listdir(root):
            if name.startswith("step_") and os.path.exists(os.path.join(root, name, "manifest.json")):
                out.append(int(name[5:]))
    return sorted(out)


def save_checkpoint(eng, root: str, step: int | None = None, concurrency_bound: int = 4,
                    gc: GcPolicy | None = None) -> dict:
    """Writes this rank's share of the checkpoint plan; returns a report (bytes written by
    this rank, peak staged host bytes, shard count)."""
    import torch

    if concurrency_bound < 1:
        raise ValueError(f"concurrency bound must be >= 1, got {concurrency_bound}")
    step = eng.step_count if step is None else int(step)
    d = step_dir(root, step)
    if eng.d.rank == 0:
        os.makedirs(d, exist_ok=True)
    _barrier(eng)
    manifest = engine_manifest(eng)
    mine = plan_checkpoint(manifest)[eng.d.rank]
    torch.cuda.synchronize(eng.device)

    def source(sh: Shard):
        # this rank's master / m / v of the bucket: the whole bucket when it is replicated
        # (or world == 1), else exactly the rank's shard the plan assigned to it
        i, part = int(sh.name[1:4]), sh.name.split(".")[1]
        return eng.bufs[i][part]

    stream = torch.cuda.Stream(device=eng.device)
    slots = threading.BoundedSemaphore(concurrency_bound)
    lock = threading.Lock()
    stats = {"staged": 0, "peak": 0, "bytes": 0}

    def write(sh: Shard):
        try:
            src = source(sh)
            host = torch.empty(src.numel(), dtype=torch.float32, pin_memory=True)
            with torch.cuda.stream(stream):
                host.copy_(src, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            ev.synchronize()
            host.numpy().tofile(os.path.join(d, sh.name + ".bin"))
            with lock:
                stats["bytes"] += sh.nbytes
                stats["staged"] -= sh.nbytes
        finally:
            slots.release()

    with ThreadPoolExecutor(max_workers=concurrency_bound) as pool:
        futs = []
        for sh in mine:
            slots.acquire()  # at most `concurrency_bound` shards staged on the host at once
            with lock:
                stats["staged"] += sh.nbytes
                stats["peak"] = max(stats["peak"], stats["staged"])
            futs.append(pool.submit(write, sh))
        for f in futs:
            f.result()
    _barrier(eng)
    if eng.d.rank == 0:
        meta = {"format": FORMAT, "step": step, "world": eng.d.world, "precision": eng.precision,
                "buckets": _layout(eng), "shards": [[s.name, s.nbytes, s.replicated, s.owner] for s in manifest.shards]}
        tmp = os.path.join(d, "manifest.json.tmp")
        with open(tmp, "w") as fh:
            json.dump(meta, fh)
        os.replace(tmp, os.path.join(d, "manifest.json"))
        if gc is not None:
            keep = gc_retained(list_steps(root), gc)
            for s in list_steps(root):
                if s not in keep:
                    shutil.rmtree(step_dir(root, s), ignore_errors=True)
    _barrier(eng)
    return {"step": step, "bytes": stats["bytes"], "peak_host_bytes": stats["peak"], "num_shards": len(mine)}


def load_checkpoint(eng, root: str, step: int | None = None) -> int:
    """Restores master / m / v, the bf16 working copy and the optimizer step from a complete
    checkpoint (the newest one when step is None), at this engine's world size."""
    import torch

    from .errors import ShapeError

    steps = list_steps(root)
    if not steps:
        raise FileNotFoundError(f"no complete checkpoint under {root}")
    step = steps[-1] if step is None else int(step)
    d = step_dir(root, step)
    with open(os.path.join(d, "manifest.json")) as fh:
        meta = json.load(fh)
    if meta.get("format") != FORMAT:
        raise ShapeError(f"{d}: not a {FORMAT} checkpoint")
    saved, layout = meta["buckets"], _layout(eng)
    if [(b["numel"], b["replicated"], b["entries"]) for b in saved] != \
            [(b["numel"], b["replicated"], b["entries"]) for b in layout]:
        raise ShapeError(f"{d}: parameter layout differs from this model's")
    world_saved = int(meta["world"])
    for i, (b, rec) in enumerate(zip(eng.buckets, eng.bufs)):
        for part in _PARTS:
            sb = saved[i]
            if sb["replicated"] or world_saved == 1:
                full = np.fromfile(os.path.join(d, _shard_name(i, part, None) + ".bin"), dtype=np.float32)
            else:
                full = np.concatenate([np.fromfile(os.path.join(d, _shard_name(i, part, r) + ".bin"), dtype=np.float32)
                                       for r in range(world_saved)])
            vals = np.zeros(rec["total"], dtype=np.float32)
            vals[:b.numel] = full[:b.numel]
            r0 = 0 if b.replicated else eng.d.rank * rec["shard"]
            dst = rec["master"] if part == "master" else rec[part]
            dst.copy_(torch.from_numpy(vals[r0:r0 + rec["shard"]]).to(eng.device))
        eng._refresh_work(i)  # own working-copy slice; peers' slices are gathered by the next step
    eng.step_count = int(meta["step"])
    torch.cuda.synchronize(eng.device)
    _barrier(eng)
    return eng.step_count
