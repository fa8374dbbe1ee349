#!/usr/bin/env python
"""Benchmark of the decoder training step (BASELINE.json metric: train tokens/s + MFU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7b] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); every rank runs the same
per-GPU batch (weak scaling) with FSDP-sharded state.  One step = forward + backward +
AdamW over one synthetic batch of [batch, seq] tokens.  Timing: W warm-up
steps, then K steps bracketed by barrier + synchronize, CUDA events on the compute
stream, max over ranks.  Rank 0 prints one JSON line.

The default workload is BASELINE.json configs[2], the Llama2-7B-shaped step (the
north-star config; 3 x 4096 tokens per GPU — the largest per-GPU batch that fits in HBM
with the one-GPU gradient ring); --config 1b selects configs[1].

--impl reference times the REFERENCE's own CPU step — ``composer.invoke`` (forward +
loss; the reference has no backward or optimizer) of the unmodified reference installed
in oracle/_ref (oracle/build_ref.sh) — on this host's cores, on a bounded sample of the
same workload (one TransformerLayer + the head at batch 1, seq 4096, extrapolated in
depth; oracle/ref_step.py), and prints the same JSON line with "impl": "reference".  When
oracle/_ref is missing it times the oracle/ float64 port (fwd+bwd+AdamW) instead and says
so in cpu_baseline.kind ("port").

Kernel attribution: the profiled steps run under CUPTI kernel activity (torch.profiler),
which sees every stream; each kernel's duration is split evenly with the kernels that
overlap it in time, so the per-kind attributed milliseconds sum to the GPU-busy time of
the step (never more than ms_per_step).  roofline.achieved uses the GEMM launches' own
CUPTI durations (algorithmic FLOPs / summed launch time).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

NOMINAL_BF16_PFLOPS = 2.25e15
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh), "measured"
    return dict(FALLBACK_PEAKS), "fallback"


def flops_per_token(module, batch, seq) -> float:
    """3 x sum of the reference's own_flops (reference mesh.py:629,644) per token."""
    total = 0
    for _, m in module.walk():
        total += m.behavior.own_flops(m.config, batch, seq)
    return 3.0 * total / (batch * seq)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        loaded = [s for s in sms if mx and s > 0.3 * mx] or sms
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# --------------------------------------------------------------------------- CPU leg
def cpu_sample(config: str, seconds_hint: float = 20.0) -> dict:
    """Times the oracle (float64 fwd+bwd+AdamW) on a bounded sample of `config`.

    Sample: the config's layer shape at 1 and 2 layers, batch 1, seq 256, full vocab;
    per-token time extrapolated linearly in depth to the configured layer count.
    """
    import torch

    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import BENCH_CONFIGS, init_state, instantiate, root_key, synthetic_batch

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    seq = 256
    full = BENCH_CONFIGS[config](batch=1, seq=seq, dtype="f32")
    L = len(full.get("model.decoder.transformer.layer"))
    times = {}
    for nl in (1, 2):
        cfg = BENCH_CONFIGS[config](batch=1, seq=seq, dtype="f32", layers=nl)
        m = instantiate(cfg)
        st = init_state(m, root_key(0))
        spec = O.spec_from_config(m.config)
        toks = synthetic_batch(0, 0, 1, seq, cfg.get("model.vocab_size"))["tokens"]
        t0 = time.perf_counter()
        O.train_step(st, toks, spec, O.AdamW(lr=1e-3))
        times[nl] = time.perf_counter() - t0
    per_layer = max(times[2] - times[1], 1e-9)
    fixed = max(times[1] - per_layer, 0.0)
    t_full = fixed + L * per_layer
    return {"value": seq / t_full, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"oracle/ float64 fwd+bwd+AdamW of the {config} layer shape at 1 and 2 layers, batch 1, seq {seq}, "
                      f"vocab {full.get('model.vocab_size')}; {times[1]:.2f}s/{times[2]:.2f}s, extrapolated linearly "
                      f"to {L} layers ({t_full:.1f} s per {seq}-token step)"}


def reference_sample(config: str) -> dict:
    """One bounded sample of the reference's own CPU step (oracle/ref_step.py), or of the
    oracle port when the reference is not installed in oracle/_ref."""
    from oracle import ref_step

    if not ref_step.available():
        out = cpu_sample(config)
        out["sample"] = "oracle/_ref missing: " + out["sample"]
        return out
    threads = os.cpu_count() or 1
    out = ref_step.reference_sample(config)
    return {"value": out["value"], "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": out["sample"] + f"; numpy/OpenBLAS on {threads} host threads"}


def workload_config(args, world: int) -> dict:
    """The workload description both arms print (the reference arm runs on this arm's config)."""
    from paper_2507_05411_b200 import BENCH_CONFIGS, instantiate
    from paper_2507_05411_b200.module import iter_param_specs

    cfg = BENCH_CONFIGS[args.config](batch=args.batch, seq=args.seq)
    params = sum(int(np.prod(shape)) for _, _, _, shape in iter_param_specs(instantiate(cfg)))
    out = {"workload": args.config, "global_batch": world * args.batch, "per_gpu_batch": args.batch,
           "seq_len": args.seq, "d_model": cfg.get("model.dim"), "layers": len(cfg.get("model.decoder.transformer.layer")),
           "vocab": cfg.get("model.vocab_size"), "params": params, "parallelism": f"fsdp{world}", "remat": args.remat,
           "l2": ("tiny parity-size config: L2-resident, not flushed (not a bench line)" if args.config == "tiny"
                  else "inputs larger than L2 (bf16 params + activations >> 126 MB)")}
    if args.config == "moe":
        out["moe_routing"] = args.moe_routing
    return out


def run_reference(args) -> None:
    """The reference arm: rank 0 alone times the reference's own CPU step on this arm's config.
    A step is one bounded sample of the workload — one reference TransformerLayer invoke at the
    config's layer shape (oracle/ref_step.py; 8.5 s for the 7B layer on 16 threads) — so the
    K timed steps run min(K, 10) samples; the head (embedding, norm, tied head, loss) is timed once with
    the warm-up sample (numpy has no warm-up state: one warm-up sample is run, not W)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref_step

    world = args.gpus
    if not ref_step.available():  # the oracle port, as round 1 (each step one port sample)
        vals = [cpu_sample(args.config) for _ in range(max(1, min(args.steps, 3)))]
        v = statistics.median(x["value"] for x in vals)
        base = {**vals[-1], "value": v, "samples_timed": len(vals)}
        base["sample"] = "oracle/_ref missing: " + base["sample"]
        ms = 1000.0 * args.batch * args.seq / v
    else:
        r = ref_step.ReferenceStep(args.config)
        t_head = r.head()
        r.layer()  # the one warm-up sample
        # at most 10 timed samples (~8 s each at the 7B shape): the arm stays within a few minutes
        # whatever --steps the driver passes
        layers = [r.layer() for _ in range(max(1, min(args.steps, 10)))]
        t_layer = statistics.median(layers)
        v = r.rate(t_head, t_layer)
        ms = 1000.0 * statistics.mean(layers)  # what one timed step (sample) took
        threads = os.cpu_count() or 1
        base = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference",
                "sample": r.describe(t_head, t_layer) + f"; median of {len(layers)} layer samples; numpy/OpenBLAS "
                          f"on {threads} host threads",
                "samples_timed": len(layers), "warmup_samples_run": 1}
    line = {
        "impl": "reference",
        "metric": "train tokens/sec and MFU per B200, decoder step",
        "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "ms_per_step_note": "wall time of one timed sample (a reference TransformerLayer invoke); "
                                               "value extrapolates the sample to the configured depth",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ kernel attribution
_FOREIGN = ("at::", "c10d::", "c10::", "cub::", "cutlass::", "flash", "Memset", "Memcpy")


def kernel_kind(name: str) -> str:
    """Kind of a CUPTI kernel record: this library's kernels by name (most live in namespace
    cb::; a few helpers are at file scope), everything from torch / NCCL / the driver as foreign."""
    n = name
    if "nccl" in n.lower():
        return "foreign (nccl)"
    if any(f in n for f in _FOREIGN):
        return "foreign (torch)"
    if "gemm" in n:
        return "gemm"
    if "tca::" in n or "fa::fwd" in n or "attn_fwd" in n:
        return "attn_fwd"
    if "tcb::" in n or "fa::" in n or "attn" in n:
        return "attn_bwd"
    for key in ("xent", "adamw", "rmsnorm", "embed", "moe", "router", "sum_parts", "init"):
        if key in n:
            return key
    if any(k in n for k in ("pad_rows", "zero_pad", "pad_offsets", "combine", "gather_rows", "sort_ids")):
        return "moe"
    return "other_cb"


def cupti_attribution(fn) -> tuple[dict, float]:
    """Runs fn() under CUPTI kernel activity; returns ({kind: {launches, busy_ms,
    attributed_ms}}, span_ms).  attributed_ms splits every instant evenly among the kernels
    running at that instant (all streams), so Σ attributed_ms = GPU-busy time <= span."""
    import torch

    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    ks = [(e.time_range.start, e.time_range.end, kernel_kind(e.name)) for e in prof.events()
          if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
          and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    out: dict = {}
    if not ks:
        return out, 0.0
    names: dict = {}  # per kind: kernel name -> busy ms (the top three are reported)
    for e in prof.events():
        if (e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
                and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()):
            nm = names.setdefault(kernel_kind(e.name), {})
            key = e.name.split("(")[0][:60]
            nm[key] = nm.get(key, 0.0) + e.time_range.elapsed_us() / 1e3
    for s0, e0, k in ks:
        d = out.setdefault(k, {"launches": 0, "busy_ms": 0.0, "attributed_ms": 0.0})
        d["launches"] += 1
        d["busy_ms"] += (e0 - s0) / 1e3
    for k in out:
        if len(names.get(k, {})) > 1:
            out[k]["top"] = sorted(names[k].items(), key=lambda kv: -kv[1])[:3]
    # sweep line over the start/end points of every kernel (all streams)
    pts = sorted({t for s0, e0, _ in ks for t in (s0, e0)})
    idx = {t: i for i, t in enumerate(pts)}
    kinds = sorted(out)
    delta = {k: [0] * len(pts) for k in kinds}
    for s0, e0, k in ks:
        delta[k][idx[s0]] += 1
        delta[k][idx[e0]] -= 1
    running = {k: 0 for k in kinds}
    for i in range(len(pts) - 1):
        for k in kinds:
            running[k] += delta[k][i]
        total = sum(running.values())
        if total:
            dt = (pts[i + 1] - pts[i]) / 1e3 / total
            for k in kinds:
                if running[k]:
                    out[k]["attributed_ms"] += dt * running[k]
    span = (max(e0 for _, e0, _ in ks) - min(s0 for s0, _, _ in ks)) / 1e3
    return out, span


# --------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # time >= 20 steps
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="7b", choices=["tiny", "1b", "7b", "moe", "70b_layer"])
    ap.add_argument("--batch", type=int, default=None, help="per-GPU batch (sequences)")
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--moe-routing", default="router", choices=["router", "balanced"],
                    help="balanced: every expert gets the same number of tokens (benchmark of dispatch / grouped "
                         "expert GEMMs / combine off the reference init's degenerate routing; not the reference numerics)")
    ap.add_argument("--remat", default=None,
                    help="remat policy alias for every layer (reference mesh.py:204-252 names); default: "
                         "save_qkvo_flash for 70b_layer (BASELINE configs[4]: FSDP + rematerialisation; the "
                         "policy of the reference's gpu-H100 mesh rule, experiments.py:49), none otherwise")
    args = ap.parse_args()
    defaults = {"tiny": (8, 256), "1b": (8, 4096), "7b": (3, 4096), "moe": (4, 4096), "70b_layer": (2, 4096)}
    if args.remat is None:
        args.remat = "save_qkvo_flash" if args.config == "70b_layer" else "save_all"
    args.batch = args.batch or defaults[args.config][0]
    args.seq = args.seq or defaults[args.config][1]
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, _lib, ops, synthetic_batch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = "f32" if args.config == "tiny" else "bf16"
    cfg = BENCH_CONFIGS[args.config](batch=args.batch, seq=args.seq, dtype=dtype)
    if args.remat != "save_all":
        from paper_2507_05411_b200.remat import POLICY_ALIASES

        for i in range(len(cfg.get("model.decoder.transformer.layer"))):
            cfg = cfg.set(f"model.decoder.transformer.layer[{i}].remat_policy", POLICY_ALIASES[args.remat])
    eng = TrainEngine(cfg, device=dev)
    if args.moe_routing == "balanced":
        eng.options["moe_balanced_routing"] = True
    V = eng.cfg.get("model.vocab_size")
    B, T = args.batch, args.seq
    nsteps = args.warmup + args.steps
    host = [synthetic_batch(rank, s, B, T, V)["tokens"] for s in range(nsteps)]
    devtok = [eng.upload_tokens(h) for h in host]
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()
    for s in range(args.warmup):
        eng.step(devtok[s])
    barrier()
    # ---- timed region: inputs resident in HBM
    sampler = ClockSampler(local)
    sampler.start()
    n0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    loss = None
    for s in range(args.steps):
        loss, _ = eng.step(devtok[args.warmup + s])
    ev1.record(stream)
    barrier()
    launches = _lib.launch_count() - n0
    clocks = sampler.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    final_loss = float(loss.item())
    tokens_step = world * B * T
    value = tokens_step / (ms / 1e3)

    mem_peak = torch.cuda.max_memory_allocated(dev)

    # ---- kernel shares: the same steps again under CUPTI kernel activity (all streams);
    # the Python-side tally gives the algorithmic FLOPs of the GEMM / attention launches
    prof = ops.KernelProfiler(events=False)
    nprof = min(args.steps, 3)

    def profiled_steps():
        ops.set_profiler(prof)
        for s in range(nprof):
            eng.step(devtok[args.warmup + s])
        ops.set_profiler(None)

    barrier()
    cupti, span_ms = cupti_attribution(profiled_steps)
    barrier()
    tally = prof.summary()

    # ---- end to end through the public API: host tokens in, loss out, every step
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for s in range(args.steps):
        l_, _ = eng.step(host[args.warmup + s])
        float(l_.item())
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk, pk_src = peaks()
    fpt = flops_per_token(eng.module, B, T)
    gflops = sum(v["flops"] for k, v in tally.items() if k.startswith("gemm"))
    g = cupti.get("gemm", {"launches": 0, "busy_ms": 0.0, "attributed_ms": 0.0})
    achieved = gflops / (g["busy_ms"] / 1e3) / 1e12 if g["busy_ms"] else 0.0
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    traffic = None
    tpath = os.path.join(REPO, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("workload") == args.config and tj.get("per_gpu_batch", args.batch) == args.batch:
            traffic = tj.get("bytes_per_launch")
    flops_by_kind = {"gemm": gflops, "attn_fwd": tally.get("attn_fwd", {}).get("flops", 0),
                     "attn_bwd": tally.get("attn_bwd", {}).get("flops", 0)}
    kernels = {}
    for k, v in sorted(cupti.items(), key=lambda kv: -kv[1]["attributed_ms"]):
        row = {"launches_per_step": v["launches"] / nprof, "busy_ms_per_step": v["busy_ms"] / nprof,
               "attributed_ms_per_step": v["attributed_ms"] / nprof}
        if "top" in v:
            row["top_ms"] = [(n, round(t / nprof, 2)) for n, t in v["top"]]
        if flops_by_kind.get(k):
            row["tflops"] = flops_by_kind[k] / (v["busy_ms"] / 1e3) / 1e12
        kernels[k] = row
    from paper_2507_05411_b200.memory import aot_device_bytes

    aot = aot_device_bytes(eng.module, world * B, T, world)
    line = {
        "metric": "train tokens/sec and MFU per B200, decoder step",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (reference synthetic_batch token stream; reference init_state weights)",
        "config": workload_config(args, world),
        "setup": {"collectives": ("none" if world == 1 else
                                  ("all-gather " + ("copy-engine/symm-mem" if eng._ce_gather else "nccl")
                                   + ", reduce-scatter " + ("copy-engine/symm-mem, sum fused into AdamW"
                                                            if eng._ce_reduce else "nccl"))),
                  "zero3": {"resharded_params": eng._reshard, "gradient_ring": eng._grad_ring}},
        "mfu": value * fpt / (world * NOMINAL_BF16_PFLOPS),
        "model_flops_per_token": fpt,
        "loss": final_loss,
        "roofline": {"bound": "tensor", "kernel": "gemm_tc2 (tcgen05 CTA-pair persistent GEMM)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": f"{pk_src} bf16_tflops_sustained (kernel timed inside the step)",
                     "achieved_how": "algorithmic GEMM FLOPs of the profiled steps / the GEMM launches' summed CUPTI "
                                     "kernel durations",
                     "traffic": traffic,
                     "traffic_source": ("ncu --set full constant (profiles/gemm_traffic.json: DRAM read+write of one "
                                        "launch of this workload's QKV GEMM), not measured by this run"
                                        if traffic is not None else None),
                     "share_of_step": g["attributed_ms"] / span_ms if span_ms else None},
        "kernels": kernels,
        "kernels_note": ("CUPTI kernel activity over %d steps; attributed_ms splits overlapping kernels evenly, so "
                         "the attributed column sums to the busy time of the profiled span (%.1f ms/step)"
                         % (nprof, span_ms / nprof)),
        "memory": {"max_allocated_gb": mem_peak / 1e9, "engine_state_gb": eng.state_bytes() / 1e9,
                   "forward_leaves_gb": getattr(eng, "last_forward_bytes", 0) / 1e9,
                   "aot_analyze_per_device_gb": aot["per_device_bytes"] / 1e9,
                   "aot_analyze_saved_activation_gb": aot["saved_activation_bytes"] / 1e9,
                   "aot_formula": aot["formula"]},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": tokens_step / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": B * T * 8,
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = reference_sample(args.config)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
