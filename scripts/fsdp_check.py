"""Multi-GPU FSDP parity: run under torchrun with N ranks.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 --master-port 29511 \
        scripts/fsdp_check.py [--precision f32|bf16] [--config txf_rope|mid|mid_moe] [--steps 3] \
        [--mode step|decomposed] [--collectives ce|nccl|both]

Each rank trains on its slice of one global batch; the all-reduced loss, the gradients and
the updated parameters must match the single-process oracle on the whole global batch
(reference SPEC.md:445 / test_mesh.py:493-507: numerics do not depend on the
partitioning).  Rank 0 prints one JSON line.

--mode step (default) drives the path the benchmark runs: TrainEngine.step() — AdamW of
each bucket on the communication stream right after its reduce-scatter, the ZeRO-3 gather
and gradient rings, copy-engine collectives between symmetric-memory barriers — for
--steps steps, and compares every step's loss, the last step's gradients, and the final
parameters and AdamW moments with the oracle's chained train_step.  f32 tensors are held to
1e-5, or to 3x the error of the same steps computed by a plain fp32 restatement where fp32
itself cannot meet 1e-5 (tests/test_step_gpu.py:fp32_oracle_errors); bf16 to 2e-2, or to 1.5x
the error of the oracle with bf16-rounded GEMM operands where that is larger.
--mode decomposed drives compute_grads() + apply_update() (the round-1 check).
--collectives both runs the step twice, with the copy-engine collectives (CB_FSDP_CE_*=1)
and with NCCL (=0), both against the oracle and against each other.
"""

import argparse
import contextlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def build(config):
    from paper_2507_05411_b200 import build_experiment
    from paper_2507_05411_b200.experiments import transformer_trainer

    if config in ("mid", "mid_moe"):
        cfg = transformer_trainer(256, 2, ("linear", "silu"), pos_kind="RoPE", heads=2, vocab=512,
                                  feed_forward_kind="MoE" if config == "mid_moe" else "FeedForward",
                                  num_experts=4, top_k=2)
        for i in range(2):
            cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
        return cfg
    return build_experiment(config)


def oracle_run(cfg, B, T, steps, precision, dtype, bf16_operands=False):
    """The oracle's chained train_step on the global batches (dtype=float32: the plain fp32
    restatement used as the fp32 error yardstick)."""
    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import init_state, instantiate, root_key, set_dtype_policy, synthetic_batch

    m = instantiate(set_dtype_policy(cfg, precision))
    st = init_state(m, root_key(0))
    spec = O.spec_from_config(m.config)
    V = m.config.get("model.vocab_size")
    mm = vv = None
    losses, summs, grads = [], [], None
    for step in range(steps):
        toks = synthetic_batch(0, step, B, T, V)["tokens"]
        with (O.bf16_operands() if bf16_operands else contextlib.nullcontext()):
            lo, go, st, mm, vv, osum = O.train_step(st, toks, spec, O.AdamW(lr=1e-3), mm, vv, step + 1, dtype=dtype)
        losses.append(lo)
        summs.append(osum)
        grads = go
    return losses, summs, dict(O.leaves(grads)), dict(O.leaves(st)), dict(O.leaves(mm))


def engine_run(cfg, precision, B, T, steps, mode, ce):
    import torch

    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
    from oracle import decoder_oracle as O

    for k in ("CB_FSDP_CE_GATHER", "CB_FSDP_CE_REDUCE"):
        os.environ[k] = "1" if ce else "0"
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    eng = TrainEngine(set_dtype_policy(cfg, precision), device=dev)
    eng.keep_grad_shards = True  # the last step's gradients are compared with the oracle's
    V = eng.cfg.get("model.vocab_size")
    per = B // world
    losses, summs = [], []
    for step in range(steps):
        toks = synthetic_batch(0, step, B, T, V)["tokens"]
        mine = toks[rank * per:(rank + 1) * per]
        if mode == "step":
            loss, col = eng.step(mine)
        else:
            loss, col = eng.compute_grads(mine)
            eng.apply_update()
        losses.append(float(loss.item()))
        summs.append({k: float(v[0]) for k, v in col.flat_summaries().items()})
    out = {"losses": losses, "summaries": summs, "grads": dict(O.leaves(eng.grads_numpy())),
           "params": dict(O.leaves(eng.state_numpy())), "m": dict(O.leaves(eng.opt_state_numpy()["m"])),
           "ce": (eng._ce_gather, eng._ce_reduce), "reshard": eng._reshard, "grad_ring": eng._grad_ring,
           "state_bytes": eng.state_bytes()}
    del eng
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--config", default="txf_rope")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8, help="global batch")
    ap.add_argument("--seq", type=int, default=8)
    ap.add_argument("--mode", default="step", choices=["step", "decomposed"])
    ap.add_argument("--collectives", default="ce", choices=["ce", "nccl", "both"])
    ap.add_argument("--ckpt", default=None, help="save a sharded checkpoint here after training")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from oracle import decoder_oracle as O

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = build(args.config)
    B, T = args.batch, args.seq
    assert B % world == 0
    tol = 1e-5 if args.precision == "f32" else 2e-2
    lo, osum, go, po, mo = oracle_run(cfg, B, T, args.steps, args.precision, torch.float64)
    if args.precision == "f32":
        _, _, g32, p32, m32 = oracle_run(cfg, B, T, args.steps, args.precision, torch.float32)
        gb = {k: max(tol, 3 * _rel(g32[k], go[k])) for k in go}
        pb = {k: max(tol, 3 * _rel(p32[k], po[k])) for k in po}
        mb = {k: max(tol, 3 * _rel(m32[k], mo[k])) for k in mo}
    else:
        # bf16: 1.5x the error of the oracle with only its GEMM operands rounded to bf16 (the
        # least rounding any bf16 path does) where that exceeds tol / 1.5 (tests/test_step_gpu.py)
        _, _, gq, pq, mq = oracle_run(cfg, B, T, args.steps, args.precision, torch.float64, bf16_operands=True)
        gb = {k: max(tol, 1.5 * _rel(gq[k], go[k])) for k in go}
        pb = {k: max(tol, 1.5 * _rel(pq[k], po[k])) for k in po}
        mb = {k: max(tol, 1.5 * _rel(mq[k], mo[k])) for k in mo}
    out = {"world": world, "precision": args.precision, "config": args.config, "mode": args.mode,
           "steps": args.steps, "runs": {}}
    ok = True
    runs = {}
    for ce in ([True, False] if args.collectives == "both" else [args.collectives == "ce"]):
        r = engine_run(cfg, args.precision, B, T, args.steps, args.mode, ce)
        runs[ce] = r
        rec = {"ce_gather_reduce": r["ce"], "reshard": r["reshard"], "grad_ring": r["grad_ring"],
               "state_bytes": r["state_bytes"],
               "loss_rel": [abs(a - b) / abs(b) for a, b in zip(r["losses"], lo)],
               "grad_worst": max((_rel(r["grads"][k], go[k]) / gb[k], k) for k in go),
               "param_worst": max((_rel(r["params"][k], po[k]) / pb[k], k) for k in po),
               "adam_m_worst": max((_rel(r["m"][k], mo[k]) / mb[k], k) for k in mo)}
        # MoE load-balance summaries are global-batch statistics (reduced across ranks)
        lb = [abs(r["summaries"][s][k] - v) / abs(v) for s, d in enumerate(osum) for k, v in d.items()
              if k.endswith("load_balance_loss") and k in r["summaries"][s]]
        rec["lb_rel_max"] = max(lb) if lb else None
        ok &= max(rec["loss_rel"]) < tol and rec["grad_worst"][0] < 1 and rec["param_worst"][0] < 1
        ok &= rec["adam_m_worst"][0] < 1 and (not lb or max(lb) < tol)
        out["runs"]["ce" if ce else "nccl"] = rec
    if len(runs) == 2:  # the two collective implementations against each other
        a, b = runs[True], runs[False]
        out["ce_vs_nccl"] = {"loss_rel": max(abs(x - y) / abs(y) for x, y in zip(a["losses"], b["losses"])),
                             "param_rel": max(_rel(a["params"][k], b["params"][k]) for k in a["params"])}
        ok &= out["ce_vs_nccl"]["loss_rel"] < tol and out["ce_vs_nccl"]["param_rel"] < tol
    out["bound_note"] = "worst entries are error / bound (< 1 passes); bound = max(tol, 3 x fp32-restatement error)"
    if args.ckpt:
        from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
        from paper_2507_05411_b200.checkpoint import save_checkpoint

        eng = TrainEngine(set_dtype_policy(cfg, args.precision), device=torch.device("cuda", local))
        per = B // world
        for step in range(args.steps):
            toks = synthetic_batch(0, step, B, T, eng.cfg.get("model.vocab_size"))["tokens"]
            eng.step(toks[rank * per:(rank + 1) * per])
        out["ckpt"] = save_checkpoint(eng, args.ckpt)
        params, opt = eng.state_numpy(), eng.opt_state_numpy()
        if rank == 0:  # reference copy of the full state for the restore test
            flat = {f"p:{k}": v for k, v in O.leaves(params)}
            flat.update({f"m:{k}": v for k, v in O.leaves(opt["m"])})
            flat.update({f"v:{k}": v for k, v in O.leaves(opt["v"])})
            np.savez(os.path.join(args.ckpt, "ref_state.npz"), **flat)
    out["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
