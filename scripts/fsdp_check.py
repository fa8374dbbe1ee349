"""Multi-GPU FSDP parity: run under torchrun with N ranks.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 --master-port 29511 \
        scripts/fsdp_check.py [--precision f32|bf16] [--config txf_rope|mid] [--steps 2]

Each rank trains on its slice of one global batch; the all-reduced loss, the gathered
gradients and the updated parameters must match the single-process oracle on the whole
global batch (parity across N).  Rank 0 prints one JSON line.
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--config", default="txf_rope")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=8, help="global batch")
    ap.add_argument("--seq", type=int, default=8)
    ap.add_argument("--ckpt", default=None, help="save a sharded checkpoint here after training")
    ap.add_argument("--decomposed", action="store_true",
                    help="hold the update to AdamW on the GPU's own gradients instead of the oracle's parameters")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import (TrainEngine, build_experiment, init_state, instantiate, root_key,
                                       set_dtype_policy, synthetic_batch)
    from paper_2507_05411_b200.experiments import transformer_trainer

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    if args.config == "mid":
        cfg = transformer_trainer(256, 2, ("linear", "silu"), pos_kind="RoPE", heads=2, vocab=512)
        for i in range(2):
            cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    else:
        cfg = build_experiment(args.config)
    cfg = set_dtype_policy(cfg, args.precision)
    eng = TrainEngine(cfg, device=dev)
    V = eng.cfg.get("model.vocab_size")
    B, T = args.batch, args.seq
    assert B % world == 0
    per = B // world

    m = instantiate(cfg)
    st = init_state(m, root_key(0))
    spec = O.spec_from_config(m.config)
    mm = vv = None
    out = {"world": world, "precision": args.precision, "config": args.config, "steps": []}
    tol = 1e-5 if args.precision == "f32" else 2e-2
    ok = True
    own_worst = 0.0  # AdamW applied in f64 to the GPU's own gradients vs the GPU's update
    for step in range(args.steps):
        toks = synthetic_batch(0, step, B, T, V)["tokens"]
        mine = toks[rank * per:(rank + 1) * per]
        loss, col = eng.compute_grads(mine)
        loss = float(loss.item())
        summ = col.flat_summaries()
        g_all = eng.grads_numpy()
        grads = g_all if step == 0 else None
        p_before, o_before = eng.state_numpy(), eng.opt_state_numpy()
        eng.apply_update()
        p_after = eng.state_numpy()
        opt = O.AdamW(lr=eng.lr, beta1=eng.beta1, beta2=eng.beta2)
        for (k, p0), (_, g0), (_, m0), (_, v0), (_, p1) in zip(O.leaves(p_before), O.leaves(g_all),
                                                                O.leaves(o_before["m"]), O.leaves(o_before["v"]),
                                                                O.leaves(p_after)):
            exp_p, _, _ = O.adamw_update(p0.astype(np.float64), g0.astype(np.float64), m0.astype(np.float64),
                                         v0.astype(np.float64), step + 1, opt)
            own_worst = max(own_worst, float(np.linalg.norm(p1 - exp_p) / max(np.linalg.norm(exp_p), 1e-30)))
        lo, go, st, mm, vv, osum = O.train_step(st, toks, spec, O.AdamW(lr=eng.lr), mm, vv, step + 1)
        rec = {"loss": loss, "oracle": lo, "loss_rel": abs(loss - lo) / lo}
        ok &= rec["loss_rel"] < tol
        # MoE load-balance summaries are global-batch statistics (reduced across ranks)
        for key, ref in sorted(osum.items()):
            if key.endswith("load_balance_loss") and key in summ:
                got = float(summ[key][0])
                rel = abs(got - ref) / abs(ref)
                rec.setdefault("lb_rel_max", 0.0)
                rec["lb_rel_max"] = max(rec["lb_rel_max"], rel)
                ok &= rel < tol
        if grads is not None:
            worst = 0.0
            for (k, a), (_, b) in zip(O.leaves(grads), O.leaves(go)):
                worst = max(worst, float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)))
            rec["grad_rel_max"] = worst
            ok &= worst < tol
        out["steps"].append(rec)
    params = eng.state_numpy()
    worst = 0.0
    for (k, a), (_, b) in zip(O.leaves(params), O.leaves(st)):
        worst = max(worst, float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)))
    out["param_rel_max"] = worst
    out["adamw_own_grads_rel_max"] = own_worst
    # --decomposed: the update is checked against AdamW on the GPU's own gradients (the
    # gradients themselves are held to tol above); step-1 AdamW ~ lr * sign(g) amplifies
    # ulp-level gradient differences of near-zero entries by 1/eps (DESIGN (c)(i))
    ok &= (own_worst < tol) if args.decomposed else (worst < tol)
    if args.ckpt:
        from paper_2507_05411_b200.checkpoint import save_checkpoint

        rep = save_checkpoint(eng, args.ckpt)
        out["ckpt"] = rep
        opt = eng.opt_state_numpy()
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
