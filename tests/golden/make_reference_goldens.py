"""Generates tests/golden/reference_goldens.json by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, which does not exist on the GPU
box):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reference_goldens.py

Everything recorded comes from the reference's own public API (composer.*): the 27
registry experiments' step-0 loss and summaries via invoke(), init_state parameter
checksums, the tiny bench config's loss, route_tokens / rope_apply outputs, and
central finite differences of the reference loss (the only pin available for
gradients, since the reference has no backward — SPEC.md:15, 248).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from composer.config import FunctionSpec, default_config  # noqa: E402
from composer.experiments import EXPERIMENTS, build_experiment, synthetic_batch  # noqa: E402
from composer.layers import rope_apply, route_tokens, load_balance_loss  # noqa: E402
from composer.module import init_state, instantiate, invoke  # noqa: E402
from composer.prng import child_key, root_key  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_goldens.json")


def leaves(tree, prefix=""):
    for k in sorted(tree):
        v = tree[k]
        p = f"{prefix}.{k}" if prefix else k
        if isinstance(v, dict):
            yield from leaves(v, p)
        else:
            yield p, v


def get_leaf(tree, path):
    for seg in path.split("."):
        tree = tree[seg]
    return tree


def tiny_config():
    """The BASELINE configs[0] tiny decoder: 2 layers, d=128, 4 heads, RoPE, SwiGLU, V=64."""
    layer = (
        default_config("TransformerLayer")
        .set("self_attention.num_heads", 4)
        .set("self_attention.pos_emb", default_config("RoPE"))
        .set("feed_forward.activation", ("linear", "silu"))
        .set("feed_forward.hidden_dim", FunctionSpec("scaled_hidden_dim", scale=8.0 / 3.0))
    )
    return (
        default_config("Trainer")
        .set("model.dim", 128)
        .set("model.vocab_size", 64)
        .set("model.decoder.transformer.layer", (layer,) * 2)
        .set("learner.lr", 1e-3)
        .set("batch_size", 8)
        .set("seq_len", 256)
    )


def run(cfg, seed=0, step=0):
    module = instantiate(cfg)
    key = root_key(seed)
    state = init_state(module, key)
    b, t, v = cfg.get("batch_size"), cfg.get("seq_len"), cfg.get("model.vocab_size")
    batch = synthetic_batch(seed, step, b, t, v)
    loss, col = invoke(module, state, child_key(key, "step", step), batch)
    return module, state, batch, loss, col


def fd_grads(cfg, picks, eps=1e-6):
    module, state, batch, loss, _ = run(cfg)
    key = child_key(root_key(0), "step", 0)
    out = []
    for path, idx in picks:
        arr = get_leaf(state, path)
        orig = arr[idx]
        arr[idx] = orig + eps
        lp, _ = invoke(module, state, key, batch)
        arr[idx] = orig - eps
        lm, _ = invoke(module, state, key, batch)
        arr[idx] = orig
        out.append({"path": path, "index": list(idx), "grad": (lp - lm) / (2 * eps)})
    return out


def main():
    gold = {"experiments": {}, "meta": {"numpy": np.__version__}}
    for name in sorted(EXPERIMENTS):
        cfg = build_experiment(name)
        module, state, batch, loss, col = run(cfg)
        gold["experiments"][name] = {
            "loss": loss,
            "batch_size": cfg.get("batch_size"),
            "seq_len": cfg.get("seq_len"),
            "tokens": batch["tokens"].tolist(),
            "summaries": {k: [float(x) for x in v] for k, v in col.flat_summaries().items()},
            "params": {p: {"shape": list(a.shape), "sum": float(a.sum()), "sumsq": float((a * a).sum()),
                           "head": [float(x) for x in a.reshape(-1)[:4]]} for p, a in leaves(state)},
        }
    # a second step/seed through the run loop (cli.py:121-124 semantics)
    cfg = build_experiment("txf_moe")
    module = instantiate(cfg)
    state = init_state(module, root_key(7))
    losses = []
    for step in range(2):
        batch = synthetic_batch(7, step, cfg.get("batch_size"), cfg.get("seq_len"), cfg.get("model.vocab_size"))
        loss, _ = invoke(module, state, child_key(root_key(7), "step", step), batch)
        losses.append(loss)
    gold["txf_moe_seed7_losses"] = losses

    tcfg = tiny_config()
    _, tstate, tbatch, tloss, _ = run(tcfg)
    gold["tiny"] = {"loss": tloss, "params": {p: {"sum": float(a.sum()), "sumsq": float((a * a).sum())}
                                             for p, a in leaves(tstate)}}

    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, 3, 5, 8))
    gold["rope"] = {"x": x.tolist(), "base": 10000.0, "out": rope_apply(x, np.arange(5), 10000.0).tolist()}

    probs = np.round(rng.random((6, 7, 8)), 1) + 1e-3  # coarse values -> many ties
    probs = probs / probs.sum(-1, keepdims=True)
    dec = route_tokens(probs, 2)
    gold["route"] = {"probs": probs.tolist(), "top_k": 2, "indices": dec.indices.tolist(),
                     "weights": dec.weights.tolist(), "dispatch": dec.dispatch_fractions.tolist(),
                     "mean_probs": dec.mean_probs.tolist(), "lbl": load_balance_loss(dec)}

    # Linear with bias (layers.py:130-170): reference invoke on a given state, and central
    # differences of sum(y * dy) for a few weight / bias / input entries
    lin = instantiate(default_config("Linear").set("input_dim", 16).set("output_dim", 24).set("bias", True))
    lx = rng.standard_normal((2, 3, 16))
    lst = {"weight": rng.standard_normal((16, 24)) * 0.25, "bias": rng.standard_normal(24) * 0.1}
    ldy = rng.standard_normal((2, 3, 24))
    ly, _ = invoke(lin, lst, root_key(0), lx)

    def lin_obj(st, x):
        return float(np.sum(invoke(lin, st, root_key(0), x)[0] * ldy))

    fd = {}
    for name, idx in (("weight", (3, 5)), ("weight", (15, 23)), ("bias", (7,)), ("x", (1, 2, 9))):
        vals = []
        for sgn in (1.0, -1.0):
            st2 = {k: v.copy() for k, v in lst.items()}
            x2 = lx.copy()
            (x2 if name == "x" else st2[name])[idx] += sgn * 1e-6
            vals.append(lin_obj(st2, x2))
        fd[f"{name}{list(idx)}"] = (vals[0] - vals[1]) / 2e-6
    gold["linear"] = {"x": lx.tolist(), "weight": lst["weight"].tolist(), "bias": lst["bias"].tolist(),
                      "dy": ldy.tolist(), "y": np.asarray(ly).tolist(), "fd": fd}

    base_picks = [
        ("model.decoder.emb.weight", (3, 5)),
        ("model.decoder.emb.weight", (44, 0)),
        ("model.decoder.output_norm.scale", (7,)),
        ("model.decoder.transformer.layer[0].self_attention.wq", (1, 2)),
        ("model.decoder.transformer.layer[0].self_attention.wk", (4, 9)),
        ("model.decoder.transformer.layer[0].self_attention.wv", (10, 3)),
        ("model.decoder.transformer.layer[1].self_attention.wo", (5, 6)),
        ("model.decoder.transformer.layer[1].self_attention_norm.scale", (11,)),
        ("model.decoder.transformer.layer[0].feed_forward_norm.scale", (2,)),
    ]
    dense_picks = base_picks + [
        ("model.decoder.transformer.layer[0].feed_forward.w1", (3, 7)),
        ("model.decoder.transformer.layer[1].feed_forward.w1_gate", (8, 1)),
        ("model.decoder.transformer.layer[1].feed_forward.w2", (2, 30)),
    ]
    moe_picks = base_picks + [
        ("model.decoder.transformer.layer[0].feed_forward.router", (3, 1)),
        ("model.decoder.transformer.layer[1].feed_forward.router", (12, 2)),
        ("model.decoder.transformer.layer[0].feed_forward.w1", (1, 3, 7)),
        ("model.decoder.transformer.layer[1].feed_forward.w1_gate", (2, 8, 1)),
        ("model.decoder.transformer.layer[0].feed_forward.w2", (3, 2, 30)),
    ]
    gold["fd_grads"] = {
        "txf_rope": fd_grads(build_experiment("txf_rope"), dense_picks),
        "txf_base": fd_grads(build_experiment("txf_base"), dense_picks),
        "txf_moe": fd_grads(build_experiment("txf_moe"), moe_picks),
        "txf_d32_l2_relu": fd_grads(build_experiment("txf_d32_l2_relu"), base_picks),
    }
    with open(OUT, "w") as fh:
        json.dump(gold, fh, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
