"""CPU float64 oracle of the decoder training step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline.  The product path
(``paper_2507_05411_b200``) never imports it and has no CPU fallback.

What it restates (all citations are /root/reference/pkg/src/composer/):
  * forward numerics of the reference step, operation for operation, in float64:
      - RMSNorm ``x / sqrt(mean(x^2)+eps) * scale``                  layers.py:188-193
      - RoPE, interleaved pairs, base^(-2i/d), positions arange(T)     layers.py:235-257, 343
      - unmasked multi-head attention, [d,d] projections, x @ W        layers.py:331-348
      - FFN, gated (act0(x@w1) * act1(x@w1_gate)) @ w2 or act(x@w1)@w2 layers.py:405-416
      - stable sigmoid / activation table                              layers.py:55-77
      - MoE: softmax router, stable top-k (ties -> lowest id), renorm,
        dense experts, slot-order combine, load_balance_loss summary   layers.py:432-449, 513-533
      - pre-norm residual layer, stack, decoder, tied head h @ E^T     layers.py:549-620
      - loss = -mean log_softmax(logits[:, :-1])[tokens[:, 1:]]         layers.py:641-651
  * the backward of that forward: torch float64 autograd on the restated graph (the
    reference has no backward, SPEC.md:15/248 — the gradient is pinned instead by central
    finite differences of the reference's own loss, tests/golden/reference_goldens.json);
  * AdamW as the fn:adamw factory (layers.py:657-663, 778-782) describes, with the
    documented extra hyper-parameters eps=1e-8, weight decay 0, bias correction.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle's loss against the
reference's ``invoke`` on all 27 registry experiments + the tiny bench config (<=1e-12),
its MoE routing against ``route_tokens`` and its gradients against finite differences.

Extension beyond the reference: ``kv_heads`` < ``num_heads`` (grouped-query attention)
for the 70B-layer config; with kv_heads == num_heads it is exactly the reference op.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

F64 = torch.float64


# ------------------------------------------------------------------------------------
# model description (read from a reference-style config via .get(); no product imports)
# ------------------------------------------------------------------------------------
@dataclass
class LayerSpec:
    heads: int
    kv_heads: int
    pos: str  # "NoPos" | "RoPE"
    rope_base: float
    ffn: str  # "FeedForward" | "MoE"
    activation: object  # str or (str, str)
    hidden: int
    experts: int = 0
    top_k: int = 0
    eps1: float = 1e-6
    eps2: float = 1e-6


@dataclass
class ModelSpec:
    dim: int
    vocab: int
    layers: list[LayerSpec] = field(default_factory=list)
    out_eps: float = 1e-6


def spec_from_config(cfg) -> ModelSpec:
    """cfg: an *instantiated* (finalized) Trainer config node (reference or product)."""
    dim = cfg.get("model.dim")
    vocab = cfg.get("model.vocab_size")
    layers = []
    for lc in cfg.get("model.decoder.transformer.layer"):
        att = lc.get("self_attention")
        ff = lc.get("feed_forward")
        heads = att.get("num_heads")
        kvh = att.get("num_kv_heads") if att.has_field("num_kv_heads") else heads
        pos = att.get("pos_emb").kind
        base = att.get("pos_emb.base") if pos == "RoPE" else 10000.0
        act = ff.get("activation")
        layers.append(LayerSpec(
            heads=heads, kv_heads=kvh, pos=pos, rope_base=base, ffn=ff.kind,
            activation=tuple(act) if isinstance(act, tuple) else act, hidden=ff.get("hidden_dim"),
            experts=ff.get("num_experts") if ff.kind == "MoE" else 0,
            top_k=ff.get("top_k") if ff.kind == "MoE" else 0,
            eps1=lc.get("self_attention_norm.eps"), eps2=lc.get("feed_forward_norm.eps"),
        ))
    return ModelSpec(dim, vocab, layers, cfg.get("model.decoder.output_norm.eps"))


# ------------------------------------------------------------------------------------
# ops
# ------------------------------------------------------------------------------------
def _sigmoid(x):
    # two-branch form of layers.py:55-61 (identical values in f64 up to rounding)
    return torch.where(x >= 0, 1.0 / (1.0 + torch.exp(-x.clamp(min=0))), torch.exp(x.clamp(max=0)) / (1.0 + torch.exp(x.clamp(max=0))))


ACT = {
    "linear": lambda x: x,
    "relu": lambda x: torch.clamp(x, min=0.0),
    "silu": lambda x: x * _sigmoid(x),
    "sigmoid": _sigmoid,
    "tanh": torch.tanh,
}


def rmsnorm(x, scale, eps):
    ms = (x * x).mean(dim=-1, keepdim=True)
    return x / torch.sqrt(ms + eps) * scale


def rope_tables(seq_len: int, dim: int, base: float):
    half = dim // 2
    freqs = base ** (-2.0 * np.arange(half) / dim)
    ang = np.arange(seq_len, dtype=np.float64)[:, None] * freqs[None, :]
    return np.cos(ang), np.sin(ang)


def rope_apply(x, base: float):
    """x [..., T, d], pairs (2i, 2i+1) — layers.py:235-257."""
    T, d = x.shape[-2], x.shape[-1]
    c, s = rope_tables(T, d, base)
    c = torch.as_tensor(c, dtype=x.dtype)
    s = torch.as_tensor(s, dtype=x.dtype)
    even, odd = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out = torch.stack((even * c - odd * s, even * s + odd * c), dim=-1).reshape(x.shape)
    return out


def attention(x, p, ls: LayerSpec):
    b, t, d = x.shape
    H, KVH = ls.heads, ls.kv_heads
    hd = d // H

    def split(y, nh):
        return y.reshape(b, t, nh, hd).transpose(1, 2)

    q = split(x @ p["wq"], H)
    k = split(x @ p["wk"], KVH)
    v = split(x @ p["wv"], KVH)
    if ls.pos == "RoPE":
        q, k = rope_apply(q, ls.rope_base), rope_apply(k, ls.rope_base)
    if KVH != H:
        rep = H // KVH
        k = k.repeat_interleave(rep, dim=1)
        v = v.repeat_interleave(rep, dim=1)
    scores = q @ k.transpose(-1, -2) / math.sqrt(hd)
    probs = torch.softmax(scores, dim=-1)
    ctx = (probs @ v).transpose(1, 2).reshape(b, t, d)
    return ctx @ p["wo"]


def _act_pair(activation):
    if isinstance(activation, str):
        return None
    return tuple(activation)


def feed_forward(x, p, ls: LayerSpec):
    pair = _act_pair(ls.activation)
    if pair:
        hidden = ACT[pair[0]](x @ p["w1"]) * ACT[pair[1]](x @ p["w1_gate"])
    else:
        hidden = ACT[ls.activation](x @ p["w1"])
    return hidden @ p["w2"]


def route_tokens(probs: torch.Tensor, top_k: int):
    """Stable top-k over -probs (ties -> lowest expert id), renormalized — layers.py:432-443."""
    order = torch.argsort(-probs.detach(), dim=-1, stable=True)
    idx = order[..., :top_k]
    picked = torch.gather(probs, -1, idx)
    w = picked / picked.sum(dim=-1, keepdim=True)
    E = probs.shape[-1]
    counts = torch.bincount(idx.reshape(-1), minlength=E).to(probs.dtype)
    dispatch = counts / idx.numel()
    mean_probs = probs.detach().reshape(-1, E).mean(dim=0)
    return idx, w, dispatch, mean_probs


def moe(x, p, ls: LayerSpec, forced_idx=None):
    """forced_idx [B, T, k]: use these expert choices instead of the top-k (the reference's
    own forced-routing oracle, tests/test_layers.py:352-359); weights still renormalize the
    router probabilities of the chosen experts."""
    probs = torch.softmax(x @ p["router"], dim=-1)
    idx, w, dispatch, mean_probs = route_tokens(probs, ls.top_k)
    if forced_idx is not None:
        idx = torch.as_tensor(np.asarray(forced_idx), dtype=torch.long)
        picked = torch.gather(probs, -1, idx)
        w = picked / picked.sum(dim=-1, keepdim=True)
        dispatch = torch.bincount(idx.reshape(-1), minlength=probs.shape[-1]).to(probs.dtype) / idx.numel()
    pair = _act_pair(ls.activation)
    hidden = torch.einsum("btd,edh->ebth", x, p["w1"])
    if pair:
        hidden = ACT[pair[0]](hidden) * ACT[pair[1]](torch.einsum("btd,edh->ebth", x, p["w1_gate"]))
    else:
        hidden = ACT[ls.activation](hidden)
    eo = torch.einsum("ebth,ehd->ebtd", hidden, p["w2"])
    b, t, _ = x.shape
    bi = torch.arange(b)[:, None]
    ti = torch.arange(t)[None, :]
    out = torch.zeros_like(x)
    for slot in range(ls.top_k):
        e = idx[..., slot]
        out = out + w[..., slot][..., None] * eo[e, bi, ti]
    lbl = float(ls.experts * torch.sum(dispatch * mean_probs))
    return out, lbl, idx


def forward_loss(params: dict, tokens: np.ndarray, spec: ModelSpec, summaries: dict | None = None,
                 forced_routing: dict | None = None, routing: dict | None = None):
    """params: nested dict of float64 torch tensors in the reference state layout.
    routing: if given, receives {layer index: top-k expert indices [B, T, k]} of MoE layers."""
    dec = params["model"]["decoder"]
    tok = torch.as_tensor(np.asarray(tokens), dtype=torch.long)
    table = dec["emb"]["weight"]
    h = table[tok]
    for i, ls in enumerate(spec.layers):
        lp = dec["transformer"][f"layer[{i}]"]
        x = h
        h = x + attention(rmsnorm(x, lp["self_attention_norm"]["scale"], ls.eps1), lp["self_attention"], ls)
        n2 = rmsnorm(h, lp["feed_forward_norm"]["scale"], ls.eps2)
        if ls.ffn == "MoE":
            f, lbl, idx = moe(n2, lp["feed_forward"], ls, (forced_routing or {}).get(i))
            if routing is not None:
                routing[i] = idx.numpy().copy()
            if summaries is not None:
                summaries[f"model.decoder.transformer.layer[{i}].feed_forward/load_balance_loss"] = lbl
        else:
            f = feed_forward(n2, lp["feed_forward"], ls)
        h = h + f
    h = rmsnorm(h, dec["output_norm"]["scale"], spec.out_eps)
    logits = h @ table.T
    logp = torch.log_softmax(logits[:, :-1, :], dim=-1)
    picked = torch.gather(logp, -1, tok[:, 1:, None])[..., 0]
    return -picked.mean()


# ------------------------------------------------------------------------------------
# state helpers + training step
# ------------------------------------------------------------------------------------
def to_torch(tree, requires_grad=False, dtype=F64):
    if isinstance(tree, dict):
        return {k: to_torch(v, requires_grad, dtype) for k, v in tree.items()}
    t = torch.tensor(np.asarray(tree, dtype=np.float64), dtype=dtype)
    if requires_grad:
        t.requires_grad_(True)
    return t


def to_numpy(tree):
    if isinstance(tree, dict):
        return {k: to_numpy(v) for k, v in tree.items()}
    return tree.detach().cpu().numpy()


def leaves(tree, prefix=""):
    if isinstance(tree, dict):
        for k in sorted(tree):
            yield from leaves(tree[k], f"{prefix}.{k}" if prefix else k)
    else:
        yield prefix, tree


def value_and_grad(state_np: dict, tokens: np.ndarray, spec: ModelSpec, forced_routing: dict | None = None,
                   dtype=F64, routing: dict | None = None):
    """dtype=torch.float32 runs the same restatement in fp32 arithmetic: the error of a plain
    fp32 implementation against the f64 oracle (what the fp32-mode parity tests measure the
    GPU's error against)."""
    params = to_torch(state_np, requires_grad=True, dtype=dtype)
    summaries: dict = {}
    loss = forward_loss(params, tokens, spec, summaries, forced_routing, routing)
    loss.backward()

    def grads(t):
        if isinstance(t, dict):
            return {k: grads(v) for k, v in t.items()}
        return (t.grad if t.grad is not None else torch.zeros_like(t)).double().numpy()

    return float(loss.detach()), grads(params), summaries


class bf16_operands:
    """Context manager: every ``@`` in the restatement rounds its two operands to bf16 (f64
    accumulation, everything else f64) — the least rounding any bf16-operand GEMM path
    performs.  Used to show which bf16-mode errors are intrinsic to bf16 operands rather than
    to a kernel (tests/test_step_gpu.py)."""

    _orig = torch.Tensor.__matmul__

    def __enter__(self):
        orig = bf16_operands._orig

        def mm(a, b):
            return orig(a.to(torch.bfloat16).to(a.dtype), b.to(torch.bfloat16).to(b.dtype))

        torch.Tensor.__matmul__ = mm
        return self

    def __exit__(self, *exc):
        torch.Tensor.__matmul__ = bf16_operands._orig
        return False


@dataclass
class AdamW:
    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


def adamw_update(p, g, m, v, step: int, opt: AdamW):
    """One AdamW step on numpy float64 arrays; returns (p, m, v)."""
    m = opt.beta1 * m + (1 - opt.beta1) * g
    v = opt.beta2 * v + (1 - opt.beta2) * g * g
    mh = m / (1 - opt.beta1 ** step)
    vh = v / (1 - opt.beta2 ** step)
    p = p - opt.lr * (mh / (np.sqrt(vh) + opt.eps) + opt.weight_decay * p)
    return p, m, v


def train_step(state_np: dict, tokens: np.ndarray, spec: ModelSpec, opt: AdamW, m=None, v=None, step: int = 1,
               forced_routing: dict | None = None, dtype=F64, routing: dict | None = None):
    """Returns loss, grads, new_state, new_m, new_v, summaries (nested numpy dicts)."""
    loss, grads, summaries = value_and_grad(state_np, tokens, spec, forced_routing, dtype, routing)

    def walk(p, g, mm, vv):
        if isinstance(p, dict):
            outs = {k: walk(p[k], g[k], None if mm is None else mm[k], None if vv is None else vv[k]) for k in p}
            return ({k: o[0] for k, o in outs.items()}, {k: o[1] for k, o in outs.items()},
                    {k: o[2] for k, o in outs.items()})
        mm = np.zeros_like(p) if mm is None else mm
        vv = np.zeros_like(p) if vv is None else vv
        return adamw_update(p, g, mm, vv, step, opt)

    new_p, new_m, new_v = walk(state_np, grads, m, v)
    return loss, grads, new_p, new_m, new_v, summaries
