"""Experiment registry and synthetic data (reference experiments.py:37-206), plus the
BASELINE.json benchmark configurations built through the same config API.

The 27 ``txf_*`` builders produce configs identical to the reference's (same fields,
same embedded mesh rules as plain data) — they are the parity corpus.  The
``bench_*`` builders are the north-star shapes (tiny / 1B / 7B / MoE / 70B-layer).
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .config import ConfigNode, FunctionSpec, default_config
from .errors import UnknownExperimentError
from .prng import child_key, generator, root_key

VOCAB_SIZE = 64
SWIGLU = ("linear", "silu")
SWIGLU_SCALE = 8.0 / 3.0

# The reference's DEFAULT_MESH_RULES in their plain-data form (reference experiments.py:44-62,
# rendered by mesh.rules_to_plain); mesh rules are config data, not code, in both packages.
DEFAULT_MESH_RULES_PLAIN = (
    {"match": "gpu-H100-*", "modifiers": (
        {"kind": "mesh_shape", "axes": {"fsdp": -1, "model": 8}},
        {"kind": "remat_spec", "policies": {"model.decoder.transformer.layer": {
            "*": "recompute", "context": "save", "k_proj": "save", "o_proj": "save", "q_proj": "save",
            "v_proj": "save"}}},
        {"kind": "dtype", "tag": "fp8", "params": {"fp8_amax_history_length": 128}})},
    {"match": "tpu-v5e-*", "modifiers": (
        {"kind": "mesh_shape", "axes": {"fsdp": 16, "model": -1}},
        {"kind": "remat_spec", "policies": {"model.decoder.transformer.layer": {"*": "offload"}}},
        {"kind": "dtype", "tag": "bf16", "params": {}})},
    {"match": "*", "modifiers": ({"kind": "mesh_shape", "axes": {"fsdp": -1}},)},
)

_HEADS_FOR_DIM = {16: 2, 32: 4, 48: 4, 64: 4}
EXPERIMENTS: dict[str, Callable[[], ConfigNode]] = {}


def register_experiment(name: str, builder: Callable[[], ConfigNode]) -> None:
    if name in EXPERIMENTS:
        raise UnknownExperimentError(f"experiment {name!r} already registered")
    EXPERIMENTS[name] = builder


def experiment_names() -> tuple[str, ...]:
    return tuple(sorted(EXPERIMENTS))


def build_experiment(name: str) -> ConfigNode:
    if name not in EXPERIMENTS:
        raise UnknownExperimentError(f"unknown experiment {name!r}")
    return EXPERIMENTS[name]()


def transformer_trainer(dim: int, num_layers: int, activation, hidden_scale: float | None = None,
                        feed_forward_kind: str = "FeedForward", pos_kind: str = "NoPos", num_experts: int = 4,
                        top_k: int = 2, heads: int | None = None, vocab: int = VOCAB_SIZE,
                        sharded=("fsdp", None)) -> ConfigNode:
    """The reference's _transformer_trainer builder (reference experiments.py:88-128)."""
    layer = (default_config("TransformerLayer")
             .set("self_attention.num_heads", heads if heads is not None else _HEADS_FOR_DIM[dim])
             .set("self_attention.param_partition_spec", sharded))
    if pos_kind != "NoPos":
        layer = layer.set("self_attention.pos_emb", default_config(pos_kind))
    if feed_forward_kind != "FeedForward":
        layer = layer.set("feed_forward", default_config(feed_forward_kind).set("num_experts", num_experts)
                          .set("top_k", top_k))
    layer = layer.set("feed_forward.activation", activation).set("feed_forward.param_partition_spec", sharded)
    if hidden_scale is not None:
        layer = layer.set("feed_forward.hidden_dim", FunctionSpec("scaled_hidden_dim", scale=hidden_scale))
    return (default_config("Trainer")
            .set("model.dim", dim)
            .set("model.vocab_size", vocab)
            .set("model.decoder.emb.param_partition_spec", sharded)
            .set("model.decoder.transformer.layer", (layer,) * num_layers)
            .set("learner.lr", 1e-3)
            .set("mesh_rules", DEFAULT_MESH_RULES_PLAIN))


def _register_builtin() -> None:
    register_experiment("txf_base", lambda: transformer_trainer(32, 2, SWIGLU, hidden_scale=SWIGLU_SCALE))
    register_experiment("txf_moe", lambda: transformer_trainer(32, 2, SWIGLU, hidden_scale=SWIGLU_SCALE,
                                                               feed_forward_kind="MoE"))
    register_experiment("txf_rope", lambda: transformer_trainer(32, 2, SWIGLU, hidden_scale=SWIGLU_SCALE,
                                                                pos_kind="RoPE"))
    for dim in (16, 32, 48, 64):
        for layers in (1, 2, 3):
            register_experiment(f"txf_d{dim}_l{layers}_relu",
                                lambda dim=dim, layers=layers: transformer_trainer(dim, layers, "relu"))
            register_experiment(f"txf_d{dim}_l{layers}_swiglu",
                                lambda dim=dim, layers=layers: transformer_trainer(dim, layers, SWIGLU,
                                                                                   hidden_scale=SWIGLU_SCALE))


_register_builtin()


def synthetic_batch(seed: int, step: int, batch_size: int, seq_len: int, vocab_size: int = VOCAB_SIZE) -> dict:
    """tokens = PCG64(child_key(root_key(seed), "data", step)).integers(0, V) (reference experiments.py:199-206)."""
    gen = generator(child_key(root_key(seed), "data", step))
    return {"tokens": gen.integers(0, vocab_size, size=(batch_size, seq_len), dtype=np.int64)}


# ----------------------------------------------------------------------------------
# BASELINE.json configurations, composed with the same API
# ----------------------------------------------------------------------------------
def _llama_layer(dim: int, heads: int, ffn: int, kv_heads: int | None = None) -> ConfigNode:
    layer = default_config("TransformerLayer")
    if kv_heads is not None and kv_heads != heads:
        layer = layer.set("self_attention", default_config("GroupedQueryAttention").set("num_kv_heads", kv_heads))
    layer = (layer.set("self_attention.num_heads", heads)
             .set("self_attention.param_partition_spec", ("fsdp", None))
             .set("self_attention.pos_emb", default_config("RoPE"))
             .set("feed_forward.activation", SWIGLU)
             .set("feed_forward.hidden_dim", ffn)
             .set("feed_forward.param_partition_spec", ("fsdp", None)))
    return layer


def _llama_trainer(dim, layers, heads, ffn, vocab, batch, seq, kv_heads=None, dtype="bf16") -> ConfigNode:
    from .engine import set_dtype_policy

    cfg = (default_config("Trainer")
           .set("model.dim", dim)
           .set("model.vocab_size", vocab)
           .set("model.decoder.emb.param_partition_spec", ("fsdp", None))
           .set("model.decoder.transformer.layer", (_llama_layer(dim, heads, ffn, kv_heads),) * layers)
           .set("learner.lr", 1e-3)
           .set("batch_size", batch)
           .set("seq_len", seq)
           .set("mesh_axis_names", ("fsdp",))
           .set("mesh_rules", DEFAULT_MESH_RULES_PLAIN))
    return set_dtype_policy(cfg, dtype)


def bench_tiny(dtype: str = "f32", batch: int = 8, seq: int = 256, layers: int = 2) -> ConfigNode:
    """configs[0]: 2 layers, d=128, 4 heads, RoPE, SwiGLU (8/3), seq 256, batch 8, V=64."""
    from .engine import set_dtype_policy

    layer = (default_config("TransformerLayer").set("self_attention.num_heads", 4)
             .set("self_attention.pos_emb", default_config("RoPE"))
             .set("feed_forward.activation", SWIGLU)
             .set("feed_forward.hidden_dim", FunctionSpec("scaled_hidden_dim", scale=SWIGLU_SCALE)))
    cfg = (default_config("Trainer").set("model.dim", 128).set("model.vocab_size", 64)
           .set("model.decoder.transformer.layer", (layer,) * layers).set("learner.lr", 1e-3)
           .set("batch_size", batch).set("seq_len", seq))
    return set_dtype_policy(cfg, dtype)


def bench_1b(batch: int = 8, seq: int = 4096, dtype: str = "bf16", layers: int = 16) -> ConfigNode:
    """configs[1]: Llama-style 1B — 16 layers, d=2048, 16 heads, ffn 5632, V=32000, seq 4096."""
    return _llama_trainer(2048, layers, 16, 5632, 32000, batch, seq, dtype=dtype)


def bench_7b(batch: int = 2, seq: int = 4096, dtype: str = "bf16", layers: int = 32) -> ConfigNode:
    """configs[2]: Llama2-7B shape — 32 layers, d=4096, 32 heads, ffn 11008, V=32000."""
    return _llama_trainer(4096, layers, 32, 11008, 32000, batch, seq, dtype=dtype)


def bench_moe(batch: int = 4, seq: int = 4096, dtype: str = "bf16", layers: int = 8) -> ConfigNode:
    """configs[3]: MoE decoder — d=2048, 8 experts, top-2, SwiGLU h=5632."""
    from .engine import set_dtype_policy

    layer = (_llama_layer(2048, 16, 5632)
             .set("feed_forward", default_config("MoE").set("num_experts", 8).set("top_k", 2)
                  .set("activation", SWIGLU).set("hidden_dim", 5632).set("param_partition_spec", ("fsdp", None))))
    cfg = (default_config("Trainer").set("model.dim", 2048).set("model.vocab_size", 32000)
           .set("model.decoder.transformer.layer", (layer,) * layers).set("learner.lr", 1e-3)
           .set("batch_size", batch).set("seq_len", seq).set("mesh_axis_names", ("fsdp",)))
    return set_dtype_policy(cfg, dtype)


def bench_70b_layer(batch: int = 1, seq: int = 4096, dtype: str = "bf16", layers: int = 4) -> ConfigNode:
    """configs[4]: Llama2-70B layer shape — d=8192, GQA 64q/8kv, ffn 28672, reduced depth."""
    return _llama_trainer(8192, layers, 64, 28672, 32000, batch, seq, kv_heads=8, dtype=dtype)


BENCH_CONFIGS = {"tiny": bench_tiny, "1b": bench_1b, "7b": bench_7b, "moe": bench_moe, "70b_layer": bench_70b_layer}
