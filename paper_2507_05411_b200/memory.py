"""Per-GPU memory: the reference's AOT prediction next to what the engine holds.

``aot_device_bytes`` restates the memory half of the reference's ``aot_analyze``
(/root/reference/pkg/src/composer/mesh.py:563-686) for a one-axis ``("fsdp",)`` mesh of
``devices`` GPUs: parameter shards in the node's compute dtype (``shard_shape``,
mesh.py:107-122; ``param_bytes += shard_b``, :619-626), optimizer state =
``optimizer_state_multiplier`` x parameter bytes (:653-654), and saved activations =
the bytes of every remat tag whose governing policy decides "save" (:630-640, decisions by
``decide_tag``), divided by ``devices`` (:648).  It is used for reporting only (bench.py
prints it beside ``torch.cuda.max_memory_allocated``).

The engine's own accounting differs by design and is reported separately
(``TrainEngine.state_bytes``): f32 master weights and f32 AdamW moments (12 B/param / N)
instead of compute-dtype optimizer state, plus the bf16 working copy and gradient buffers.
"""

from __future__ import annotations

import math

from .remat import SAVE, decide_tag, resolve_policy

DTYPE_BYTES = {"f32": 4, "bf16": 2, "int8": 1, "fp8": 1}  # mesh.py:33


def _shard(shape, spec, devices: int) -> tuple:
    out = []
    for dim, axis in zip(shape, tuple(spec) + (None,) * (len(shape) - len(tuple(spec)))):
        out.append(dim // devices if axis == "fsdp" and dim % devices == 0 else dim)
    return tuple(out)


def aot_device_bytes(module, batch: int, seq_len: int, devices: int) -> dict:
    """module: an instantiated Trainer; batch: the GLOBAL batch (sequences)."""
    cfg = module.config
    mult = cfg.get("optimizer_state_multiplier") if cfg.has_field("optimizer_state_multiplier") else 2
    tot = {"param": 0, "saved": 0.0, "offload": 0.0}

    def walk(m, policy):
        mcfg = m.config
        if mcfg.has_field("remat_policy") and mcfg.get("remat_policy"):
            policy = resolve_policy(mcfg.get("remat_policy"))
        dsize = DTYPE_BYTES[mcfg.get("dtype")] if mcfg.has_field("dtype") else 4
        specs = m.behavior.param_specs(mcfg)
        for name, shape in m.behavior.param_shapes(mcfg).items():
            spec = specs.get(name, (None,) * len(shape))
            tot["param"] += math.prod(_shard(shape, spec, devices)) * dsize
        for tag in m.behavior.remat_tags(mcfg, batch, seq_len):
            d = decide_tag(tag.name, policy) if policy else SAVE
            if d == SAVE:
                tot["saved"] += tag.saved_bytes
            elif d == "offload":
                tot["offload"] += tag.saved_bytes
        for c in m.children.values():
            walk(c, policy)

    walk(module, None)
    saved = int(tot["saved"] // devices)
    return {"param_bytes": tot["param"], "optimizer_bytes": mult * tot["param"], "saved_activation_bytes": saved,
            "per_device_bytes": tot["param"] * (1 + mult) + saved,
            "formula": "reference aot_analyze (mesh.py:563-686): compute-dtype param shards x (1 + optimizer "
                       "multiplier) + saved remat-tag activations / devices"}
