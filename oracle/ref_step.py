"""Times the REFERENCE's own CPU step — BASELINE INFRASTRUCTURE ONLY.

Only ``bench.py --impl reference`` / its ``cpu_baseline`` leg and ``tests/`` may import
this module.  It never runs on the product path.

What it times: the reference's ``invoke(module, state, key, batch)``
(/root/reference/pkg/src/composer/module.py:351-365) — its forward pass and loss; the
reference has no backward or optimizer — on the unmodified reference
package installed (``oracle/build_ref.sh``) into ``oracle/_ref`` (git-ignored; it travels
to the GPU box with the snapshot like the built ``.so`` files).  A full 1B/7B reference
step would need 7-53 GB of float64 weights, so the sample is:

* one reference ``TransformerLayer`` at the config's layer shape, batch 1, seq T
  (``invoke`` on the layer module with a [1, T, d] float64 input), and
* the reference ``Trainer`` with zero layers at batch 1, seq T (embedding gather, output
  norm, tied head over the full vocab, log-softmax loss — ``layers.py:573-651``),

combined as ``t_step = t_head + L * t_layer`` for T tokens.  The 70B-layer shape uses the
reference's only attention kind (MHA: the reference has no GQA) at T=1024, and the MoE
layer T=256 (the reference's ``np.einsum`` expert path, ``layers.py:519-525``, takes >25 min
at T=4096) — both per BASELINE.md §2.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

# layer shapes of the bench workloads (must match
# paper_2507_05411_b200.experiments.BENCH_CONFIGS)
SHAPES = {
    "tiny": dict(dim=128, heads=4, ffn=None, layers=2, vocab=64, seq=256, batch=8),
    "1b": dict(dim=2048, heads=16, ffn=5632, layers=16, vocab=32000, seq=4096, batch=1),
    "7b": dict(dim=4096, heads=32, ffn=11008, layers=32, vocab=32000, seq=4096, batch=1),
    "moe": dict(dim=2048, heads=16, ffn=5632, layers=8, vocab=32000, seq=256, batch=1, experts=8, top_k=2),
    "70b_layer": dict(dim=8192, heads=64, ffn=28672, layers=4, vocab=32000, seq=1024, batch=1),
}


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "composer"))


def load():
    """Imports the reference package from oracle/_ref (raises ImportError if absent)."""
    if not available():
        raise ImportError("oracle/_ref/composer missing: run oracle/build_ref.sh where /root/reference exists")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import composer

    if not os.path.abspath(composer.__file__).startswith(REF_DIR):
        raise ImportError(f"composer imported from {composer.__file__}, not oracle/_ref")
    return composer


def _layer_cfg(c, sh):
    swiglu = ("linear", "silu")
    layer = (c.default_config("TransformerLayer")
             .set("input_dim", sh["dim"])
             .set("self_attention.num_heads", sh["heads"])
             .set("self_attention.pos_emb", c.default_config("RoPE")))
    if sh.get("experts"):
        layer = layer.set("feed_forward", c.default_config("MoE").set("num_experts", sh["experts"])
                          .set("top_k", sh["top_k"]).set("activation", swiglu).set("hidden_dim", sh["ffn"]))
    elif sh["ffn"] is None:  # tiny: scaled_hidden_dim(8/3) as experiments.py:39
        layer = (layer.set("feed_forward.activation", swiglu)
                 .set("feed_forward.hidden_dim", c.FunctionSpec("scaled_hidden_dim", scale=8.0 / 3.0)))
    else:
        layer = layer.set("feed_forward.activation", swiglu).set("feed_forward.hidden_dim", sh["ffn"])
    return layer


def _trainer_cfg(c, sh, layers: int):
    lc = _layer_cfg(c, sh)
    return (c.default_config("Trainer").set("model.dim", sh["dim"]).set("model.vocab_size", sh["vocab"])
            .set("model.decoder.transformer.layer", (lc,) * layers).set("learner.lr", 1e-3))


def time_invoke(c, module, state, key, *args) -> float:
    t0 = time.perf_counter()
    c.invoke(module, state, key, *args)
    return time.perf_counter() - t0


class ReferenceStep:
    """The reference's CPU step at `config`, prepared once (modules, init_state, inputs) so
    samples time only `invoke`: `layer()` times one TransformerLayer invoke, `head()` the 0-layer
    Trainer invoke, and `rate(t_head, t_layer)` extrapolates tokens/s for the full depth."""

    def __init__(self, config: str):
        c = self.c = load()
        sh = self.sh = SHAPES[config]
        self.config = config
        B, T = sh["batch"], sh["seq"]
        root = c.root_key(0)
        self.key = c.child_key(root, "step", 0)
        from composer.experiments import synthetic_batch

        self.toks = synthetic_batch(0, 0, B, T, sh["vocab"])
        if config == "tiny":  # the full reference step
            self.full = c.instantiate(_trainer_cfg(c, sh, sh["layers"]))
            self.full_state = c.init_state(self.full, root)
            return
        self.lm = c.instantiate(_layer_cfg(c, sh))
        self.lst = c.init_state(self.lm, root)
        self.x = np.random.default_rng(0).standard_normal((B, T, sh["dim"]))
        self.hm = c.instantiate(_trainer_cfg(c, sh, 0))
        self.hst = c.init_state(self.hm, root)

    def layer(self) -> float:
        if self.config == "tiny":
            return time_invoke(self.c, self.full, self.full_state, self.key, self.toks)
        return time_invoke(self.c, self.lm, self.lst, self.key, self.x)

    def head(self) -> float:
        return 0.0 if self.config == "tiny" else time_invoke(self.c, self.hm, self.hst, self.key, self.toks)

    def rate(self, t_head: float, t_layer: float) -> float:
        sh = self.sh
        t_step = t_layer if self.config == "tiny" else t_head + sh["layers"] * t_layer
        return sh["batch"] * sh["seq"] / t_step

    def describe(self, t_head: float, t_layer: float) -> str:
        sh = self.sh
        if self.config == "tiny":
            return f"reference invoke: full tiny step, {sh['batch']}x{sh['seq']} tokens, {t_layer:.2f} s"
        kind = "MoE" if sh.get("experts") else ("MHA (the reference has no GQA)" if self.config == "70b_layer" else "MHA")
        t_step = t_head + sh["layers"] * t_layer
        return (f"reference composer.invoke (forward + loss; the reference has no backward/optimizer): one "
                f"{self.config} TransformerLayer ({kind}, d={sh['dim']}) at batch {sh['batch']}, seq {sh['seq']}: "
                f"{t_layer:.2f} s; 0-layer Trainer (embedding, output norm, tied head V={sh['vocab']}, loss): "
                f"{t_head:.2f} s; step = head + {sh['layers']} x layer = {t_step:.1f} s per {sh['batch'] * sh['seq']} "
                f"tokens")


def reference_sample(config: str) -> dict:
    """One bounded sample of the reference's CPU step at `config` (a head and a layer invoke)."""
    r = ReferenceStep(config)
    t_head, t_layer = r.head(), r.layer()
    return {"value": r.rate(t_head, t_layer), "t_layer_s": t_layer, "t_head_s": t_head,
            "sample": r.describe(t_head, t_layer)}
