"""Component kinds of the decoder step: reference schemas + B200 execution.

Each kind is registered exactly as the reference registers it (same kind name, same
fields, kinds and defaults — reference layers.py:671-796) so reference configs and
golden files drive this package unchanged; the metadata hooks (param shapes, partition
specs, init, FLOPs, remat tags) return what the reference's do.  What differs is
execution: ``forward`` runs the step on the GPU through ``ops`` (one C-ABI kernel call
per operation, no PyTorch arithmetic, no CPU fallback) and every differentiable kind
also has a ``backward``.

Precision (``options['precision']``): "f32" runs every contraction in f32 (SIMT GEMM,
SIMT attention) — the 1e-5 parity mode; "bf16" runs tcgen05 GEMMs and tensor-core
attention on bf16 operands with f32 accumulation, an f32 residual stream, f32
statistics and f32 gradients/master weights — the 2e-2 mode.

Fused parameter layout: the engine stores an attention block's wq|wk|wv (and an FFN's
w1|w1_gate) as column slices of one [d, 3d] ([d, 2h]) matrix; the behaviors detect it
and issue one wide GEMM instead of three (two).  Plain separate tensors still work.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .config import ComponentSchema, ConfigNode, FieldSpec, FunctionSpec, ValueKind, register_component, register_factory
from .errors import BadPathError, BadTopKError, OddDimError, ShapeError, TypeMismatchError, UnknownActivationError
from .module import (
    Behavior,
    RematTag,
    add_summary,
    backward_child,
    current_context,
    get_shared_grad,
    get_shared_state,
    invoke_child,
    is_recording,
    param,
    param_grad,
    param_key,
    register_behavior,
    register_spec_function,
    save,
    saved,
)
from .prng import RngKey, uniform
from .remat import OFFLOAD, RECOMPUTE, SAVE, decide_tag, resolve_policy

DTYPE_BYTES = {"f32": 4, "bf16": 2, "int8": 1, "fp8": 1}
ACTIVATION_NAMES = ("linear", "relu", "silu", "sigmoid", "tanh")
_TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16}


# ------------------------------------------------------------------ shared helpers
def option(name: str, default=None):
    return current_context().options.get(name, default)


def act_dtype() -> torch.dtype:
    return _TORCH_DT[option("precision", "f32")]


# ------------------------------------------------------------- rematerialisation
def remat_decision(tag: str) -> str:
    """The governing decision for one of the current module's remat tags: the policy of the
    nearest enclosing module with a non-empty ``remat_policy`` (inherited down the tree as
    the reference's aot_analyze does, mesh.py:601-611), applied by ``decide_tag``
    (mesh.py:240-252: exact key, then the longest matching glob, default save)."""
    ctx = current_context()
    while ctx is not None:
        cfg = ctx.module.config
        if cfg.has_field("remat_policy"):
            pol = cfg.get("remat_policy")
            if pol:
                return decide_tag(tag, resolve_policy(pol))
        ctx = ctx.parent
    return SAVE


def remat_plan(*tags: str) -> str:
    """One decision for a group of tags that share a tensor (e.g. q_proj/k_proj/v_proj: the
    fused qkv buffer): recompute if any tag recomputes, else offload if any offloads, else
    save.  Only meaningful while recording (a forward-only call saves nothing)."""
    ds = {remat_decision(t) for t in tags}
    return RECOMPUTE if RECOMPUTE in ds else (OFFLOAD if OFFLOAD in ds else SAVE)


_D2H: dict = {}


class Offloaded:
    """A saved activation parked in pinned host memory (remat decision "offload"): copied out
    by the copy engine on a side stream right after it is produced (the device block is
    released when that copy completes), copied back on the consumer's stream in backward."""

    def __init__(self, t: torch.Tensor):
        dev = t.device
        st = _D2H.get(dev)
        if st is None:
            st = _D2H[dev] = torch.cuda.Stream(dev)
        self.device = dev
        self.host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(st):
            st.wait_event(ready)
            self.host.copy_(t, non_blocking=True)
            t.record_stream(st)
            self.done = torch.cuda.Event()
            self.done.record(st)

    def load(self) -> torch.Tensor:
        torch.cuda.current_stream(self.device).wait_event(self.done)
        return self.host.to(self.device, non_blocking=True)


def keep(t, decision: str):
    """What a forward saves for `t` under a remat decision (None = recompute in backward)."""
    if t is None or decision == SAVE:
        return t
    if decision == OFFLOAD:
        return Offloaded(t)
    return None


def restore(v):
    return v.load() if isinstance(v, Offloaded) else v


def check_activation(name) -> None:
    if name not in ACTIVATION_NAMES:
        raise UnknownActivationError(f"unknown activation {name!r}")


def activation_pair(value):
    """(linear_branch, gate_branch) for gated configs, None for a single name (layers.py:99-105)."""
    if isinstance(value, str):
        return None
    if isinstance(value, tuple) and len(value) == 2 and all(isinstance(a, str) for a in value):
        return value
    raise ShapeError(f"activation must be a name or a pair of names, got {value!r}")


def scaled_hidden_dim(fields, scale: float) -> int:
    """floor(input_dim * scale + 0.5) (layers.py:91-96)."""
    base = fields.get("input_dim")
    if not isinstance(base, int) or isinstance(base, bool):
        raise ValueError("input_dim is not set yet")
    return int(math.floor(base * scale + 0.5))


def fan_in_uniform(key: RngKey, shape, fan_in: int) -> np.ndarray:
    bound = 1.0 / math.sqrt(fan_in)
    return uniform(key, -bound, bound, tuple(shape))


def uniform_spec(fan_in: int) -> tuple:
    """param_init entry equivalent to fan_in_uniform (layers.py:114-116)."""
    bound = 1.0 / math.sqrt(fan_in)
    return ("uniform", -bound, bound)


def _pspec(cfg):
    return tuple(cfg.get("param_partition_spec"))


def _dbytes(cfg):
    return DTYPE_BYTES[cfg.get("dtype")]


def infer_bias_spec(spec) -> tuple:
    spec = tuple(spec)
    if not spec:
        raise ShapeError("weight spec must have at least one entry")
    return (spec[-1],)


def fused_columns(*views: torch.Tensor) -> torch.Tensor | None:
    """If `views` are adjacent column slices of one row-major matrix, return that matrix."""
    first = views[0]
    if first.dim() != 2 or first.stride(1) != 1:
        return None
    total = 0
    for v in views:
        if v.dim() != 2 or v.stride() != first.stride() or v.shape[0] != first.shape[0] or v.dtype != first.dtype:
            return None
        if v.data_ptr() != first.data_ptr() + total * first.element_size():
            return None
        total += v.shape[1]
    if total > first.stride(0):
        return None
    return first.as_strided((first.shape[0], total), first.stride())


def _checked_3d(x: torch.Tensor, dim: int, who: str):
    if not isinstance(x, torch.Tensor) or x.dim() != 3 or x.shape[-1] != dim:
        raise ShapeError(f"{who} expects [batch, seq, {dim}] input")
    return x.shape[0], x.shape[1]


def _out_f32(rows, cols, device):
    return torch.empty((rows, cols), device=device, dtype=torch.float32)


def _linear_fwd(x2: torch.Tensor, w: torch.Tensor, out_dtype: torch.dtype) -> torch.Tensor:
    out = torch.empty((x2.shape[0], w.shape[1]), device=x2.device, dtype=out_dtype)
    return ops.gemm(x2, w, out)


def _wave_efficiency(m: int, n: int, tile: int = 256, units: int = 74) -> float:
    """Busy fraction of the CTA-pair GEMM's waves for an m x n output (256 x 256 tiles over
    74 SM pairs): 1B step QKV / wo wgrad 0.86, w2 0.79, w1|w1_gate 0.95; 7B wo 0.86, others >= 0.93."""
    tiles = -(-m // tile) * -(-n // tile)
    waves = -(-tiles // units)
    return tiles / (waves * units)


def _wgrad(x2: torch.Tensor, dy: torch.Tensor, dw: torch.Tensor) -> None:
    """dw += x2^T dy.  With the engine's weight-gradient stream (option "wgrad_stream") the
    product runs there, beside the data-gradient chain: weight gradients have few output tiles
    (1B step: QKV 192, w2 176, wo 64 CTA-pair tiles over 74 pairs, K = all tokens), so their
    last wave leaves SMs idle that the next data-gradient / attention kernel fills.  Only those
    whose waves are less than option "wgrad_wave_eff" busy go there: on the power-capped B200
    the extra concurrency lowers the SM clock (7B step with every wgrad on the side stream:
    -1%, 1376 -> 1316 MHz), so it pays only where there is a real tail to fill.  At most
    option "wgrad_depth" weight gradients are in flight: beyond that the compute stream waits
    for the oldest, whose operands are then released in compute-stream order (no record_stream:
    its deferred frees made the caching allocator thrash on the memory-tight 7B step).  The
    engine's update / reduce-scatter of a bucket waits for this stream (engine._join_wgrad)."""
    ws = option("wgrad_stream")
    if ws is not None and _wave_efficiency(dw.shape[0], dw.shape[1]) >= option("wgrad_wave_eff", 0.9):
        ws = None  # a full last wave: nothing to fill, and concurrent kernels only raise power
    if ws is None:
        ops.gemm(x2, dy, dw, trans_a=True, accumulate=True)
        return
    cur = torch.cuda.current_stream(x2.device)
    pending = option("wgrad_pending")  # [(done event, operands)] of the GEMMs in flight
    while len(pending) >= option("wgrad_depth", 1):
        cur.wait_event(pending.pop(0)[0])
    ready = torch.cuda.Event()
    ready.record(cur)
    ws.wait_event(ready)
    with torch.cuda.stream(ws):
        ops.gemm(x2, dy, dw, trans_a=True, accumulate=True)
    done = torch.cuda.Event()
    done.record(ws)
    pending.append((done, (x2, dy)))


def _linear_bwd(x2: torch.Tensor, w: torch.Tensor, dy: torch.Tensor, dw: torch.Tensor | None, dx_dtype):
    """dw += x^T dy ; returns dx = dy w^T (dy already in the operand dtype)."""
    if dw is not None:
        _wgrad(x2, dy, dw)
    dx = torch.empty((dy.shape[0], w.shape[0]), device=dy.device, dtype=dx_dtype)
    return ops.gemm(dy, w, dx, trans_b=True)


# ------------------------------------------------------------------------- Linear
class LinearBehavior(Behavior):
    """y = x @ weight + bias, weight [in, out] (reference layers.py:130-170)."""

    def param_shapes(self, cfg):
        shapes = {"weight": (cfg.get("input_dim"), cfg.get("output_dim"))}
        if cfg.get("bias"):
            shapes["bias"] = (cfg.get("output_dim"),)
        return shapes

    def param_specs(self, cfg):
        spec = _pspec(cfg)
        specs = {"weight": spec}
        if cfg.get("bias"):
            specs["bias"] = infer_bias_spec(spec)
        return specs

    def init_params(self, cfg, key):
        out = {"weight": fan_in_uniform(param_key(key, "weight"), self.param_shapes(cfg)["weight"], cfg.get("input_dim"))}
        if cfg.get("bias"):
            out["bias"] = np.zeros((cfg.get("output_dim"),), dtype=np.float64)
        return out

    def param_init(self, cfg):
        out = {"weight": uniform_spec(cfg.get("input_dim"))}
        if cfg.get("bias"):
            out["bias"] = ("const", 0.0)
        return out

    def own_flops(self, cfg, batch, seq_len):
        return 2 * batch * seq_len * cfg.get("input_dim") * cfg.get("output_dim")

    def remat_tags(self, cfg, batch, seq_len):
        rows = batch * seq_len
        return [RematTag("output", rows * cfg.get("output_dim") * _dbytes(cfg), self.own_flops(cfg, batch, seq_len))]

    def forward(self, module, x):
        cfg = module.config
        if x.shape[-1] != cfg.get("input_dim"):
            raise ShapeError(f"Linear expects trailing dim {cfg.get('input_dim')}, got {x.shape[-1]}")
        lead = x.shape[:-1]
        x2 = ops.cast(ops.rows2d(x), act_dtype())
        y = _linear_fwd(x2, param("weight"), torch.float32)
        if cfg.get("bias"):
            ones = torch.ones((1, y.shape[0]), device=y.device, dtype=torch.float32)
            ops.gemm(ones.t().contiguous(), param("bias").view(1, -1).float(), y, accumulate=True)
        save(x2=x2)
        return y.view(*lead, y.shape[-1])

    def backward(self, module, dy):
        s = saved()
        g = ops.cast(ops.rows2d(dy), act_dtype())
        if module.config.get("bias"):
            ones = torch.ones((g.shape[0], 1), device=g.device, dtype=g.dtype)
            ops.gemm(ones, g, param_grad("bias").view(1, -1), trans_a=True, accumulate=True)
        dx = _linear_bwd(s["x2"], param("weight"), g, param_grad("weight"), torch.float32)
        return dx.view(*dy.shape[:-1], dx.shape[-1])


# ------------------------------------------------------------------------ RMSNorm
class RMSNormBehavior(Behavior):
    """x / sqrt(mean(x^2) + eps) * scale (reference layers.py:176-193)."""

    def param_shapes(self, cfg):
        return {"scale": (cfg.get("input_dim"),)}

    def param_specs(self, cfg):
        return {"scale": (None,)}

    def init_params(self, cfg, key):
        return {"scale": np.ones((cfg.get("input_dim"),), dtype=np.float64)}

    def param_init(self, cfg):
        return {"scale": ("const", 1.0)}

    def forward(self, module, x):
        cfg = module.config
        if x.shape[-1] != cfg.get("input_dim"):
            raise ShapeError(f"RMSNorm expects trailing dim {cfg.get('input_dim')}")
        scale = param("scale")
        y, rstd = ops.rmsnorm_fwd(x, _f32(scale), cfg.get("eps"), act_dtype())
        save(x=x, rstd=rstd)
        return y

    def backward(self, module, dy, dres=None):
        """dres: gradient arriving on the residual branch of the same input (fused add).

        In bf16 mode the same pass also writes the bf16 copy of dx that the next
        backward GEMM consumes (attached as ``dx._bf16``; ``ops.cast`` picks it up).
        """
        s = saved()
        want = act_dtype() == torch.bfloat16
        out = ops.rmsnorm_bwd(s["x"], _f32(param("scale")), s["rstd"], dy, dres=dres, dscale=param_grad("scale"),
                              want_bf16=want)
        if want:
            dx, dxb = out
            dx._bf16 = dxb
            return dx
        return out


def _f32(t: torch.Tensor) -> torch.Tensor:
    return t if t.dtype == torch.float32 else t.float()


# ---------------------------------------------------------------------- Embedding
class EmbeddingBehavior(Behavior):
    """Token id -> row of an [num_embeddings, dim] table (reference layers.py:199-229)."""

    def param_shapes(self, cfg):
        return {"weight": (cfg.get("num_embeddings"), cfg.get("dim"))}

    def param_specs(self, cfg):
        return {"weight": _pspec(cfg)}

    def init_params(self, cfg, key):
        return {"weight": fan_in_uniform(param_key(key, "weight"), self.param_shapes(cfg)["weight"], cfg.get("dim"))}

    def param_init(self, cfg):
        return {"weight": uniform_spec(cfg.get("dim"))}

    def remat_tags(self, cfg, batch, seq_len):
        return [RematTag("output", batch * seq_len * cfg.get("dim") * _dbytes(cfg), 0)]

    def forward(self, module, ids):
        cfg = module.config
        if not isinstance(ids, torch.Tensor) or ids.dtype not in (torch.int64, torch.int32):
            raise ShapeError("Embedding expects integer token ids")
        if ids.dtype != torch.int64:
            raise ShapeError("Embedding expects int64 token ids on the device")
        vocab = cfg.get("num_embeddings")
        if option("validate_ids", True) and ids.numel():
            lo, hi = int(ids.min()), int(ids.max())  # host sync; the engine validates on the host instead
            if lo < 0 or hi >= vocab:
                raise ShapeError(f"token ids out of range [0, {vocab})")
        out = ops.embedding_fwd(ids, param("weight"), torch.float32)
        sort = None
        if ids.is_cuda and is_recording():
            # the backward's deterministic id sort depends only on the ids: run it now on a side
            # stream, hidden behind the forward
            side = _sort_stream(ids.device)
            ready = torch.cuda.Event()
            ready.record()
            side.wait_event(ready)
            with torch.cuda.stream(side):
                offsets, perm = ops.sort_ids(ids, vocab)
                done = torch.cuda.Event()
                done.record(side)
            sort = (offsets, perm, done)
        save(ids=ids, sort=sort)
        return out

    def backward(self, module, dout):
        s = saved()
        if s.get("sort") is not None:
            offsets, perm, done = s["sort"]
            cur = torch.cuda.current_stream(dout.device)
            cur.wait_event(done)
            offsets.record_stream(cur)  # allocated on the side stream, consumed on this one
            perm.record_stream(cur)
        else:
            offsets, perm = ops.sort_ids(s["ids"], module.config.get("num_embeddings"))
        ops.embedding_bwd(offsets, perm, dout, param_grad("weight"))
        return None


_SORT_STREAMS: dict = {}


def _sort_stream(device) -> torch.cuda.Stream:
    if device not in _SORT_STREAMS:
        _SORT_STREAMS[device] = torch.cuda.Stream(device)
    return _SORT_STREAMS[device]


# -------------------------------------------------------------- positional kinds
_ROPE_CACHE: dict = {}


def rope_tables(seq_len: int, dim: int, base: float, device):
    """cos/sin [T, dim/2] computed in float64 on the host, stored f32."""
    key = (seq_len, dim, float(base), str(device))
    hit = _ROPE_CACHE.get(key)
    if hit is None:
        half = dim // 2
        freqs = base ** (-2.0 * np.arange(half) / dim)
        ang = np.arange(seq_len, dtype=np.float64)[:, None] * freqs[None, :]
        hit = (torch.tensor(np.cos(ang), dtype=torch.float32, device=device),
               torch.tensor(np.sin(ang), dtype=torch.float32, device=device))
        _ROPE_CACHE[key] = hit
    return hit


class NoPosBehavior(Behavior):
    """Identity positional embedding (reference layers.py:260-264)."""

    def forward(self, module, q, k, positions):
        return q, k

    def backward(self, module, dq, dk):
        return dq, dk


class RoPEBehavior(Behavior):
    """Rotary embedding on queries and keys, in place (reference layers.py:267-276).

    q / k are [B*T, heads*hd] row views; `positions` is the sequence length T (the
    reference passes arange(T), layers.py:343).
    """

    def validate(self, cfg):
        if cfg.get("dim") % 2:
            raise OddDimError(f"rotary embedding needs an even dim, got {cfg.get('dim')}")

    def _apply(self, module, q, k, seq_len, inverse):
        hd = module.config.get("dim")
        cs, sn = rope_tables(seq_len, hd, module.config.get("base"), q.device)
        ops.rope_(q, seq_len, q.shape[1] // hd, hd, cs, sn, inverse=inverse)
        ops.rope_(k, seq_len, k.shape[1] // hd, hd, cs, sn, inverse=inverse)

    def forward(self, module, q, k, positions):
        seq_len = int(positions) if not hasattr(positions, "__len__") else len(positions)
        self._apply(module, q, k, seq_len, False)
        save(seq_len=seq_len)
        return q, k

    def backward(self, module, dq, dk):
        self._apply(module, dq, dk, saved()["seq_len"], True)
        return dq, dk


# ---------------------------------------------------------------------- Attention
class AttentionBehavior(Behavior):
    """Unmasked multi-head attention with bias-free [d, d] projections (reference layers.py:282-348)."""

    def kv_heads(self, cfg) -> int:
        return cfg.get("num_heads")

    def propagate(self, cfg):
        dim, heads = cfg.get("input_dim"), cfg.get("num_heads")
        if isinstance(dim, int) and isinstance(heads, int):
            if heads < 1 or dim % heads:
                raise ShapeError(f"input_dim {dim} must divide into num_heads {heads}")
            cfg = cfg.set("pos_emb.dim", dim // heads)
        return cfg

    def param_shapes(self, cfg):
        d = cfg.get("input_dim")
        kv = d // cfg.get("num_heads") * self.kv_heads(cfg)
        return {"wq": (d, d), "wk": (d, kv), "wv": (d, kv), "wo": (d, d)}

    def param_specs(self, cfg):
        spec = _pspec(cfg)
        rev = tuple(reversed(spec))
        return {"wq": spec, "wk": spec, "wv": spec, "wo": rev}

    def init_params(self, cfg, key):
        d = cfg.get("input_dim")
        return {n: fan_in_uniform(param_key(key, n), s, d) for n, s in self.param_shapes(cfg).items()}

    def param_init(self, cfg):
        return {n: uniform_spec(cfg.get("input_dim")) for n in self.param_shapes(cfg)}

    def own_flops(self, cfg, batch, seq_len):
        d = cfg.get("input_dim")
        rows = batch * seq_len
        return 8 * rows * d * d + 4 * rows * seq_len * d

    def remat_tags(self, cfg, batch, seq_len):
        d = cfg.get("input_dim")
        rows = batch * seq_len
        nbytes = rows * d * _dbytes(cfg)
        proj = 2 * rows * d * d
        return [RematTag("q_proj", nbytes, proj), RematTag("k_proj", nbytes, proj), RematTag("v_proj", nbytes, proj),
                RematTag("context", nbytes, 4 * rows * seq_len * d), RematTag("o_proj", nbytes, proj)]

    fuses_residual = True  # forward(x, residual=r) returns r + attn(x) from the wo GEMM epilogue

    def _project(self, module, x2, T, rope_ok: bool):
        """qkv = x2 @ (wq|wk|wv) (+ RoPE in the epilogue); returns (qkv, rope tables or None)."""
        cfg = module.config
        d, H = cfg.get("input_dim"), cfg.get("num_heads")
        hd = d // H
        kvd = hd * self.kv_heads(cfg)
        adt = act_dtype()
        wq, wk, wv = param("wq"), param("wk"), param("wv")
        wqkv = fused_columns(wq, wk, wv)
        pos = module.children["pos_emb"]
        # RoPE folded into the QKV GEMM epilogue (and its inverse into the attention
        # backward's dQ/dK stores) when the positional child is the stock RoPE kind
        rope = None
        if rope_ok and wqkv is not None and pos.kind == "RoPE" and option("fuse_rope", True):
            rope = rope_tables(T, hd, pos.config.get("base"), x2.device)
        if wqkv is not None:
            qkv = torch.empty((x2.shape[0], wqkv.shape[1]), device=x2.device, dtype=adt)
            if rope is not None:
                ops.gemm_rope(x2, wqkv, qkv, T, hd, d + kvd, rope[0], rope[1])
            else:
                ops.gemm(x2, wqkv, qkv)
        else:
            qkv = torch.empty((x2.shape[0], d + 2 * kvd), device=x2.device, dtype=adt)
            for w, c0, c1 in ((wq, 0, d), (wk, d, d + kvd), (wv, d + kvd, d + 2 * kvd)):
                ops.gemm(x2, w, qkv[:, c0:c1])
        return qkv, rope

    def forward(self, module, x, residual=None):
        """Remat tags (reference layers.py:318-329): q_proj/k_proj/v_proj = the fused qkv
        buffer, context = the attention output o (+ its log-sum-exp), o_proj = this block's
        output (not needed by the backward, so nothing is kept for it either way)."""
        cfg = module.config
        d, H = cfg.get("input_dim"), cfg.get("num_heads")
        KVH = self.kv_heads(cfg)
        B, T = _checked_3d(x, d, "Attention")
        hd = d // H
        kvd = hd * KVH
        adt = act_dtype()
        x2 = ops.cast(ops.rows2d(x), adt)
        qkv, rope = self._project(module, x2, T, True)
        q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
        if rope is None:
            invoke_child("pos_emb", q, k, T)
        scale = 1.0 / math.sqrt(hd)
        rec = is_recording()
        # bf16: o's rounding residual too, for the backward's delta (cb_attention_fwd o_lo)
        o, lse, *lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=rec)
        o_lo = lo[0] if lo else None
        out = torch.empty((o.shape[0], d), device=x.device, dtype=torch.float32)
        ops.gemm(o, param("wo"), out, residual=ops.rows2d(residual) if residual is not None else None)
        if rec:
            dq = remat_plan("q_proj", "k_proj", "v_proj")
            dc = remat_plan("context")
            if dq == RECOMPUTE and rope is None:
                dq = SAVE  # an unfused positional child would have to be re-run as well
            save(x2=x2, qkv=keep(qkv, dq), o=keep(o, dc), lse=keep(lse, dc), o_lo=keep(o_lo, dc), rope=rope,
                 geom=(B, T, H, KVH, hd, d, kvd))
        return out.view(B, T, d)

    def backward(self, module, dout):
        s = saved()
        B, T, H, KVH, hd, d, kvd = s["geom"]
        adt = act_dtype()
        qkv = restore(s["qkv"])
        if qkv is None:  # q/k/v projections rematerialised from the saved block input
            qkv, _ = self._project(module, s["x2"], T, True)
        q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
        o, lse, o_lo = restore(s["o"]), restore(s["lse"]), restore(s["o_lo"])
        if o is None:  # context rematerialised: the attention forward again
            o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, 1.0 / math.sqrt(hd), want_lo=True)
        g = ops.rows2d(ops.cast(dout, adt))
        do = _linear_bwd(o, param("wo"), g, param_grad("wo"), adt)
        dqkv = torch.empty_like(qkv)
        dq, dk, dv = dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:]
        if s["rope"] is not None:
            ops.attention_bwd_rope(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd,
                                   1.0 / math.sqrt(hd), s["rope"][0], s["rope"][1], o_lo=o_lo)
        else:
            ops.attention_bwd(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, 1.0 / math.sqrt(hd), o_lo=o_lo)
            backward_child("pos_emb", dq, dk)
        wq, wk, wv = param("wq"), param("wk"), param("wv")
        wqkv = fused_columns(wq, wk, wv)
        gq, gk, gv = param_grad("wq"), param_grad("wk"), param_grad("wv")
        gqkv = fused_columns(gq, gk, gv)
        x2 = s["x2"]
        if wqkv is not None and gqkv is not None:
            dx = _linear_bwd(x2, wqkv, dqkv, gqkv, torch.float32)
        else:
            dx = None
            for w, gw, dpart in ((wq, gq, dq), (wk, gk, dk), (wv, gv, dv)):
                ops.gemm(x2, dpart, gw, trans_a=True, accumulate=True)
                if dx is None:
                    dx = torch.empty((x2.shape[0], d), device=x2.device, dtype=torch.float32)
                    ops.gemm(dpart, w, dx, trans_b=True)
                else:
                    ops.gemm(dpart, w, dx, trans_b=True, accumulate=True)
        return dx.view(B, T, d)


class GroupedQueryAttentionBehavior(AttentionBehavior):
    """Attention with num_kv_heads <= num_heads key/value heads (new kind; the 70B layer).

    Not in the reference (it has only [d,d] K/V, reference layers.py:297-299); with
    num_kv_heads == num_heads it is exactly the reference's Attention.
    """

    def kv_heads(self, cfg) -> int:
        return cfg.get("num_kv_heads")

    def validate(self, cfg):
        h, kv = cfg.get("num_heads"), cfg.get("num_kv_heads")
        if kv < 1 or h % kv:
            raise ShapeError(f"num_heads {h} must be a multiple of num_kv_heads {kv}")

    def own_flops(self, cfg, batch, seq_len):
        d = cfg.get("input_dim")
        kvd = d // cfg.get("num_heads") * cfg.get("num_kv_heads")
        rows = batch * seq_len
        return 2 * rows * d * (2 * d + 2 * kvd) + 4 * rows * seq_len * d


# ------------------------------------------------------------------- FeedForward
class FeedForwardBehavior(Behavior):
    """w2(act(w1 x)) or w2(act0(w1 x) * act1(w1_gate x)) (reference layers.py:354-416)."""

    def validate(self, cfg):
        pair = activation_pair(cfg.get("activation"))
        for n in pair if pair else (cfg.get("activation"),):
            check_activation(n)

    def param_shapes(self, cfg):
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        shapes = {"w1": (d, h), "w2": (h, d)}
        if activation_pair(cfg.get("activation")):
            shapes["w1_gate"] = (d, h)
        return shapes

    def param_specs(self, cfg):
        spec = _pspec(cfg)
        specs = {"w1": spec, "w2": tuple(reversed(spec))}
        if activation_pair(cfg.get("activation")):
            specs["w1_gate"] = spec
        return specs

    def init_params(self, cfg, key):
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        out = {"w1": fan_in_uniform(param_key(key, "w1"), (d, h), d),
               "w2": fan_in_uniform(param_key(key, "w2"), (h, d), h)}
        if activation_pair(cfg.get("activation")):
            out["w1_gate"] = fan_in_uniform(param_key(key, "w1_gate"), (d, h), d)
        return out

    def param_init(self, cfg):
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        out = {"w1": uniform_spec(d), "w2": uniform_spec(h)}
        if activation_pair(cfg.get("activation")):
            out["w1_gate"] = uniform_spec(d)
        return out

    def own_flops(self, cfg, batch, seq_len):
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        rows = batch * seq_len
        br = 2 if activation_pair(cfg.get("activation")) else 1
        return br * 2 * rows * d * h + 2 * rows * h * d

    def remat_tags(self, cfg, batch, seq_len):
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        rows = batch * seq_len
        nb = _dbytes(cfg)
        br = 2 if activation_pair(cfg.get("activation")) else 1
        return [RematTag("hidden", br * rows * h * nb, br * 2 * rows * d * h),
                RematTag("output", rows * d * nb, 2 * rows * h * d)]

    fuses_residual = True

    def _up(self, module, x2):
        """pre = x2 @ (w1|w1_gate) and hidden = act(pre) (gated activation in the GEMM epilogue
        when the layout is fused)."""
        cfg = module.config
        h = cfg.get("hidden_dim")
        adt = act_dtype()
        pair = activation_pair(cfg.get("activation"))
        fused = None
        if pair:
            w1, wg = param("w1"), param("w1_gate")
            wcat = fused_columns(w1, wg)
            if wcat is not None and option("fuse_glu", True):
                fused = ops.gemm_gated_fwd(x2, wcat, pair[0], pair[1])
            if fused is not None:
                pre, hidden = fused
            elif wcat is not None:
                pre = _linear_fwd(x2, wcat, adt)
            else:
                pre = torch.empty((x2.shape[0], 2 * h), device=x2.device, dtype=adt)
                ops.gemm(x2, w1, pre[:, :h])
                ops.gemm(x2, wg, pre[:, h:])
            if fused is None:
                hidden = ops.act_fwd(pre[:, :h], pre[:, h:], pair[0], pair[1])
        else:
            pre = _linear_fwd(x2, param("w1"), adt)
            hidden = ops.act_fwd(pre, None, cfg.get("activation"))
        return pre, hidden

    def forward(self, module, x, residual=None):
        """Remat tags (reference layers.py:395-403): hidden = the up-projection (pre-activation
        and activation), output = this block's output (not needed by the backward).
        Recomputing "hidden" re-runs only the up-projection GEMM in the backward."""
        cfg = module.config
        if x.shape[-1] != cfg.get("input_dim"):
            raise ShapeError(f"FeedForward expects trailing dim {cfg.get('input_dim')}")
        lead = x.shape[:-1]
        x2 = ops.cast(ops.rows2d(x), act_dtype())
        pre, hidden = self._up(module, x2)
        out = torch.empty((x2.shape[0], cfg.get("input_dim")), device=x.device, dtype=torch.float32)
        ops.gemm(hidden, param("w2"), out, residual=ops.rows2d(residual) if residual is not None else None)
        if is_recording():
            dh = remat_plan("hidden")
            save(x2=x2, pre=keep(pre, dh), hidden=keep(hidden, dh))
        return out.view(*lead, cfg.get("input_dim"))

    def backward(self, module, dout):
        cfg = module.config
        s = saved()
        adt = act_dtype()
        h = cfg.get("hidden_dim")
        g = ops.rows2d(ops.cast(dout, adt))
        x2 = s["x2"]
        pre, hidden = restore(s["pre"]), restore(s["hidden"])
        if pre is None:  # "hidden" rematerialised: the up-projection again
            pre, hidden = self._up(module, x2)
        pair = activation_pair(cfg.get("activation"))
        dw2 = param_grad("w2")
        dpre = None
        if pair and option("fuse_glu", True):
            # dhidden = g @ w2^T formed and consumed by the gated-activation backward in one
            # GEMM epilogue (dhidden never reaches HBM)
            dpre = ops.gemm_gated_bwd(g, param("w2"), pre, pair[0], pair[1])
        if dpre is not None:
            if dw2 is not None:
                _wgrad(hidden, g, dw2)
        else:
            dhidden = _linear_bwd(hidden, param("w2"), g, dw2, adt)
            dpre = torch.empty_like(pre)
            if pair:
                ops.act_bwd(pre[:, :h], pre[:, h:], dhidden, dpre[:, :h], dpre[:, h:], pair[0], pair[1])
            else:
                ops.act_bwd(pre, None, dhidden, dpre, None, cfg.get("activation"))
        if pair:
            w1, wg = param("w1"), param("w1_gate")
            wcat = fused_columns(w1, wg)
            gcat = fused_columns(param_grad("w1"), param_grad("w1_gate"))
            if wcat is not None and gcat is not None:
                dx = _linear_bwd(x2, wcat, dpre, gcat, torch.float32)
            else:
                ops.gemm(x2, dpre[:, :h], param_grad("w1"), trans_a=True, accumulate=True)
                ops.gemm(x2, dpre[:, h:], param_grad("w1_gate"), trans_a=True, accumulate=True)
                dx = torch.empty((x2.shape[0], x2.shape[1]), device=x2.device, dtype=torch.float32)
                ops.gemm(dpre[:, :h], w1, dx, trans_b=True)
                ops.gemm(dpre[:, h:], wg, dx, trans_b=True, accumulate=True)
        else:
            dx = _linear_bwd(x2, param("w1"), dpre, param_grad("w1"), torch.float32)
        return dx.view(*dout.shape[:-1], x2.shape[1])


# ----------------------------------------------------------------------------- MoE
@dataclass(frozen=True)
class GateDecision:
    """Routing outcome (reference layers.py:422-429)."""

    indices: np.ndarray
    weights: np.ndarray
    dispatch_fractions: np.ndarray
    mean_probs: np.ndarray


def load_balance_loss(decision: GateDecision) -> float:
    e = decision.dispatch_fractions.shape[0]
    return float(e * np.sum(decision.dispatch_fractions * decision.mean_probs))


from .moe import MoEBehavior  # noqa: E402  (kernels + behavior live in moe.py)


# ------------------------------------------------------------- layer / stack / LM
class TransformerLayerBehavior(Behavior):
    """Pre-norm residual block: h = x + attn(norm(x)); out = h + ffn(norm(h)) (reference layers.py:539-551)."""

    def propagate(self, cfg):
        dim = cfg.get("input_dim")
        if isinstance(dim, int):
            for child in ("self_attention", "feed_forward", "self_attention_norm", "feed_forward_norm"):
                cfg = cfg.set(f"{child}.input_dim", dim)
        return cfg

    @staticmethod
    def _branch(module, name: str, normed, residual):
        """residual + child(normed); fused into the child's output GEMM when it supports it."""
        if getattr(module.children[name].behavior, "fuses_residual", False):
            return invoke_child(name, normed, residual=residual)
        return ops.add_(invoke_child(name, normed), residual)

    # Rematerialisation is per tag: the layer's remat_policy governs its subtree and each
    # child behavior keeps, offloads or recomputes its own tagged activations
    # (remat_decision; reference mesh.py:204-252, tags layers.py:318-329, 395-403, 501-511).

    def forward(self, module, x):
        h = self._branch(module, "self_attention", invoke_child("self_attention_norm", x), x)
        return self._branch(module, "feed_forward", invoke_child("feed_forward_norm", h), h)

    def backward(self, module, dout):
        dn2 = backward_child("feed_forward", dout)
        dh = backward_child("feed_forward_norm", dn2, dres=dout)
        dn1 = backward_child("self_attention", dh)
        return backward_child("self_attention_norm", dn1, dres=dh)


class TransformerStackBehavior(Behavior):
    """Sequential stack over the "layer" collection (reference layers.py:554-567)."""

    def propagate(self, cfg):
        dim = cfg.get("input_dim")
        if isinstance(dim, int):
            for i in range(len(cfg.get("layer"))):
                cfg = cfg.set(f"layer[{i}].input_dim", dim)
        return cfg

    def forward(self, module, x):
        for i in range(len(module.config.get("layer"))):
            x = invoke_child(f"layer[{i}]", x)
        return x

    def backward(self, module, dout):
        for i in reversed(range(len(module.config.get("layer")))):
            dout = backward_child(f"layer[{i}]", dout)
        return dout


class TiedLmHeadBehavior(Behavior):
    """logits = h @ table.T with the table read through shared state (reference layers.py:573-597)."""

    def own_flops(self, cfg, batch, seq_len):
        return 2 * batch * seq_len * cfg.get("dim") * cfg.get("vocab_size")

    def remat_tags(self, cfg, batch, seq_len):
        rows = batch * seq_len
        return [RematTag("logits", rows * cfg.get("vocab_size") * _dbytes(cfg), self.own_flops(cfg, batch, seq_len))]

    def _table(self, cfg):
        shared = get_shared_state(cfg.get("tied_to"))
        table = shared.get("weight") if isinstance(shared, dict) else shared
        if not isinstance(table, torch.Tensor) or table.dim() != 2 or table.shape[1] != cfg.get("dim"):
            raise BadPathError(f"tied_to path {cfg.get('tied_to')!r} does not hold an embedding table")
        return table

    def forward(self, module, h):
        cfg = module.config
        if h.shape[-1] != cfg.get("dim"):
            raise ShapeError(f"TiedLmHead expects trailing dim {cfg.get('dim')}")
        table = self._table(cfg)
        h2 = ops.cast(ops.rows2d(h), act_dtype())
        logits = torch.empty((h2.shape[0], table.shape[0]), device=h.device, dtype=torch.float32)
        ops.gemm(h2, table, logits, trans_b=True)
        save(h2=h2)
        return logits.view(*h.shape[:-1], table.shape[0])

    def backward(self, module, dlogits):
        cfg = module.config
        table = self._table(cfg)
        g = ops.rows2d(dlogits)
        shared = get_shared_grad(cfg.get("tied_to"))
        gtable = shared.get("weight") if isinstance(shared, dict) else shared
        ops.gemm(g, saved()["h2"], gtable, trans_a=True, accumulate=True)  # dE += dlogits^T h
        dh = torch.empty((g.shape[0], table.shape[1]), device=g.device, dtype=act_dtype())
        ops.gemm(g, table, dh)  # dh = dlogits @ E
        return dh.view(*dlogits.shape[:-1], table.shape[1])


class DecoderBehavior(Behavior):
    """Embedding -> stack -> final norm -> tied head (reference layers.py:600-620)."""

    def propagate(self, cfg):
        dim, vocab = cfg.get("dim"), cfg.get("vocab_size")
        if isinstance(dim, int):
            cfg = (cfg.set("emb.dim", dim).set("transformer.input_dim", dim).set("output_norm.input_dim", dim)
                   .set("lm_head.dim", dim))
        if isinstance(vocab, int):
            cfg = cfg.set("emb.num_embeddings", vocab).set("lm_head.vocab_size", vocab)
        return cfg

    def forward(self, module, ids):
        h = invoke_child("emb", ids)
        h = invoke_child("transformer", h)
        h = invoke_child("output_norm", h)
        return invoke_child("lm_head", h)

    def backward(self, module, dlogits):
        dh = backward_child("lm_head", dlogits)
        dh = backward_child("output_norm", dh)
        dh = backward_child("transformer", dh)
        backward_child("emb", dh)
        return None


class CausalLMBehavior(Behavior):
    """Model wrapper so trainer paths start at "model" (reference layers.py:623-635)."""

    def propagate(self, cfg):
        dim, vocab = cfg.get("dim"), cfg.get("vocab_size")
        if isinstance(dim, int):
            cfg = cfg.set("decoder.dim", dim)
        if isinstance(vocab, int):
            cfg = cfg.set("decoder.vocab_size", vocab)
        return cfg

    def forward(self, module, ids):
        return invoke_child("decoder", ids)

    def backward(self, module, dlogits):
        return backward_child("decoder", dlogits)


class TrainerBehavior(Behavior):
    """Root: next-token cross-entropy over B*(T-1) positions (reference layers.py:638-651).

    Forward-only invocations return the loss as a Python float (the reference's return
    type, one device sync); recorded (training) invocations keep it on the device and
    compute d(loss)/d(logits) in the same kernel pass as the loss.
    """

    def forward(self, module, batch):
        tokens = batch["tokens"]
        if not isinstance(tokens, torch.Tensor) or tokens.dim() != 2 or tokens.shape[1] < 2:
            raise ShapeError("trainer expects integer tokens of shape [batch, seq>=2]")
        B, T = tokens.shape
        logits = invoke_child("model", tokens)
        l2 = logits.view(B * T, logits.shape[-1])
        if is_recording():
            dl = torch.empty(l2.shape, device=l2.device, dtype=act_dtype())
            loss = ops.xent(l2, tokens, dl, 1.0 / (B * (T - 1)))
            save(dlogits=dl, shape=logits.shape)
            add_summary("loss", loss)
            return loss
        loss = ops.xent(l2, tokens, None, 1.0)
        value = float(loss.item())
        add_summary("loss", value)
        return value

    def backward(self, module, seed=1.0):
        s = saved()
        dl = s["dlogits"]
        if seed != 1.0:
            ops.copy2d(dl, dl, alpha=float(seed))
        backward_child("model", dl.view(*s["shape"]))
        return None


@dataclass(frozen=True)
class OptimizerSpec:
    """Product of the adamw external factory (reference layers.py:657-663)."""

    lr: float
    beta1: float
    beta2: float


_UNSHARDED_2D = (None, None)


def _register_all() -> None:
    register_spec_function("scaled_hidden_dim", scaled_hidden_dim)
    F = FieldSpec
    K = ValueKind
    register_component(ComponentSchema("Linear", {
        "input_dim": F(K.INT), "output_dim": F(K.INT), "bias": F(K.BOOL, True),
        "param_partition_spec": F(K.SEQ, _UNSHARDED_2D), "dtype": F(K.TEXT, "f32")}))
    register_behavior("Linear", LinearBehavior())
    register_component(ComponentSchema("RMSNorm", {"input_dim": F(K.INT), "eps": F(K.FLOAT, 1e-6)}))
    register_behavior("RMSNorm", RMSNormBehavior())
    register_component(ComponentSchema("Embedding", {
        "num_embeddings": F(K.INT), "dim": F(K.INT), "param_partition_spec": F(K.SEQ, _UNSHARDED_2D),
        "dtype": F(K.TEXT, "f32")}))
    register_behavior("Embedding", EmbeddingBehavior())
    register_component(ComponentSchema("NoPos", {"dim": F(K.INT)}))
    register_behavior("NoPos", NoPosBehavior())
    register_component(ComponentSchema("RoPE", {"dim": F(K.INT), "base": F(K.FLOAT, 10000.0)}))
    register_behavior("RoPE", RoPEBehavior())
    register_component(ComponentSchema("Attention", {
        "input_dim": F(K.INT), "num_heads": F(K.INT, 2), "pos_emb": F(K.CONFIG, "NoPos"),
        "param_partition_spec": F(K.SEQ, _UNSHARDED_2D), "dtype": F(K.TEXT, "f32")}))
    register_behavior("Attention", AttentionBehavior())
    register_component(ComponentSchema("GroupedQueryAttention", {
        "input_dim": F(K.INT), "num_heads": F(K.INT, 2), "num_kv_heads": F(K.INT, 1), "pos_emb": F(K.CONFIG, "NoPos"),
        "param_partition_spec": F(K.SEQ, _UNSHARDED_2D), "dtype": F(K.TEXT, "f32")}))
    register_behavior("GroupedQueryAttention", GroupedQueryAttentionBehavior())
    register_component(ComponentSchema("FeedForward", {
        "input_dim": F(K.INT), "hidden_dim": F(K.INT, FunctionSpec("scaled_hidden_dim", scale=4.0)),
        "activation": F(K.ANY, "relu"), "param_partition_spec": F(K.SEQ, _UNSHARDED_2D),
        "dtype": F(K.TEXT, "f32")}))
    register_behavior("FeedForward", FeedForwardBehavior())
    register_component(ComponentSchema("MoE", {
        "input_dim": F(K.INT), "hidden_dim": F(K.INT, FunctionSpec("scaled_hidden_dim", scale=4.0)),
        "num_experts": F(K.INT, 8), "top_k": F(K.INT, 2), "activation": F(K.ANY, "relu"),
        "param_partition_spec": F(K.SEQ, _UNSHARDED_2D), "dtype": F(K.TEXT, "f32")}))
    register_behavior("MoE", MoEBehavior())
    register_component(ComponentSchema("TransformerLayer", {
        "input_dim": F(K.INT), "self_attention": F(K.CONFIG, "Attention"),
        "feed_forward": F(K.CONFIG, "FeedForward"), "self_attention_norm": F(K.CONFIG, "RMSNorm"),
        "feed_forward_norm": F(K.CONFIG, "RMSNorm"), "remat_policy": F(K.MAP, {})}))
    register_behavior("TransformerLayer", TransformerLayerBehavior())
    register_component(ComponentSchema("TransformerStack", {"input_dim": F(K.INT), "layer": F(K.CONFIG_LIST, ())}))
    register_behavior("TransformerStack", TransformerStackBehavior())
    register_component(ComponentSchema("TiedLmHead", {
        "dim": F(K.INT), "vocab_size": F(K.INT), "tied_to": F(K.TEXT, "model.decoder.emb"),
        "dtype": F(K.TEXT, "f32")}))
    register_behavior("TiedLmHead", TiedLmHeadBehavior())
    register_component(ComponentSchema("Decoder", {
        "dim": F(K.INT), "vocab_size": F(K.INT), "emb": F(K.CONFIG, "Embedding"),
        "transformer": F(K.CONFIG, "TransformerStack"), "output_norm": F(K.CONFIG, "RMSNorm"),
        "lm_head": F(K.CONFIG, "TiedLmHead")}))
    register_behavior("Decoder", DecoderBehavior())
    register_component(ComponentSchema("CausalLM", {
        "dim": F(K.INT), "vocab_size": F(K.INT), "decoder": F(K.CONFIG, "Decoder")}))
    register_behavior("CausalLM", CausalLMBehavior())
    register_factory("adamw", {"lr": F(K.FLOAT), "beta1": F(K.FLOAT, 0.9), "beta2": F(K.FLOAT, 0.999)},
                     lambda lr, beta1, beta2: OptimizerSpec(lr, beta1, beta2))
    register_component(ComponentSchema("Trainer", {
        "model": F(K.CONFIG, "CausalLM"), "learner": F(K.CONFIG, "fn:adamw"), "batch_size": F(K.INT, 4),
        "seq_len": F(K.INT, 8), "mesh_axis_names": F(K.SEQ, ("data",)), "mesh_shape": F(K.SEQ, (-1,)),
        "mesh_rules": F(K.SEQ, ()), "optimizer_state_multiplier": F(K.INT, 2),
        "offload_optimizer_state": F(K.BOOL, False), "dtype_params": F(K.MAP, {})}))
    register_behavior("Trainer", TrainerBehavior())


_register_all()
