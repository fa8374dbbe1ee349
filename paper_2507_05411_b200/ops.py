"""Thin tensor-level wrappers over the C ABI (device pointers + stream from torch).

PyTorch is used only for device memory and streams: every arithmetic operation below
is one call into ``libcomposer_b200.so``.  Shapes/dtypes are checked here, before the
launch, and raise the reference's error classes.  All functions run on the current
torch stream.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ShapeError, TypeMismatchError

_DT = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16}
ACT_IDS = {"linear": 0, "relu": 1, "silu": 2, "sigmoid": 3, "tanh": 4}


def dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeMismatchError(f"unsupported tensor dtype {t.dtype}") from None


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def ld(t: torch.Tensor, what: str = "tensor") -> int:
    """Row stride of a 2-D row-major view (stride(1) == 1)."""
    if t.dim() != 2 or (t.stride(1) != 1 and t.shape[1] > 1):
        raise ShapeError(f"{what} must be a 2-D row-major view")
    return t.stride(0)


def rows2d(t: torch.Tensor) -> torch.Tensor:
    """[..., d] -> [rows, d] view (no copy; raises if not viewable)."""
    return t.reshape(-1, t.shape[-1]) if t.dim() != 2 else t


# ----------------------------------------------------------------- launch profiler
class KernelProfiler:
    """Tallies the algorithmic FLOPs of selected launches (bench.py).

    Records are (kind, algorithmic_flops, start_event, end_event); with ``events=False``
    (bench.py's default: kernel durations come from CUPTI kernel activity instead, which
    sees every stream) the events are None and only launches/FLOPs are counted.
    """

    def __init__(self, events: bool = True):
        self.events = events
        self.records: list = []

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for kind, flops, s, e in self.records:
            d = out.setdefault(kind, {"launches": 0, "flops": 0, "ms": 0.0})
            d["launches"] += 1
            d["flops"] += flops
            if s is not None:
                d["ms"] += s.elapsed_time(e)
        return out


_PROFILER: KernelProfiler | None = None


def set_profiler(p: KernelProfiler | None) -> None:
    global _PROFILER
    _PROFILER = p


def _profiled(kind: str, flops: int, fn, *args):
    if _PROFILER is None:
        return fn(*args)
    if not _PROFILER.events:
        _PROFILER.records.append((kind, flops, None, None))
        return fn(*args)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = fn(*args)
    e.record()
    _PROFILER.records.append((kind, flops, s, e))
    return out


# ----------------------------------------------------------------------------- GEMM
def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, trans_a: bool = False, trans_b: bool = False,
         alpha: float = 1.0, accumulate: bool = False, residual: torch.Tensor | None = None) -> torch.Tensor:
    """out = alpha * op(a) @ op(b) (+ out) (+ residual); op(x) = x.T when trans_x."""
    M = a.shape[1] if trans_a else a.shape[0]
    K = a.shape[0] if trans_a else a.shape[1]
    Kb = b.shape[1] if trans_b else b.shape[0]
    N = b.shape[0] if trans_b else b.shape[1]
    if K != Kb:
        raise ShapeError(f"gemm: inner dims differ ({K} vs {Kb})")
    if tuple(out.shape) != (M, N):
        raise ShapeError(f"gemm: out shape {tuple(out.shape)} != {(M, N)}")
    if a.dtype != b.dtype:
        raise TypeMismatchError("gemm: operand dtypes differ")
    ldr = 0
    if residual is not None:
        if tuple(residual.shape) != (M, N):
            raise ShapeError("gemm: residual shape mismatch")
        ldr = ld(residual, "residual")
    if _f32_on_tc(a, b, out, M, N, K):
        return _gemm_bf16x6(a, b, out, trans_a, trans_b, alpha, accumulate, residual)
    kind = "gemm_bf16" if a.dtype == torch.bfloat16 else "gemm_f32"
    wgrad = accumulate and residual is None and out.dtype == torch.float32  # a weight-gradient-style GEMM
    ow = _OVERWRITE
    if ow is not None and wgrad and ow.lo <= out.data_ptr() < ow.hi:
        # the whole gradient of these elements: written, not added to a cleared buffer
        accumulate = False
        ow.covered += M * N
    fu = _FUSED_UPDATE
    if fu is not None and wgrad and fu.lo <= out.data_ptr() < fu.hi:
        # the whole gradient of these elements: the bucket's AdamW runs in this GEMM's epilogue
        off = (out.data_ptr() - fu.lo) // 4
        last = off + (M - 1) * ld(out, "out") + N
        if last > fu.numel:
            raise ShapeError("gemm: fused-update output leaves its bucket")
        fu.covered += M * N
        _profiled(kind, 2 * M * N * K, _lib.call, "cb_gemm_adamw", M, N, K, dt(a), a.data_ptr(), ld(a, "A"),
                  int(trans_a), b.data_ptr(), ld(b, "B"), int(trans_b), out.data_ptr(), ld(out, "out"), float(alpha),
                  fu.master + 4 * off, fu.m + 4 * off, fu.v + 4 * off, (fu.bf + 2 * off) if fu.bf else None,
                  fu.lr, fu.beta1, fu.beta2, fu.eps, fu.wd, fu.step, stream_ptr())
        return out
    _profiled(kind, 2 * M * N * K, _lib.call, "cb_gemm", M, N, K, dt(a), a.data_ptr(), ld(a, "A"), int(trans_a),
              b.data_ptr(), ld(b, "B"), int(trans_b), out.data_ptr(), ld(out, "out"), dt(out), _ptr(residual), ldr,
              dt(residual) if residual is not None else 0, float(alpha), int(accumulate), stream_ptr())
    return out


class FusedUpdate:
    """A bucket whose AdamW runs in its weight-gradient GEMMs' epilogues (cb_gemm_adamw): any
    accumulating f32 GEMM into [lo, hi) — the bucket's gradient buffer — becomes the update of
    those elements of master / m / v / bf16 copy (same flat layout).  `covered` counts the
    elements updated, which the engine checks against the bucket's parameter count."""

    def __init__(self, grad, master, m, v, bf, lr, beta1, beta2, eps, wd, step):
        self.lo, self.numel = grad.data_ptr(), grad.numel()
        self.hi = self.lo + 4 * self.numel
        self.master, self.m, self.v = master.data_ptr(), m.data_ptr(), v.data_ptr()
        self.bf = bf.data_ptr() if bf is not None else 0
        self.lr, self.beta1, self.beta2, self.eps, self.wd = (float(x) for x in (lr, beta1, beta2, eps, wd))
        self.step = int(step)
        self.covered = 0


_FUSED_UPDATE: FusedUpdate | None = None


class Overwrite:
    """A layer's gradient buffer [lo, hi) whose every element gets exactly one weight-gradient
    GEMM per step: an accumulating GEMM into it writes instead (the same values as adding to a
    cleared buffer, up to the sign of zero), so the buffer is never cleared.  `covered` counts
    the elements written, which the engine checks against the bucket's parameter count."""

    def __init__(self, grad):
        self.lo = grad.data_ptr()
        self.hi = self.lo + 4 * grad.numel()
        self.covered = 0


_OVERWRITE: Overwrite | None = None


def set_overwrite(ow: Overwrite | None) -> None:
    global _OVERWRITE
    _OVERWRITE = ow


def set_fused_update(fu: FusedUpdate | None) -> None:
    global _FUSED_UPDATE
    _FUSED_UPDATE = fu


# f32 parity mode on the tensor cores: an f32 GEMM large enough for the tcgen05 engine runs as
# six bf16 products of the operands' three-term bf16 splits (cb_split_bf16x3), accumulated in
# the f32 output by the same CTA-pair / 1-CTA kernels and epilogues the bf16 step uses — the
# "BF16x6" FP32 emulation, ~fp32-accurate (the dropped terms are O(2^-24); each pass's f32
# result is added in the epilogue).  Opt-in (CB_F32_TC=1, or ops.set_f32_tc(True)): the SIMT
# engine is a little more accurate on ill-conditioned shapes (the sigmoid-FFN stack: 8e-6 vs
# 1.3e-5 on one gradient), so the parity mode defaults to it and the tests run both.
_F32_TC = __import__("os").environ.get("CB_F32_TC", "0") == "1"


def set_f32_tc(enable: bool) -> None:
    global _F32_TC
    _F32_TC = bool(enable)
_F32_TC_MIN_WORK = 1 << 22  # the tcgen05 dispatch threshold of cb_gemm (gemm_impl)
# products x_i * y_j of the splits, smallest first so the f32 accumulation adds small to small
_BF16X6_TERMS = ((2, 0), (0, 2), (1, 1), (1, 0), (0, 1), (0, 0))


def _f32_on_tc(a, b, out, M, N, K) -> bool:
    return (_F32_TC and a.dtype == torch.float32 and b.dtype == torch.float32 and out.dtype == torch.float32
            and M * N * K >= _F32_TC_MIN_WORK and _GEMM_PATH == 0)


def _split3(x: torch.Tensor):
    x2 = rows2d(x)
    parts = [torch.empty(x2.shape, device=x.device, dtype=torch.bfloat16) for _ in range(3)]
    _lib.call("cb_split_bf16x3", x2.shape[0], x2.shape[1], x2.data_ptr(), ld(x2), parts[0].data_ptr(),
              parts[1].data_ptr(), parts[2].data_ptr(), stream_ptr())
    return parts


# K per pass: the tensor core's f32 accumulation inside one GEMM loses ~2^-24 per K=16 step
# (measured: ~1e-5 relative at K = 4096, ~1e-6 at 256), so K is cut into 128-long chunks whose results are
# added in the epilogue's round-to-nearest f32 adds
_BF16X6_KCHUNK = 128


def _gemm_bf16x6(a, b, out, trans_a, trans_b, alpha, accumulate, residual):
    sa, sb = _split3(a), _split3(b)
    K = a.shape[0] if trans_a else a.shape[1]
    n = 0
    for k0 in range(0, K, _BF16X6_KCHUNK):
        k1 = min(K, k0 + _BF16X6_KCHUNK)
        for i, j in _BF16X6_TERMS:
            ai = sa[i][k0:k1] if trans_a else sa[i][:, k0:k1]
            bj = sb[j][:, k0:k1] if trans_b else sb[j][k0:k1]
            gemm(ai, bj, out, trans_a=trans_a, trans_b=trans_b, alpha=alpha,
                 accumulate=accumulate if n == 0 else True, residual=residual if n == 0 else None)
            n += 1
    return out


def gemm_rope(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, seq_len: int, head_dim: int, rope_cols: int,
              cos_t: torch.Tensor, sin_t: torch.Tensor) -> torch.Tensor:
    """out = a @ b with RoPE applied to out[:, :rope_cols] (fused into the tcgen05 epilogue)."""
    M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K or tuple(out.shape) != (M, N):
        raise ShapeError("gemm_rope: shape mismatch")
    if _f32_on_tc(a, b, out, M, N, K):  # six accumulated products, then the rotation
        _gemm_bf16x6(a, b, out, False, False, 1.0, False, None)
        rope_(out[:, :rope_cols], seq_len, rope_cols // head_dim, head_dim, cos_t, sin_t)
        return out
    _profiled("gemm_bf16" if a.dtype == torch.bfloat16 else "gemm_f32", 2 * M * N * K, _lib.call, "cb_gemm_rope",
              M, N, K, dt(a), a.data_ptr(), ld(a, "A"), 0, b.data_ptr(), ld(b, "B"), 0, out.data_ptr(),
              ld(out, "out"), dt(out), int(seq_len), int(head_dim), int(rope_cols), cos_t.data_ptr(),
              sin_t.data_ptr(), stream_ptr())
    return out


def gemm_gated_fwd(x2: torch.Tensor, wcat: torch.Tensor, act0: str, act1: str, pre=None, hidden=None):
    """pre = x2 @ wcat and hidden = act0(pre[:, :H]) * act1(pre[:, H:]) from one CTA-pair GEMM
    (activation in the epilogue), into `pre` / `hidden` when given.  Returns (pre, hidden),
    or None when the fused form does not apply (the caller then runs gemm + act_fwd)."""
    M, K = x2.shape
    if x2.dtype != torch.bfloat16 or wcat.dtype != torch.bfloat16 or wcat.shape[0] != K or wcat.shape[1] % 2:
        return None
    H = wcat.shape[1] // 2
    if pre is None:
        pre = torch.empty((M, 2 * H), device=x2.device, dtype=torch.bfloat16)
    if hidden is None:
        hidden = torch.empty((M, H), device=x2.device, dtype=torch.bfloat16)
    if tuple(pre.shape) != (M, 2 * H) or tuple(hidden.shape) != (M, H):
        raise ShapeError("gemm_gated_fwd: output shape mismatch")
    ok = _profiled("gemm_bf16", 2 * M * 2 * H * K, _lib.try_call, "cb_gemm_gated_fwd", M, H, K, x2.data_ptr(),
                   ld(x2, "A"), 0, wcat.data_ptr(), ld(wcat, "B"), 0, pre.data_ptr(), ld(pre), hidden.data_ptr(),
                   ld(hidden), ACT_IDS[act0], ACT_IDS[act1], stream_ptr())
    return (pre, hidden) if ok else None


def gemm_gated_bwd(dy: torch.Tensor, w2: torch.Tensor, pre: torch.Tensor, act0: str, act1: str, dpre=None):
    """dpre = d/d(pre) of act0(a) * act1(g) given d(out) = dy and out = hidden @ w2, with
    dhidden = dy @ w2^T formed and consumed inside one CTA-pair GEMM (into `dpre` when
    given).  None when the fused form does not apply."""
    M, K = dy.shape
    H = w2.shape[0]
    if dy.dtype != torch.bfloat16 or w2.dtype != torch.bfloat16 or w2.shape[1] != K or pre.shape != (M, 2 * H):
        return None
    if dpre is None:
        dpre = torch.empty_like(pre)
    ok = _profiled("gemm_bf16", 2 * M * H * K, _lib.try_call, "cb_gemm_gated_bwd", M, H, K, dy.data_ptr(),
                   ld(dy, "A"), 0, w2.data_ptr(), ld(w2, "B"), 1, pre.data_ptr(), ld(pre), dpre.data_ptr(),
                   ld(dpre), ACT_IDS[act0], ACT_IDS[act1], stream_ptr())
    return dpre if ok else None


_GEMM_WS: dict = {}


# --------------------------------------------------------------------- grouped GEMMs
def gemm_grouped_rows(a: torch.Tensor, b_stacked: torch.Tensor, out: torch.Tensor, grp_off: torch.Tensor,
                      groups: int, trans_b: bool = False, accumulate: bool = False, alpha: float = 1.0,
                      rows: int = 0):
    """out[rows of g] = a[rows of g] @ op(B_g) for all groups in one launch (cb_gemm_grouped
    mode 1); B_g = block g of b_stacked ([G*K, N], or [G*N, K] read transposed).  rows: the
    real (unpadded) row count, for the algorithmic FLOP tally only."""
    M, K = a.shape
    N = b_stacked.shape[0] // groups if trans_b else b_stacked.shape[1]
    if tuple(out.shape) != (M, N):
        raise ShapeError(f"gemm_grouped: out shape {tuple(out.shape)} != {(M, N)}")
    _profiled("gemm_bf16", 2 * rows * N * K, _lib.call, "cb_gemm_grouped", 1, groups, grp_off.data_ptr(), M, N, K, a.data_ptr(),
              ld(a, "A"), 0, b_stacked.data_ptr(), ld(b_stacked, "B"), int(trans_b), out.data_ptr(), ld(out, "D"),
              dt(out), float(alpha), int(accumulate), stream_ptr())
    return out


def gemm_grouped_k(a: torch.Tensor, b: torch.Tensor, out_stacked: torch.Tensor, grp_off: torch.Tensor, groups: int,
                   accumulate: bool = True, rows: int = 0):
    """out_g (+)= a[rows of g]^T @ b[rows of g] for all groups in one launch (cb_gemm_grouped
    mode 2, the experts' weight gradients); out_g = rows [g*M, (g+1)*M) of out_stacked."""
    Kcap, M = a.shape
    N = b.shape[1]
    if tuple(out_stacked.shape) != (groups * M, N):
        raise ShapeError("gemm_grouped_k: out must be [groups * M, N]")
    _profiled("gemm_bf16", 2 * rows * M * N, _lib.call, "cb_gemm_grouped", 2, groups, grp_off.data_ptr(), M, N, Kcap, a.data_ptr(),
              ld(a, "A"), 1, b.data_ptr(), ld(b, "B"), 0, out_stacked.data_ptr(), ld(out_stacked, "D"),
              dt(out_stacked), 1.0, int(accumulate), stream_ptr())
    return out_stacked


def gemm_gated_fwd_grouped(x: torch.Tensor, wcat_stacked: torch.Tensor, grp_off: torch.Tensor, groups: int,
                           act0: str, act1: str, pre: torch.Tensor, hidden: torch.Tensor, rows: int = 0):
    M, K = x.shape
    H = wcat_stacked.shape[1] // 2
    _profiled("gemm_bf16", 2 * rows * 2 * H * K, _lib.call, "cb_gemm_gated_fwd_grouped", groups, grp_off.data_ptr(), M, H, K,
              x.data_ptr(), ld(x, "A"), wcat_stacked.data_ptr(), ld(wcat_stacked, "B"), pre.data_ptr(), ld(pre),
              hidden.data_ptr(), ld(hidden), ACT_IDS[act0], ACT_IDS[act1], stream_ptr())
    return pre, hidden


def gemm_gated_bwd_grouped(dy: torch.Tensor, w2_stacked: torch.Tensor, grp_off: torch.Tensor, groups: int,
                           pre: torch.Tensor, act0: str, act1: str, dpre: torch.Tensor, rows: int = 0):
    M, K = dy.shape
    H = w2_stacked.shape[0] // groups
    _profiled("gemm_bf16", 2 * rows * H * K, _lib.call, "cb_gemm_gated_bwd_grouped", groups, grp_off.data_ptr(), M, H, K,
              dy.data_ptr(), ld(dy, "A"), w2_stacked.data_ptr(), ld(w2_stacked, "B"), pre.data_ptr(), ld(pre),
              dpre.data_ptr(), ld(dpre), ACT_IDS[act0], ACT_IDS[act1], stream_ptr())
    return dpre


def ensure_gemm_workspace(device, nbytes: int = 256 << 20) -> None:
    """Registers a split-K workspace for the tcgen05 GEMM on this device (PyTorch-owned)."""
    key = str(device)
    if key in _GEMM_WS and _GEMM_WS[key].numel() * 4 >= nbytes:
        return
    buf = torch.empty(nbytes // 4, device=device, dtype=torch.float32)
    _GEMM_WS[key] = buf
    _lib.call("cb_gemm_set_workspace", buf.data_ptr(), buf.numel() * 4)


_GEMM_PATH = 0


def set_gemm_path(path: int) -> None:
    """0: automatic, 1: SIMT engine only (f32 GEMMs then stay f32 SIMT), 2: tcgen05 only."""
    global _GEMM_PATH
    _lib.call("cb_gemm_set_path", int(path))
    _GEMM_PATH = int(path)


_ATTN_PATH = 0


def set_attention_path(path: int) -> None:
    """0: automatic (tcgen05 kernels, head_dim < 128 zero-padded to them), 1: SIMT engine."""
    global _ATTN_PATH
    _lib.call("cb_attention_set_path", int(path))
    _ATTN_PATH = int(path)


# -------------------------------------------------------------------------- RMSNorm
def rmsnorm_fwd(x: torch.Tensor, scale: torch.Tensor, eps: float, out_dtype: torch.dtype):
    x2 = rows2d(x)
    rows, dim = x2.shape
    y = torch.empty((rows, dim), device=x.device, dtype=out_dtype)
    rstd = torch.empty((rows,), device=x.device, dtype=torch.float32)
    _lib.call("cb_rmsnorm_fwd", rows, dim, x2.data_ptr(), ld(x2), dt(x2), scale.data_ptr(), float(eps), y.data_ptr(),
              ld(y), dt(y), rstd.data_ptr(), stream_ptr())
    return y.view(*x.shape[:-1], dim), rstd


def rmsnorm_bwd(x, scale, rstd, dy, dres=None, dscale=None, want_bf16=False):
    """Returns dx (f32), or (dx, dx_bf16) when want_bf16 (the bf16 copy written in the same pass)."""
    x2, g2 = rows2d(x), rows2d(dy)
    rows, dim = x2.shape
    dx = torch.empty((rows, dim), device=x.device, dtype=torch.float32)
    dxb = torch.empty((rows, dim), device=x.device, dtype=torch.bfloat16) if want_bf16 else None
    ws = None
    if dscale is not None:
        nbytes = ctypes.c_int64(0)
        _lib.call("cb_rmsnorm_bwd_workspace", rows, dim, ctypes.byref(nbytes))
        ws = torch.empty((max(1, nbytes.value // 4),), device=x.device, dtype=torch.float32)
    r2 = rows2d(dres) if dres is not None else None
    _lib.call("cb_rmsnorm_bwd", rows, dim, x2.data_ptr(), ld(x2), dt(x2), scale.data_ptr(), rstd.data_ptr(),
              g2.data_ptr(), ld(g2), dt(g2), _ptr(r2), ld(r2) if r2 is not None else 0, dx.data_ptr(), ld(dx),
              _ptr(dxb), ld(dxb) if dxb is not None else 0, _ptr(dscale), _ptr(ws), stream_ptr())
    dx = dx.view(*x.shape[:-1], dim)
    if want_bf16:
        return dx, dxb.view(*x.shape[:-1], dim)
    return dx


# ------------------------------------------------------------------------ embedding
def embedding_fwd(ids: torch.Tensor, table: torch.Tensor, out_dtype: torch.dtype):
    flat = ids.reshape(-1)
    n = flat.numel()
    dim = table.shape[1]
    out = torch.empty((n, dim), device=table.device, dtype=out_dtype)
    _lib.call("cb_embedding_fwd", n, dim, flat.data_ptr(), table.data_ptr(), ld(table), dt(table), out.data_ptr(),
              ld(out), dt(out), stream_ptr())
    return out.view(*ids.shape, dim)


def sort_ids(ids: torch.Tensor, vocab: int):
    flat = ids.reshape(-1)
    n = flat.numel()
    offsets = torch.empty((vocab + 1,), device=ids.device, dtype=torch.int32)
    cursor = torch.empty((int(_lib.load().cb_sort_ids_scratch(n, vocab)),), device=ids.device, dtype=torch.int32)
    perm = torch.empty((max(n, 1),), device=ids.device, dtype=torch.int32)
    _lib.call("cb_sort_ids", n, vocab, flat.data_ptr(), offsets.data_ptr(), cursor.data_ptr(), perm.data_ptr(),
              stream_ptr())
    return offsets, perm


def embedding_bwd(offsets, perm, dout: torch.Tensor, dtable: torch.Tensor):
    g2 = rows2d(dout)
    vocab, dim = dtable.shape
    _lib.call("cb_embedding_bwd", vocab, dim, offsets.data_ptr(), perm.data_ptr(), g2.data_ptr(), ld(g2), dt(g2),
              dtable.data_ptr(), ld(dtable), stream_ptr())


# ----------------------------------------------------------------------------- RoPE
def rope_(x2d: torch.Tensor, seq_len: int, heads: int, head_dim: int, cos_t, sin_t, inverse: bool = False):
    rows = x2d.shape[0]
    _lib.call("cb_rope", rows, seq_len, heads, head_dim, x2d.data_ptr(), ld(x2d), dt(x2d), cos_t.data_ptr(),
              sin_t.data_ptr(), int(inverse), stream_ptr())


# ---------------------------------------------------------------------- activations
def act_fwd(a: torch.Tensor, g: torch.Tensor | None, act0: str, act1: str = "linear", out=None):
    rows, cols = a.shape
    if out is None:
        out = torch.empty((rows, cols), device=a.device, dtype=a.dtype)
    _lib.call("cb_act_fwd", rows, cols, ACT_IDS[act0], ACT_IDS[act1], a.data_ptr(), ld(a), _ptr(g),
              ld(g) if g is not None else 0, out.data_ptr(), ld(out), dt(a), stream_ptr())
    return out


def act_bwd(a, g, dout, da, dg, act0: str, act1: str = "linear"):
    rows, cols = a.shape
    _lib.call("cb_act_bwd", rows, cols, ACT_IDS[act0], ACT_IDS[act1], a.data_ptr(), ld(a), _ptr(g),
              ld(g) if g is not None else 0, dout.data_ptr(), ld(dout), da.data_ptr(), ld(da), _ptr(dg),
              ld(dg) if dg is not None else 0, dt(a), stream_ptr())


def sum_parts(parts: list, out: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
    """out = scale * sum(parts) in list order (f32, deterministic; cb_sum_parts)."""
    import ctypes

    for t in parts:
        if t.dtype != torch.float32 or out.dtype != torch.float32 or t.numel() != out.numel():
            raise ShapeError("sum_parts: f32 parts of out's size expected")
    ptrs = (ctypes.c_void_p * len(parts))(*[t.data_ptr() for t in parts])
    _lib.call("cb_sum_parts", len(parts), out.numel(), ctypes.addressof(ptrs), out.data_ptr(), float(scale),
              stream_ptr())
    return out


def copy2d(src: torch.Tensor, dst: torch.Tensor, alpha: float = 1.0, accumulate: bool = False):
    s2, d2 = rows2d(src), rows2d(dst)
    if s2.shape != d2.shape:
        raise ShapeError("copy2d: shape mismatch")
    _lib.call("cb_copy2d", s2.shape[0], s2.shape[1], s2.data_ptr(), ld(s2), dt(s2), d2.data_ptr(), ld(d2), dt(d2),
              float(alpha), int(accumulate), stream_ptr())
    return dst


def cast(src: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    """dtype copy of `src`; reuses a copy a producing kernel already attached as `_bf16`."""
    if src.dtype == dtype:
        return src
    cached = getattr(src, "_bf16", None)
    if dtype == torch.bfloat16 and cached is not None:
        return cached.reshape(src.shape)
    out = torch.empty(src.shape, device=src.device, dtype=dtype)
    return copy2d(src, out)


def add_(dst: torch.Tensor, src: torch.Tensor, alpha: float = 1.0):
    return copy2d(src, dst, alpha=alpha, accumulate=True)


def zero_(t: torch.Tensor):
    if not t.is_contiguous():
        raise ShapeError("zero_: tensor must be contiguous")
    _lib.call("cb_memset_zero", t.data_ptr(), t.numel() * t.element_size(), stream_ptr())
    return t


# ------------------------------------------------------------------------ attention
# head dims the tcgen05 kernels (head_dim 128) serve through zero padding: every head's hd
# columns are copied into a 128-column slot whose other columns are zero — S = Q K^T and the
# softmax are unchanged (the scale is passed explicitly), O / dQ / dK / dV come back in the
# first hd columns; half the MMA work is wasted, against a SIMT fallback
_PAD_HD = (16, 32, 64)
_TC_HD = 128
_pad_heads_enabled = True


def _pad_ok(q: torch.Tensor, hd: int) -> bool:
    return q.dtype == torch.bfloat16 and hd in _PAD_HD and _pad_heads_enabled and _ATTN_PATH == 0


def _pad(x: torch.Tensor, nh: int, hd: int) -> torch.Tensor:
    out = torch.empty((x.shape[0], nh * _TC_HD), device=x.device, dtype=x.dtype)
    zero_(out)
    for h in range(nh):
        copy2d(x[:, h * hd:(h + 1) * hd], out[:, h * _TC_HD:h * _TC_HD + hd])
    return out


def _unpad(xp: torch.Tensor, out: torch.Tensor, nh: int, hd: int) -> torch.Tensor:
    for h in range(nh):
        copy2d(xp[:, h * _TC_HD:h * _TC_HD + hd], out[:, h * hd:(h + 1) * hd])
    return out


def attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo: bool = False):
    """Returns (o, lse) or, with want_lo (bf16), (o, lse, o_lo): o_lo = o - bf16(o) for the
    backward's delta (cb_attention_fwd)."""
    o = torch.empty((B * T, H * hd), device=q.device, dtype=q.dtype)
    lse = torch.empty((B, H, T), device=q.device, dtype=torch.float32)
    o_lo = torch.empty_like(o) if (want_lo and q.dtype == torch.bfloat16) else None
    if _pad_ok(q, hd):
        qp, kp, vp = _pad(q, H, hd), _pad(k, KVH, hd), _pad(v, KVH, hd)
        op = torch.empty((B * T, H * _TC_HD), device=q.device, dtype=q.dtype)
        olp = torch.empty_like(op) if o_lo is not None else None
        _profiled("attn_fwd", 4 * B * T * T * H * hd, _lib.call, "cb_attention_fwd", B, T, H, KVH, _TC_HD, dt(q),
                  qp.data_ptr(), ld(qp), kp.data_ptr(), ld(kp), vp.data_ptr(), ld(vp), op.data_ptr(), ld(op),
                  _ptr(olp), lse.data_ptr(), float(scale), stream_ptr())
        _unpad(op, o, H, hd)
        if o_lo is not None:
            _unpad(olp, o_lo, H, hd)
    else:
        _profiled("attn_fwd", 4 * B * T * T * H * hd, _lib.call, "cb_attention_fwd", B, T, H, KVH, hd, dt(q),
                  q.data_ptr(), ld(q), k.data_ptr(), ld(k), v.data_ptr(), ld(v), o.data_ptr(), ld(o), _ptr(o_lo),
                  lse.data_ptr(), float(scale), stream_ptr())
    return (o, lse, o_lo) if want_lo else (o, lse)


def _attention_bwd_padded(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, scale, o_lo):
    qp, kp, vp, op, dop = _pad(q, H, hd), _pad(k, KVH, hd), _pad(v, KVH, hd), _pad(o, H, hd), _pad(do, H, hd)
    olp = _pad(o_lo, H, hd) if o_lo is not None else None
    dqp, dkp, dvp = torch.empty_like(qp), torch.empty_like(kp), torch.empty_like(vp)
    delta = torch.empty((B, H, T), device=q.device, dtype=torch.float32)
    ws = _ds_workspace(qp, B, T, H, _TC_HD)
    _profiled("attn_bwd", 8 * B * T * T * H * hd, _lib.call, "cb_attention_bwd", B, T, H, KVH, _TC_HD, dt(q),
              qp.data_ptr(), ld(qp), kp.data_ptr(), ld(kp), vp.data_ptr(), ld(vp), op.data_ptr(), ld(op), _ptr(olp),
              lse.data_ptr(), dop.data_ptr(), ld(dop), delta.data_ptr(), dqp.data_ptr(), ld(dqp), dkp.data_ptr(),
              ld(dkp), dvp.data_ptr(), ld(dvp), float(scale), _ptr(ws), ws.numel() * 2 if ws is not None else 0,
              stream_ptr())
    _unpad(dqp, dq, H, hd)
    _unpad(dkp, dk, KVH, hd)
    _unpad(dvp, dv, KVH, hd)


# tcgen05 backward with dQ as a GEMM over the dS^T the dK/dV sweep stores (cb_attention_bwd
# ds_ws): 5 MMA units per tile pair instead of 7.  Measured no faster (7B 1693 vs 1693 us,
# 1B 3532 vs 3230 us, profiles/r02_attn_dq_gemm_ab.log): staging dS^T through shared memory
# costs the already shared-memory-bound dK/dV sweep +28-43%, and the dQ GEMM streams dS at
# ~4.2 TB/s.  Opt-in with CB_ATTN_DQ_GEMM=1 (tested either way).
_DQ_GEMM = __import__("os").environ.get("CB_ATTN_DQ_GEMM", "0") == "1"


# the backward's dQ sweep on CTA pairs (cb_attention_set_dq_pair; seq_len % 256 == 0):
# bit-identical to the single-CTA sweep and 11-14% faster in the step (profiles/r02_attn_dq_pair_ab.txt).
# Default on; CB_ATTN_DQ_PAIR=0 restores the single-CTA sweep.  Applied on first use.
_DQ_PAIR = __import__("os").environ.get("CB_ATTN_DQ_PAIR", "1") == "1"
_DQ_PAIR_SET = None


_DKDV_PAIR = __import__("os").environ.get("CB_ATTN_DKDV_PAIR", "0") == "1"
_DKDV_PAIR_SET = None


def set_dq_pair(enable: bool) -> None:
    global _DQ_PAIR, _DQ_PAIR_SET
    _DQ_PAIR = bool(enable)
    _lib.call("cb_attention_set_dq_pair", int(_DQ_PAIR))
    _DQ_PAIR_SET = _DQ_PAIR


def set_dkdv_pair(enable: bool) -> None:
    """The backward's dK/dV sweep on CTA pairs (cb_attention_set_dkdv_pair; seq_len % 256 == 0)."""
    global _DKDV_PAIR, _DKDV_PAIR_SET
    _DKDV_PAIR = bool(enable)
    _lib.call("cb_attention_set_dkdv_pair", int(_DKDV_PAIR))
    _DKDV_PAIR_SET = _DKDV_PAIR


def _sync_dq_pair() -> None:
    if _DQ_PAIR_SET != _DQ_PAIR:
        set_dq_pair(_DQ_PAIR)
    if _DKDV_PAIR_SET != _DKDV_PAIR:
        set_dkdv_pair(_DKDV_PAIR)


def _ds_workspace(q, B, T, H, hd):
    """The dS^T workspace (B*H*T*T bf16) when the dS path applies, else None."""
    _sync_dq_pair()
    if not (_DQ_GEMM and q.dtype == torch.bfloat16 and hd == _TC_HD and T % 128 == 0 and _ATTN_PATH == 0):
        return None
    return torch.empty((B * H * T * T,), device=q.device, dtype=torch.bfloat16)


def attention_bwd_rope(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, scale, cos_t, sin_t, o_lo=None):
    if _pad_ok(q, hd):
        _attention_bwd_padded(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, scale, o_lo)
        rope_(dq, T, H, hd, cos_t, sin_t, inverse=True)
        rope_(dk, T, KVH, hd, cos_t, sin_t, inverse=True)
        return
    delta = torch.empty((B, H, T), device=q.device, dtype=torch.float32)
    ws = _ds_workspace(q, B, T, H, hd)
    # algorithmic FLOPs: 2x forward (dP, dV, dQ, dK), the reference's backward_multiplier (mesh.py:644)
    _profiled("attn_bwd", 8 * B * T * T * H * hd, _lib.call, "cb_attention_bwd_rope", B, T, H, KVH, hd, dt(q),
              q.data_ptr(), ld(q), k.data_ptr(), ld(k), v.data_ptr(), ld(v), o.data_ptr(), ld(o), _ptr(o_lo),
              lse.data_ptr(), do.data_ptr(), ld(do), delta.data_ptr(), dq.data_ptr(), ld(dq), dk.data_ptr(), ld(dk),
              dv.data_ptr(), ld(dv), float(scale), cos_t.data_ptr(), sin_t.data_ptr(), _ptr(ws),
              ws.numel() * 2 if ws is not None else 0, stream_ptr())


def attention_bwd(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, scale, o_lo=None):
    if _pad_ok(q, hd):
        return _attention_bwd_padded(q, k, v, o, lse, do, dq, dk, dv, B, T, H, KVH, hd, scale, o_lo)
    delta = torch.empty((B, H, T), device=q.device, dtype=torch.float32)
    ws = _ds_workspace(q, B, T, H, hd)
    _profiled("attn_bwd", 8 * B * T * T * H * hd, _lib.call, "cb_attention_bwd", B, T, H, KVH, hd, dt(q),
              q.data_ptr(), ld(q), k.data_ptr(), ld(k), v.data_ptr(), ld(v), o.data_ptr(), ld(o), _ptr(o_lo),
              lse.data_ptr(), do.data_ptr(), ld(do), delta.data_ptr(), dq.data_ptr(), ld(dq), dk.data_ptr(), ld(dk),
              dv.data_ptr(), ld(dv), float(scale), _ptr(ws), ws.numel() * 2 if ws is not None else 0, stream_ptr())


def xent(logits2d: torch.Tensor, tokens: torch.Tensor, dlogits: torch.Tensor | None, grad_scale: float):
    B, T = tokens.shape
    V = logits2d.shape[1]
    row_loss = torch.empty((B * T,), device=logits2d.device, dtype=torch.float32)
    loss = torch.empty((1,), device=logits2d.device, dtype=torch.float64)
    _lib.call("cb_xent_fwd_bwd", B, T, V, logits2d.data_ptr(), ld(logits2d), dt(logits2d), tokens.data_ptr(),
              row_loss.data_ptr(), _ptr(dlogits), ld(dlogits) if dlogits is not None else 0,
              dt(dlogits) if dlogits is not None else 0, float(grad_scale), loss.data_ptr(), None, stream_ptr())
    return loss


# ---------------------------------------------------------------------------- AdamW
def adamw(param, grad, m, v, param_bf16, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0):
    n = param.numel()
    _lib.call("cb_adamw", n, param.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), _ptr(param_bf16),
              float(lr), float(beta1), float(beta2), float(eps), float(weight_decay), int(step), float(grad_scale),
              stream_ptr())


def adamw_parts(parts: list, scale: float, grad_out, param, m, v, param_bf16, lr, beta1, beta2, eps, weight_decay,
                step):
    """AdamW with grad = scale * sum(parts) in list order (cb_adamw_parts: bit-identical to
    sum_parts + adamw, without the summed gradient's HBM round trip)."""
    import ctypes

    n = param.numel()
    for t in parts:
        if t.dtype != torch.float32 or t.numel() != n:
            raise ShapeError("adamw_parts: f32 parts of the parameter's size expected")
    ptrs = (ctypes.c_void_p * len(parts))(*[t.data_ptr() for t in parts])
    _lib.call("cb_adamw_parts", n, len(parts), ctypes.addressof(ptrs), float(scale), _ptr(grad_out), param.data_ptr(),
              m.data_ptr(), v.data_ptr(), _ptr(param_bf16), float(lr), float(beta1), float(beta2), float(eps),
              float(weight_decay), int(step), stream_ptr())
