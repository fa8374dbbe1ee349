"""Thin tensor-level wrappers over the C ABI (device pointers + stream from torch).

PyTorch is used only for device memory and streams: every arithmetic operation below
is one call into ``libcomposer_b200.so``.  Shapes/dtypes are checked here, before the
launch, and raise the reference's error classes.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import ShapeError, TypeMismatchError

_DT = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16}


def dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeMismatchError(f"unsupported tensor dtype {t.dtype}") from None


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _rowmajor_ld(t: torch.Tensor, what: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ShapeError(f"{what} must be a 2-D row-major view (stride(1) == 1)")
    return t.stride(0)


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
        ldr = _rowmajor_ld(residual, "residual")
    _lib.call(
        "cb_gemm", M, N, K, dt(a), a.data_ptr(), _rowmajor_ld(a, "A"), int(trans_a), b.data_ptr(),
        _rowmajor_ld(b, "B"), int(trans_b), out.data_ptr(), _rowmajor_ld(out, "out"), dt(out), _ptr(residual), ldr,
        dt(residual) if residual is not None else 0, float(alpha), int(accumulate), stream_ptr(),
    )
    return out


def set_gemm_path(path: int) -> None:
    _lib.call("cb_gemm_set_path", int(path))
