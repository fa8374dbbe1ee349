"""ctypes binding of the C ABI in ``include/composer_b200.h``.

The library is loaded from the package's ``_lib/`` directory (built by ``_build.py``).
There is no fallback: if the shared object is missing or a symbol is absent the caller
gets ``MissingExtensionError``.  Non-zero statuses become the matching ComposerError
subclass (CB_ERR_SHAPE -> ShapeError, CB_ERR_UNSUPPORTED -> TypeMismatchError,
otherwise KernelError) carrying the library's thread-local message.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import KernelError, MissingExtensionError, ShapeError, TypeMismatchError

_PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG_DIR, "_lib", "libcomposer_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG_DIR), "include", "composer_b200.h")

CB_OK, CB_ERR_SHAPE, CB_ERR_ARG, CB_ERR_CUDA, CB_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
DT_F32, DT_BF16 = 0, 1

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_F = ctypes.c_float
_D = ctypes.c_double

# name -> argtypes; the return type is always int (status) except those in RESTYPES.
RESTYPES = {"cb_sort_ids_scratch": ctypes.c_int64}
SIGNATURES: dict[str, list] = {
    "cb_abi_version": [],
    "cb_gemm_set_path": [_I],
    "cb_gemm_set_multicast": [_I],
    "cb_gemm_set_staged_epilogue": [_I],
    "cb_gemm": [_I, _I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _I, _P, _L, _I, _F, _I, _P],
    "cb_gemm_adamw": [_I, _I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _F, _P, _P, _P, _P, _F, _F, _F, _F, _F, _I,
                      _P],
    "cb_rmsnorm_fwd": [_I, _I, _P, _L, _I, _P, _F, _P, _L, _I, _P, _P],
    "cb_rmsnorm_bwd_workspace": [_I, _I, ctypes.POINTER(ctypes.c_int64)],
    "cb_rmsnorm_bwd": [_I, _I, _P, _L, _I, _P, _P, _P, _L, _I, _P, _L, _P, _L, _P, _L, _P, _P, _P],
    "cb_col_reduce": [_I, _I, _P, _P, _I, _P],
    "cb_embedding_fwd": [_L, _I, _P, _P, _L, _I, _P, _L, _I, _P],
    "cb_sort_ids_scratch": [_I, _I],
    "cb_sort_ids": [_I, _I, _P, _P, _P, _P, _P],
    "cb_embedding_bwd": [_I, _I, _P, _P, _P, _L, _I, _P, _L, _P],
    "cb_rope": [_L, _I, _I, _I, _P, _L, _I, _P, _P, _I, _P],
    "cb_act_fwd": [_L, _I, _I, _I, _P, _L, _P, _L, _P, _L, _I, _P],
    "cb_act_bwd": [_L, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _P, _L, _I, _P],
    "cb_copy2d": [_L, _I, _P, _L, _I, _P, _L, _I, _F, _I, _P],
    "cb_memset_zero": [_P, _L, _P],
    "cb_sum_parts": [_I, _L, _P, _P, _F, _P],
    "cb_split_bf16x3": [_L, _I, _P, _L, _P, _P, _P, _P],
    "cb_gemm_set_raster": [_I],
    "cb_stream_signal": [_P, _I, ctypes.c_uint32, _P],
    "cb_stream_wait": [_P, _I, ctypes.c_uint32, _P],
    "cb_attention_fwd": [_I, _I, _I, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _P, _P, _F, _P],
    "cb_attention_bwd": [_I, _I, _I, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _P, _P, _P, _L, _P, _P, _L, _P,
                         _L, _P, _L, _F, _P, _L, _P],
    "cb_attention_set_path": [_I],
    "cb_attention_set_dq_pair": [_I],
    "cb_attention_set_dkdv_pair": [_I],
    "cb_gemm_rope": [_I, _I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _I, _I, _I, _I, _P, _P, _P],
    "cb_gemm_set_workspace": [_P, _L],
    "cb_gemm_gated_fwd": [_I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _P, _L, _I, _I, _P],
    "cb_gemm_gated_bwd": [_I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _P, _L, _I, _I, _P],
    "cb_attention_bwd_rope": [_I, _I, _I, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _P, _P, _P, _L, _P, _P, _L,
                              _P, _L, _P, _L, _F, _P, _P, _P, _L, _P],
    "cb_attention_set_tc": [_I],
    "cb_gemm_grouped": [_I, _I, _P, _I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _I, _F, _I, _P],
    "cb_gemm_gated_fwd_grouped": [_I, _P, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _I, _I, _P],
    "cb_gemm_gated_bwd_grouped": [_I, _P, _I, _I, _I, _P, _L, _P, _L, _P, _L, _P, _L, _I, _I, _P],
    "cb_moe_dispatch_padded": [_L, _I, _I, _I, _P, _P, _P, _L, _I, _P, _P, _P, _L, _I, _P],
    "cb_moe_zero_pad_rows": [_I, _I, _I, _P, _P, _P, _L, _I, _P],
    "cb_xent_fwd_bwd": [_I, _I, _I, _P, _L, _I, _P, _P, _P, _L, _I, _F, _P, _P, _P],
    "cb_adamw": [_L, _P, _P, _P, _P, _P, _F, _F, _F, _F, _F, _I, _F, _P],
    "cb_adamw_parts": [_L, _I, _P, _F, _P, _P, _P, _P, _P, _F, _F, _F, _F, _F, _I, _P],
    "cb_moe_route": [_L, _I, _I, _I, _P, _L, _I, _P, _P, _P, _P, _P],
    "cb_moe_stats": [_L, _I, _I, _P, _P, _P, _P],
    "cb_gather_rows": [_L, _I, _P, _I, _P, _L, _P, _L, _I, _P],
    "cb_moe_combine_residual": [_L, _I, _I, _P, _P, _P, _L, _P, _L, _P, _L, _P],
    "cb_moe_combine": [_L, _I, _I, _P, _P, _P, _L, _I, _P, _L, _I, _P],
    "cb_moe_combine_bwd": [_L, _I, _I, _P, _P, _P, _L, _P, _L, _P, _L, _I, _P, _P],
    "cb_moe_router_bwd": [_L, _I, _I, _P, _P, _P, _P, _P, _P],
    "cb_invert_perm": [_L, _P, _P, _P],
    "cb_moe_router_bwd_gemms": [_L, _I, _I, _P, _L, _I, _P, _P, _P, _P, _L, _P, _P],
    "cb_widen_i32": [_L, _P, _P, _P],
    "cb_init_uniform": [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _L, _D, _D, _L, _L, _L,
                        _L, _P, _L, _L, _P, _I, _P],
    "cb_init_const": [_L, _F, _L, _L, _L, _L, _P, _L, _L, _P, _I, _P],
}

_lib = None


def declared_symbols() -> list[str]:
    """Function names declared with CB_API in the public header."""
    with open(HEADER_PATH, "r", encoding="utf-8") as fh:
        text = fh.read()
    return re.findall(r"CB_API\s+[\w\s\*]+?\b(cb_\w+)\s*\(", text)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MissingExtensionError(
            f"kernel library not built: {LIB_PATH} (run __graft_entry__.build() or python -m paper_2507_05411_b200._build)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            raise MissingExtensionError(f"kernel library lacks symbol {name}") from None
        fn.argtypes = argtypes
        fn.restype = RESTYPES.get(name, ctypes.c_int)
    lib.cb_last_error.argtypes = []
    lib.cb_last_error.restype = ctypes.c_char_p
    lib.cb_launch_count.argtypes = []
    lib.cb_launch_count.restype = ctypes.c_longlong
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels launched through the library so far in this process."""
    return int(load().cb_launch_count())


def check(status: int, what: str = "") -> None:
    if status == CB_OK:
        return
    msg = (_lib.cb_last_error() or b"").decode("utf-8", "replace") if _lib is not None else ""
    text = f"{what}: {msg}" if what else msg
    if status == CB_ERR_SHAPE:
        raise ShapeError(text)
    if status == CB_ERR_UNSUPPORTED:
        raise TypeMismatchError(text)
    raise KernelError(f"status {status}: {text}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def try_call(name: str, *args) -> bool:
    """Like call(), but CB_ERR_UNSUPPORTED (the entry point declined; nothing launched)
    returns False so the caller can take its unfused GPU route."""
    lib = load()
    status = getattr(lib, name)(*args)
    if status == CB_ERR_UNSUPPORTED:
        return False
    check(status, name)
    return True
