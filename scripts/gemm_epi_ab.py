"""A/B of the CTA-pair GEMM epilogue on the 1B layer shapes: shared-memory-staged (coalesced)
vs per-lane row stores; TFLOP/s per shape, interleaved on the same box.  Masks (see
cb_gemm_set_staged_epilogue): 3 bf16 outputs and gated backward staged, 0 none."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import _lib, ops

dev = torch.device("cuda")
T, d, qkv, ffn = 32768, 2048, 6144, 5632


def timed(fn, n=40):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


x = torch.randn(T, d, device=dev).bfloat16()
cases = {}
w = torch.randn(d, qkv, device=dev).bfloat16()
o = torch.empty(T, qkv, device=dev, dtype=torch.bfloat16)
cases["fwd_qkv_bf16"] = (lambda: ops.gemm(x, w, o), 2 * T * qkv * d)
wo = torch.randn(d, d, device=dev).bfloat16()
res = torch.randn(T, d, device=dev)
o32 = torch.empty(T, d, device=dev)
cases["fwd_o_f32_residual"] = (lambda: ops.gemm(x, wo, o32, residual=res), 2 * T * d * d)
h = torch.randn(T, ffn, device=dev).bfloat16()
w2 = torch.randn(ffn, d, device=dev).bfloat16()
cases["fwd_down_f32_residual"] = (lambda: ops.gemm(h, w2, o32, residual=res), 2 * T * d * ffn)
wq = torch.randn(d, qkv, device=dev).bfloat16()
dq = torch.randn(T, qkv, device=dev).bfloat16()
cases["dgrad_qkv_f32_acc"] = (lambda: ops.gemm(dq, wq, o32, trans_b=True, accumulate=True), 2 * T * d * qkv)
pre = torch.randn(T, 2 * ffn, device=dev).bfloat16()
dy = torch.randn(T, d, device=dev).bfloat16()
dpre = torch.empty_like(pre)
cases["glu_bwd"] = (lambda: ops.gemm_gated_bwd(dy, w2, pre, "linear", "silu", dpre=dpre), 2 * T * ffn * d)
wcat = torch.randn(d, 2 * ffn, device=dev).bfloat16()
cases["glu_fwd"] = (lambda: ops.gemm_gated_fwd(x, wcat, "linear", "silu", pre=pre, hidden=h), 2 * T * 2 * ffn * d)
for name, (fn, flops) in cases.items():
    r = {"gemm": name}
    for rep in range(3):
        for mode in (3, 0):
            _lib.call("cb_gemm_set_staged_epilogue", mode)
            ms = timed(fn)
            r.setdefault(f"mask{mode}", []).append(round(flops / ms / 1e9, 1))
    _lib.call("cb_gemm_set_staged_epilogue", 1)
    print(json.dumps(r), flush=True)
