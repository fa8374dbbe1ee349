"""Times the fused gated-activation GEMMs against gemm + act kernels at the 1B FFN shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_05411_b200 import ops

dev = torch.device("cuda")
M, K, H = 32768, 2048, 5632
x = torch.randn(M, K, device=dev).bfloat16()
wcat = (torch.randn(K, 2 * H, device=dev) / K ** 0.5).bfloat16()
w2 = (torch.randn(H, K, device=dev) / H ** 0.5).bfloat16()
dy = torch.randn(M, K, device=dev).bfloat16()
pre = torch.empty(M, 2 * H, device=dev, dtype=torch.bfloat16)
dh = torch.empty(M, H, device=dev, dtype=torch.bfloat16)


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


res = {
    "fwd_fused_ms": t(lambda: ops.gemm_gated_fwd(x, wcat, "linear", "silu")),
    "fwd_gemm_ms": t(lambda: ops.gemm(x, wcat, pre)),
    "fwd_act_ms": t(lambda: ops.act_fwd(pre[:, :H], pre[:, H:], "linear", "silu")),
    "bwd_fused_ms": t(lambda: ops.gemm_gated_bwd(dy, w2, pre, "linear", "silu")),
    "bwd_gemm_ms": t(lambda: ops.gemm(dy, w2, dh, trans_b=True)),
}
dpre = torch.empty_like(pre)
res["bwd_act_ms"] = t(lambda: ops.act_bwd(pre[:, :H], pre[:, H:], dh, dpre[:, :H], dpre[:, H:], "linear", "silu"))
print({k: round(v, 3) for k, v in res.items()})
