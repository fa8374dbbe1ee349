"""GEMM engine parity against a plain PyTorch fp32 reference of the same op."""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 128, 64),
    (256, 512, 256),
    (264, 520, 200),  # ragged M/N/K tails (TMA OOB fill + predicated epilogue)
    (1024, 2048, 2048),
    (2048, 5632, 2048),
    (4096, 2048, 5632),
]


def _ref(a, b, ta, tb):
    A = a.float().t() if ta else a.float()
    B = b.float().t() if tb else b.float()
    return A @ B


def _operands(M, N, K, ta, tb, dtype, dev):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    a = torch.randn((K, M) if ta else (M, K), generator=g).to(dev, dtype)
    b = torch.randn((N, K) if tb else (K, N), generator=g).to(dev, dtype)
    return a, b


@pytest.mark.parametrize("M,N,K", SHAPES + [(384, 768, 512), (640, 256, 128)])  # odd tile-pair counts
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("mc", [1, 2, 0])  # CTA pair, B-multicast pair, single CTA
def test_gemm_tcgen05_bf16(cuda, M, N, K, ta, tb, mc):
    from paper_2507_05411_b200 import _lib, ops

    a, b = _operands(M, N, K, ta, tb, torch.bfloat16, cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.float32)
    ops.set_gemm_path(2)
    _lib.call("cb_gemm_set_multicast", mc)
    try:
        ops.gemm(a, b, out, trans_a=ta, trans_b=tb)
    finally:
        ops.set_gemm_path(0)
        _lib.call("cb_gemm_set_multicast", 1)
    torch.cuda.synchronize()
    ref = _ref(a, b, ta, tb)
    rel = (out - ref).norm() / ref.norm()
    assert rel < 1e-5, f"rel err {rel}"


@pytest.mark.parametrize("M,N,K", SHAPES[:3])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False)])
def test_gemm_simt_f32(cuda, M, N, K, ta, tb):
    from paper_2507_05411_b200 import ops

    a, b = _operands(M, N, K, ta, tb, torch.float32, cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.float32)
    ops.gemm(a, b, out, trans_a=ta, trans_b=tb)
    ref = _ref(a.double(), b.double(), ta, tb).float()
    rel = (out - ref).norm() / ref.norm()
    assert rel < 1e-6, f"rel err {rel}"


def test_gemm_epilogues(cuda):
    from paper_2507_05411_b200 import ops

    M, N, K = 512, 768, 320
    a, b = _operands(M, N, K, False, False, torch.bfloat16, cuda)
    ref = _ref(a, b, False, False)
    for path in (1, 2):
        ops.set_gemm_path(path)
        try:
            r = torch.randn(M, N, device=cuda)
            out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
            ops.gemm(a, b, out, alpha=0.5, residual=r)
            exp = 0.5 * ref + r
            assert ((out.float() - exp).norm() / exp.norm()) < 1e-2
            acc = torch.randn(M, N, device=cuda)
            exp2 = acc + ref
            ops.gemm(a, b, acc, accumulate=True)
            assert ((acc - exp2).norm() / exp2.norm()) < 1e-5
        finally:
            ops.set_gemm_path(0)
