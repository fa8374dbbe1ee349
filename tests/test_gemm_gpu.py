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
    ops.set_gemm_path(1)  # the SIMT engine itself (large f32 GEMMs otherwise take the BF16x6 path)
    try:
        ops.gemm(a, b, out, trans_a=ta, trans_b=tb)
    finally:
        ops.set_gemm_path(0)
    ref = _ref(a.double(), b.double(), ta, tb).float()
    rel = (out - ref).norm() / ref.norm()
    assert rel < 1e-6, f"rel err {rel}"


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (264, 520, 200), (1024, 768, 2048), (512, 256, 4096)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False)])
def test_gemm_f32_bf16x6_on_tcgen05(cuda, M, N, K, ta, tb):
    """f32 GEMMs of the parity mode on the tcgen05 engine: six bf16 products of the operands'
    three-term splits accumulated in f32 (the BF16x6 FP32 emulation) agree with an fp64 GEMM to
    fp32 accuracy, alpha / accumulate / residual included, and with the SIMT f32 engine."""
    from paper_2507_05411_b200 import ops

    a, b = _operands(M, N, K, ta, tb, torch.float32, cuda)
    g = torch.Generator(device="cpu").manual_seed(K)
    res = torch.randn(M, N, generator=g).to(cuda)
    out0 = torch.randn(M, N, generator=g).to(cuda)
    out = out0.clone()
    ops.set_f32_tc(True)
    try:
        ops.gemm(a, b, out, trans_a=ta, trans_b=tb, alpha=0.5, accumulate=True, residual=res)
    finally:
        ops.set_f32_tc(False)
    torch.cuda.synchronize()
    ref = 0.5 * _ref(a.double(), b.double(), ta, tb) + out0.double() + res.double()
    # fp32-level: ~1e-7 per 128-long K chunk, ~sqrt(passes) * 2^-24 from the epilogue adds
    assert ((out.double() - ref).norm() / ref.norm()).item() < 2e-6
    simt = out0.clone()
    ops.set_gemm_path(1)
    try:
        ops.gemm(a, b, simt, trans_a=ta, trans_b=tb, alpha=0.5, accumulate=True, residual=res)
    finally:
        ops.set_gemm_path(0)
    torch.cuda.synchronize()
    assert ((out - simt).norm() / simt.norm()).item() < 2e-6


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


@pytest.mark.parametrize("M,K,H", [(512, 256, 384), (300, 128, 640), (1024, 512, 1152)])
@pytest.mark.parametrize("acts", [("linear", "silu"), ("relu", "linear"), ("silu", "tanh")])
def test_gemm_gated_epilogues_match_unfused(cuda, M, K, H, acts):
    """The CTA-pair GEMM with the gated activation in its epilogue (forward) and the
    activation backward fused into the w2 dgrad GEMM equal the unfused gemm + act kernels."""
    from paper_2507_05411_b200 import ops

    g = torch.Generator(device="cpu").manual_seed(M + K + H)
    x = (torch.randn(M, K, generator=g) * 0.5).to(cuda, torch.bfloat16)
    wcat = (torch.randn(K, 2 * H, generator=g) / K ** 0.5).to(cuda, torch.bfloat16)
    w2 = (torch.randn(H, K, generator=g) / H ** 0.5).to(cuda, torch.bfloat16)
    dy = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)

    fused = ops.gemm_gated_fwd(x, wcat, *acts)
    assert fused is not None, "fused forward declined an eligible shape"
    pre_f, hid_f = fused
    pre_u = torch.empty(M, 2 * H, device=cuda, dtype=torch.bfloat16)
    ops.gemm(x, wcat, pre_u)
    hid_u = ops.act_fwd(pre_u[:, :H], pre_u[:, H:], *acts)
    torch.cuda.synchronize()
    assert torch.equal(pre_f, pre_u)
    assert ((hid_f.float() - hid_u.float()).norm() / hid_u.float().norm()) < 1e-6

    dpre_f = ops.gemm_gated_bwd(dy, w2, pre_u, *acts)
    assert dpre_f is not None, "fused backward declined an eligible shape"
    dh = torch.empty(M, H, device=cuda, dtype=torch.bfloat16)
    ops.gemm(dy, w2, dh, trans_b=True)
    dpre_u = torch.empty_like(pre_u)
    ops.act_bwd(pre_u[:, :H], pre_u[:, H:], dh, dpre_u[:, :H], dpre_u[:, H:], *acts)
    torch.cuda.synchronize()
    err = (dpre_f.float() - dpre_u.float()).norm() / dpre_u.float().norm()
    assert err < 1e-4, f"rel err {err}"  # a few bf16 ulps from operation order


def test_gemm_gated_declines_ineligible(cuda):
    """Shapes the fused epilogue cannot take return None (nothing launched) instead of failing."""
    from paper_2507_05411_b200 import ops

    x = torch.randn(128, 64, device=cuda).bfloat16()  # M < 256: no CTA pair
    wcat = torch.randn(64, 256, device=cuda).bfloat16()
    assert ops.gemm_gated_fwd(x, wcat, "linear", "silu") is None
    x = torch.randn(512, 64, device=cuda).bfloat16()
    wcat = torch.randn(64, 2 * 96, device=cuda).bfloat16()  # H % 128 != 0
    assert ops.gemm_gated_fwd(x, wcat, "linear", "silu") is None


@pytest.mark.parametrize("M,N,K,ta,tb", [(512, 512, 16384, 1, 0), (640, 768, 8192, 0, 1), (2048, 1024, 32768, 1, 0)])
def test_gemm_split_k_matches(cuda, M, N, K, ta, tb):
    """Few tiles + long K take the split-K route (f32 partials in the registered workspace,
    summed in a fixed order by a second kernel): same result as the single pass within f32
    rounding, bit-reproducible across calls, and the epilogue (alpha / accumulate / residual /
    bf16 out) applied exactly once."""
    from paper_2507_05411_b200 import _lib, ops

    a, b = _operands(M, N, K, ta, tb, torch.bfloat16, cuda)
    ref = _ref(a, b, ta, tb)
    ws = torch.empty((64 << 20) // 4, device=cuda)
    r = torch.randn(M, N, device=cuda)
    outs = {}
    try:
        for mode in ("plain", "split", "split2"):
            _lib.call("cb_gemm_set_workspace", ws.data_ptr() if mode != "plain" else None,
                      ws.numel() * 4 if mode != "plain" else 0)
            acc = torch.ones(M, N, device=cuda)
            ops.gemm(a, b, acc, trans_a=bool(ta), trans_b=bool(tb), accumulate=True)
            bo = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
            ops.gemm(a, b, bo, trans_a=bool(ta), trans_b=bool(tb), alpha=0.5, residual=r)
            outs[mode] = (acc, bo)
    finally:
        _lib.call("cb_gemm_set_workspace", None, 0)
    torch.cuda.synchronize()
    for mode in ("plain", "split"):
        acc, bo = outs[mode]
        assert ((acc - 1.0 - ref).norm() / ref.norm()) < 1e-4, mode  # f32 accumulation over K up to 32768
        exp = 0.5 * ref + r
        assert ((bo.float() - exp).norm() / exp.norm()) < 1e-2, mode
    assert torch.equal(outs["split"][0], outs["split2"][0])  # deterministic


@pytest.mark.parametrize("M,N,K", [(512, 768, 320), (300, 640, 256), (1000, 2048, 512)])
def test_staged_epilogue_bit_identical(cuda, M, N, K):
    """The CTA-pair GEMM's shared-memory-staged epilogue (coalesced output / addend / gated-pre
    I/O) writes exactly what the per-lane epilogue writes, for every output mode, including
    ragged row blocks (M % 32 != 0)."""
    from paper_2507_05411_b200 import _lib, ops
    from paper_2507_05411_b200.layers import rope_tables

    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    b = (torch.randn(K, N, generator=g) / K ** 0.5).to(cuda, torch.bfloat16)
    r32 = torch.randn(M, N, generator=g).to(cuda)
    acc0 = torch.randn(M, N, generator=g).to(cuda)
    cs, sn = rope_tables(128, 128, 10000.0, cuda)
    H = N // 2
    w2 = (torch.randn(H, K, generator=g) / H ** 0.5).to(cuda, torch.bfloat16)
    pre = torch.randn(M, 2 * H, generator=g).to(cuda, torch.bfloat16)

    def run():
        outs = {}
        o = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        outs["bf16"] = ops.gemm(a, b, o).clone()
        o = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        outs["bf16_rope"] = ops.gemm_rope(a, b, o, 128, 128, max(128, N // 256 * 128), cs, sn).clone()
        o = torch.empty(M, N, device=cuda)
        outs["f32"] = ops.gemm(a, b, o, alpha=0.75).clone()
        o = torch.empty(M, N, device=cuda)
        outs["f32_res"] = ops.gemm(a, b, o, residual=r32).clone()
        o = acc0.clone()
        outs["f32_acc"] = ops.gemm(a, b, o, accumulate=True).clone()
        o = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        outs["bf16_res"] = ops.gemm(a, b, o, residual=r32).clone()  # not staged: per-lane path both times
        d = ops.gemm_gated_bwd(a, w2, pre, "linear", "silu")
        if d is not None:
            outs["glu_bwd"] = d.clone()
        torch.cuda.synchronize()
        return outs

    try:
        _lib.call("cb_gemm_set_staged_epilogue", 1)
        staged = run()
        _lib.call("cb_gemm_set_staged_epilogue", 0)
        plain = run()
    finally:
        _lib.call("cb_gemm_set_staged_epilogue", 1)
    assert staged.keys() == plain.keys()
    for k in staged:
        assert torch.equal(staged[k], plain[k]), k


def _padded_offsets(counts, dev):
    import numpy as np

    po = np.zeros(len(counts) + 1, dtype=np.int32)
    po[1:] = np.cumsum([(c + 255) // 256 * 256 for c in counts])
    return torch.tensor(po, device=dev, dtype=torch.int32), po


@pytest.mark.parametrize("counts", [[300, 0, 513, 256], [1, 1, 1, 1, 1, 1, 1, 1], [4096, 0, 0, 0, 0, 0, 0, 1000]])
def test_grouped_gemm_matches_per_group(cuda, counts):
    """cb_gemm_grouped (one launch, device offsets) == one cb_gemm per group, bit for bit:
    mode 1 (rows; B stacked along K, and transposed along N) and mode 2 (K; the experts'
    weight gradients, empty groups untouched), plus the gated forward / backward forms."""
    from paper_2507_05411_b200 import ops

    G, d, h = len(counts), 256, 512
    goff, po = _padded_offsets(counts, cuda)
    cap = int(po[-1]) + 256
    g = torch.Generator(device="cpu").manual_seed(sum(counts))
    x = torch.zeros(cap, d, dtype=torch.bfloat16)
    for e in range(G):
        x[po[e]:po[e] + counts[e]] = torch.randn(counts[e], d, generator=g)
    x = x.to(cuda)
    w = (0.05 * torch.randn(G * d, 2 * h, generator=g)).to(cuda, torch.bfloat16)  # [W1|Wg] stacked
    w2 = (0.05 * torch.randn(G * h, d, generator=g)).to(cuda, torch.bfloat16)
    # mode 1, B stacked along K
    out = torch.zeros(cap, 2 * h, device=cuda)
    ops.gemm_grouped_rows(x, w, out, goff, G)
    ref = torch.zeros_like(out)
    for e in range(G):
        r0, r1 = int(po[e]), int(po[e + 1])
        if r1 > r0:
            ops.gemm(x[r0:r1], w[e * d:(e + 1) * d], ref[r0:r1])
    torch.cuda.synchronize()
    assert torch.equal(out[:int(po[-1])], ref[:int(po[-1])])
    # mode 1, B read transposed (stacked along N): dx = dy @ W2_g^T
    dy = torch.randn(cap, d, generator=g).to(cuda, torch.bfloat16)
    dh = torch.zeros(cap, h, device=cuda)
    ops.gemm_grouped_rows(dy, w2, dh, goff, G, trans_b=True)
    ref = torch.zeros_like(dh)
    for e in range(G):
        r0, r1 = int(po[e]), int(po[e + 1])
        if r1 > r0:
            ops.gemm(dy[r0:r1], w2[e * h:(e + 1) * h], ref[r0:r1], trans_b=True)
    torch.cuda.synchronize()
    assert torch.equal(dh[:int(po[-1])], ref[:int(po[-1])])
    # mode 2: weight gradients, accumulate into a non-zero buffer; empty groups untouched
    gw = torch.randn(G * d, d, generator=g).to(cuda)
    ref = gw.clone()
    ops.gemm_grouped_k(x, dy, gw, goff, G)
    for e in range(G):
        r0, r1 = int(po[e]), int(po[e + 1])
        if r1 > r0:
            ops.gemm(x[r0:r1], dy[r0:r1], ref[e * d:(e + 1) * d], trans_a=True, accumulate=True)
    torch.cuda.synchronize()
    assert torch.equal(gw, ref)
    # gated forward / backward
    pre = torch.zeros(cap, 2 * h, device=cuda, dtype=torch.bfloat16)
    hid = torch.zeros(cap, h, device=cuda, dtype=torch.bfloat16)
    ops.gemm_gated_fwd_grouped(x, w, goff, G, "linear", "silu", pre, hid)
    dpre = torch.zeros_like(pre)
    ops.gemm_gated_bwd_grouped(dy, w2, goff, G, pre, "linear", "silu", dpre)
    rpre, rhid, rdpre = torch.zeros_like(pre), torch.zeros_like(hid), torch.zeros_like(dpre)
    for e in range(G):
        r0, r1 = int(po[e]), int(po[e + 1])
        if r1 > r0:
            ops.gemm_gated_fwd(x[r0:r1], w[e * d:(e + 1) * d], "linear", "silu", pre=rpre[r0:r1], hidden=rhid[r0:r1])
            ops.gemm_gated_bwd(dy[r0:r1], w2[e * h:(e + 1) * h], rpre[r0:r1], "linear", "silu", dpre=rdpre[r0:r1])
    torch.cuda.synchronize()
    n = int(po[-1])
    assert torch.equal(pre[:n], rpre[:n]) and torch.equal(hid[:n], rhid[:n]) and torch.equal(dpre[:n], rdpre[:n])


def test_moe_dispatch_padded(cuda):
    """cb_moe_dispatch_padded: each expert's rows start on a 256-row boundary in stable sorted
    order, pad rows are zero, and pinv maps every assignment to its padded row."""
    import numpy as np

    from paper_2507_05411_b200 import _lib, ops

    n, k, E, d = 300, 2, 4, 64
    g = torch.Generator(device="cpu").manual_seed(5)
    ids = torch.randint(0, E, (n * k,), generator=g)
    ids[ids == 2] = 1  # an empty expert
    x = torch.randn(n, d, generator=g).to(cuda, torch.bfloat16)
    off, perm = ops.sort_ids(ids.to(cuda), E)
    cap = n * k + 255 * E
    xe = torch.full((cap, d), 7.0, device=cuda, dtype=torch.bfloat16)
    poff = torch.empty(E + 1, device=cuda, dtype=torch.int32)
    pinv = torch.empty(n * k, device=cuda, dtype=torch.int32)
    _lib.call("cb_moe_dispatch_padded", n * k, d, E, k, off.data_ptr(), perm.data_ptr(), x.data_ptr(), ops.ld(x),
              ops.dt(x), poff.data_ptr(), pinv.data_ptr(), xe.data_ptr(), ops.ld(xe), cap, ops.stream_ptr())
    torch.cuda.synchronize()
    idsn, po, pi = ids.numpy(), poff.cpu().numpy(), pinv.cpu().numpy()
    counts = np.bincount(idsn, minlength=E)
    assert list(po) == [0] + list(np.cumsum([(c + 255) // 256 * 256 for c in counts]))
    xc, xec = x.cpu(), xe.cpu()
    for e in range(E):
        mine = np.nonzero(idsn == e)[0]  # stable order of the assignments
        rows = po[e] + np.arange(len(mine))
        assert np.array_equal(pi[mine], rows)
        assert torch.equal(xec[rows], xc[mine // k])
        assert not xec[po[e] + len(mine):po[e + 1]].float().any()


@pytest.mark.parametrize("M,N,K,ldd,path", [
    (2048, 3072, 1024, 3072, 0),   # CTA-pair engine, whole chunks
    (512, 384, 768, 1024, 0),      # a column block of a wider buffer (fused wq|wk|wv slice)
    (520, 200, 264, 200, 0),       # ragged tails: per-element epilogue
    (256, 96, 512, 96, 0),         # N <= 128 engine
    (96, 80, 64, 80, 0),           # below the tcgen05 work threshold: SIMT epilogue
    (256, 512, 256, 512, 1),       # forced SIMT
    (128, 256, 0, 256, 0),         # K = 0: the zero gradient's update (momentum only)
])
def test_gemm_adamw_matches_gemm_then_adamw(cuda, M, N, K, ldd, path):
    """cb_gemm_adamw (AdamW in the weight-gradient GEMM's epilogue) = cb_gemm accumulating
    into a zeroed gradient followed by cb_adamw, bit for bit, on every engine and epilogue path;
    the gradient buffer itself is never written."""
    from paper_2507_05411_b200 import _lib, ops

    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    x = torch.randn(max(K, 1), M, generator=g).to(cuda, torch.bfloat16)[:K]  # A = x^T (trans_a)
    dy = torch.randn(max(K, 1), N, generator=g).to(cuda, torch.bfloat16)[:K]
    rows = M * ldd
    p0 = torch.randn(rows, generator=g).to(cuda)
    m0 = torch.randn(rows, generator=g).to(cuda) * 1e-3
    v0 = torch.rand(rows, generator=g).to(cuda) * 1e-6
    hyper = (1e-3, 0.9, 0.999, 1e-8, 0.01, 3)
    ops.set_gemm_path(path)
    try:
        # unfused: gradient into a zeroed buffer, then AdamW over the whole buffer
        grad = torch.zeros(rows, device=cuda)
        gv = grad.view(M, ldd)[:, :N]
        ops.gemm(x, dy, gv, trans_a=True, accumulate=True, alpha=0.5)
        p1, m1, v1 = p0.clone(), m0.clone(), v0.clone()
        bf1 = torch.empty(rows, device=cuda, dtype=torch.bfloat16)
        ops.adamw(p1, grad, m1, v1, bf1, *hyper)
        # fused: only the GEMM's own elements are touched
        p2, m2, v2 = p0.clone(), m0.clone(), v0.clone()
        sentinel = torch.full((rows,), 7.0, device=cuda)
        sv = sentinel.view(M, ldd)[:, :N]
        _lib.call("cb_gemm_adamw", M, N, K, ops.dt(x), x.data_ptr(), M, 1, dy.data_ptr(), N, 0, sv.data_ptr(), ldd,
                  0.5, p2.data_ptr(), m2.data_ptr(), v2.data_ptr(), None, *[float(h) for h in hyper[:5]], hyper[5],
                  ops.stream_ptr())
    finally:
        ops.set_gemm_path(0)
    assert torch.equal(sentinel, torch.full_like(sentinel, 7.0))
    sel = torch.zeros(M, ldd, dtype=torch.bool, device=cuda)
    sel[:, :N] = True
    sel = sel.view(-1)
    assert torch.equal(p2[sel], p1[sel]) and torch.equal(m2[sel], m1[sel]) and torch.equal(v2[sel], v1[sel])
    assert torch.equal(p2[~sel], p0[~sel]) and torch.equal(m2[~sel], m0[~sel])
