"""Kernel-level numerics against plain PyTorch fp32/fp64 references of the same op."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("rows,dim,dt", [(64, 128, torch.float32), (300, 2048, torch.bfloat16), (7, 32, torch.float32)])
def test_rmsnorm(cuda, rows, dim, dt):
    from paper_2507_05411_b200 import ops

    g = torch.Generator().manual_seed(rows)
    x = torch.randn(rows, dim, generator=g).to(cuda)
    s = (1 + 0.1 * torch.randn(dim, generator=g)).to(cuda)
    y, rstd = ops.rmsnorm_fwd(x, s, 1e-6, dt)
    xr = x.double().requires_grad_(True)
    sr = s.double().requires_grad_(True)
    yr = xr / torch.sqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * sr
    assert _rel(y.float(), yr.detach()) < (1e-6 if dt == torch.float32 else 8e-3)
    dy = torch.randn(rows, dim, generator=g).to(cuda)
    dres = torch.randn(rows, dim, generator=g).to(cuda)
    yr.backward(dy.double())
    dscale = torch.zeros(dim, device=cuda)
    dx = ops.rmsnorm_bwd(x, s, rstd, dy.to(dt), dres=dres, dscale=dscale)
    tol = 1e-5 if dt == torch.float32 else 1e-2
    assert _rel(dx, xr.grad + dres.double()) < tol
    assert _rel(dscale, sr.grad) < tol


@pytest.mark.parametrize("V,scale,gdt", [
    (1000, 3.0, torch.float32),      # register-resident row kernel
    (32000, 3.0, torch.bfloat16),    # the 1B / 7B head: bf16 gradient
    (32000, 60.0, torch.float32),    # wide logit range: per-thread maxima far below the row max
    (1001, 3.0, torch.float32),      # V % 4 != 0: streaming kernel
    (40000, 3.0, torch.float32),     # row larger than the register kernel holds
])
def test_xent_matches_torch(cuda, V, scale, gdt):
    from paper_2507_05411_b200 import ops

    B, T = 3, 17
    g = torch.Generator().manual_seed(V)
    logits = (scale * torch.randn(B * T, V, generator=g)).to(cuda)
    toks = torch.randint(0, V, (B, T), generator=g).to(cuda)
    dl = torch.empty(B * T, V, device=cuda, dtype=gdt)
    loss = ops.xent(logits, toks, dl, 1.0 / (B * (T - 1)))
    lr = logits.double().view(B, T, V).requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lr[:, :-1].reshape(-1, V), toks[:, 1:].reshape(-1))
    ref.backward()
    refv = float(ref.detach())
    assert abs(float(loss.item()) - refv) < 1e-6 * max(1.0, refv)
    assert _rel(dl.float(), lr.grad.view(B * T, V)) < (1e-5 if gdt == torch.float32 else 1e-2)


@pytest.mark.parametrize("B,T,H,KVH,hd,dt,path", [
    (2, 64, 4, 4, 32, torch.float32, 1),
    (1, 100, 4, 2, 16, torch.float32, 1),
    (2, 256, 8, 8, 128, torch.bfloat16, 0),
    (1, 384, 8, 2, 128, torch.bfloat16, 0),
    (2, 128, 4, 4, 64, torch.bfloat16, 0),   # head_dim 64: zero-padded onto the tcgen05 kernels
    (2, 128, 4, 2, 32, torch.bfloat16, 0),   # head_dim 32: same
    (2, 200, 4, 2, 128, torch.bfloat16, 0),  # ragged T: masked key tiles + rows crossing into the next sequence
    (2, 200, 4, 2, 128, torch.bfloat16, 2),  # same, tcgen05 disabled: the SIMT engine
    (4, 128, 2, 2, 128, torch.bfloat16, 0),  # single key tile; second query tile of the CTA is padding
    (4, 128, 2, 2, 128, torch.bfloat16, 2),
    (3, 64, 2, 1, 128, torch.bfloat16, 0),   # T < tile
    (1, 1152, 4, 4, 128, torch.bfloat16, 0),  # 9 key / query tiles: every smem ring and TMEM phase wraps
])
def test_attention_fwd_bwd(cuda, B, T, H, KVH, hd, dt, path):
    from paper_2507_05411_b200 import _lib, ops

    g = torch.Generator().manual_seed(T + hd)
    tc_off = path == 2
    if tc_off:
        _lib.call("cb_attention_set_tc", 0)
        path = 0
    d, kvd = H * hd, KVH * hd
    qkv = torch.randn(B * T, d + 2 * kvd, generator=g).to(cuda, dt)
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    scale = 1 / math.sqrt(hd)
    ops.set_attention_path(path)
    try:
        o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
        do = torch.randn(B * T, d, generator=g).to(cuda, dt)
        dqkv = torch.empty_like(qkv)
        ops.attention_bwd(q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd,
                          scale)
        # the backward is deterministic (no atomics): a second run is bit-identical
        again = torch.empty_like(qkv)
        ops.attention_bwd(q, k, v, o, lse, do, again[:, :d], again[:, d:d + kvd], again[:, d + kvd:], B, T, H, KVH,
                          hd, scale)
        assert torch.equal(again, dqkv)
    finally:
        ops.set_attention_path(0)
        _lib.call("cb_attention_set_tc", 1)
    torch.cuda.synchronize()
    Q = q.double().view(B, T, H, hd).transpose(1, 2).requires_grad_(True)
    K = k.double().view(B, T, KVH, hd).transpose(1, 2).requires_grad_(True)
    Vv = v.double().view(B, T, KVH, hd).transpose(1, 2).requires_grad_(True)
    rep = H // KVH
    P = torch.softmax(Q @ K.repeat_interleave(rep, 1).transpose(-1, -2) * scale, -1)
    O = P @ Vv.repeat_interleave(rep, 1)
    O.backward(do.double().view(B, T, H, hd).transpose(1, 2))
    # bf16: identical bf16 inputs, so the error is the kernels' own rounding (bf16 O, P and dS
    # operands of the second GEMMs, f32 accumulation): ~3e-3 expected
    tol = 1e-5 if dt == torch.float32 else 5e-3
    assert _rel(o.view(B, T, H, hd).transpose(1, 2), O.detach()) < tol
    if dt == torch.bfloat16:
        # o_lo: the forward's bf16 rounding residual; o + o_lo carries ~16 significant bits on
        # the tcgen05 path (zero from the other engines), and the backward with it agrees
        ops.set_attention_path(path)
        if tc_off:
            _lib.call("cb_attention_set_tc", 0)
        try:
            o2, _, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
            d2 = torch.empty_like(qkv)
            ops.attention_bwd(q, k, v, o2, lse, do, d2[:, :d], d2[:, d:d + kvd], d2[:, d + kvd:], B, T, H, KVH, hd,
                              scale, o_lo=o_lo)
        finally:
            ops.set_attention_path(0)
            _lib.call("cb_attention_set_tc", 1)
        torch.cuda.synchronize()
        assert torch.equal(o2, o)
        full = (o2.double() + o_lo.double()).view(B, T, H, hd).transpose(1, 2)
        if path == 0 and not tc_off:  # tcgen05 forward: the residual is real
            # o + o_lo is the kernel's f32 output: at least as close to the f64 reference as o
            # (its own error is P's bf16 rounding inside the forward)
            o_ref = O.detach()
            assert _rel(full, o_ref) <= _rel(o.view(B, T, H, hd).transpose(1, 2), o_ref)
            assert o_lo.any()
        else:
            assert not o_lo.any()
        assert _rel(d2[:, :d].view(B, T, H, hd).transpose(1, 2), Q.grad) < tol
    assert _rel(dqkv[:, :d].view(B, T, H, hd).transpose(1, 2), Q.grad) < tol
    assert _rel(dqkv[:, d:d + kvd].view(B, T, KVH, hd).transpose(1, 2), K.grad) < tol
    assert _rel(dqkv[:, d + kvd:].view(B, T, KVH, hd).transpose(1, 2), Vv.grad) < tol


@pytest.mark.parametrize("B,T,H,KVH", [(2, 256, 2, 2), (4, 128, 2, 1), (1, 200, 4, 2)])
def test_fused_rope_projection_and_backward(cuda, B, T, H, KVH):
    """cb_gemm_rope == gemm then rope; cb_attention_bwd_rope == attention bwd then inverse rope."""
    from paper_2507_05411_b200 import ops
    from paper_2507_05411_b200.layers import rope_tables

    hd = 128
    d, kvd = H * hd, KVH * hd
    g = torch.Generator().manual_seed(B * T)
    x = torch.randn(B * T, 256, generator=g).to(cuda, torch.bfloat16)
    w = (0.05 * torch.randn(256, d + 2 * kvd, generator=g)).to(cuda, torch.bfloat16)
    cs, sn = rope_tables(T, hd, 10000.0, cuda)
    fused = torch.empty(B * T, d + 2 * kvd, device=cuda, dtype=torch.bfloat16)
    ops.gemm_rope(x, w, fused, T, hd, d + kvd, cs, sn)
    plain = torch.empty_like(fused)
    ops.gemm(x, w, plain)
    ops.rope_(plain[:, :d], T, H, hd, cs, sn)
    ops.rope_(plain[:, d:d + kvd], T, KVH, hd, cs, sn)
    assert _rel(fused.float(), plain.float()) < 1e-2
    q, k, v = fused[:, :d], fused[:, d:d + kvd], fused[:, d + kvd:]
    scale = 1 / math.sqrt(hd)
    o, lse = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale)
    do = torch.randn(B * T, d, generator=g).to(cuda, torch.bfloat16)
    d1, d2 = torch.empty_like(fused), torch.empty_like(fused)
    ops.attention_bwd_rope(q, k, v, o, lse, do, d1[:, :d], d1[:, d:d + kvd], d1[:, d + kvd:], B, T, H, KVH, hd, scale,
                           cs, sn)
    ops.attention_bwd(q, k, v, o, lse, do, d2[:, :d], d2[:, d:d + kvd], d2[:, d + kvd:], B, T, H, KVH, hd, scale)
    ops.rope_(d2[:, :d], T, H, hd, cs, sn, inverse=True)
    ops.rope_(d2[:, d:d + kvd], T, KVH, hd, cs, sn, inverse=True)
    assert _rel(d1.float(), d2.float()) < 1e-2


@pytest.mark.parametrize("name", ["txf_moe", "txf_rope", "txf_d48_l3_relu"])
def test_device_init_bit_exact(cuda, name):
    """The device PCG64 initialiser reproduces the reference init_state bit for bit (as f32)."""
    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import TrainEngine, build_experiment, init_state, instantiate, root_key

    cfg = build_experiment(name)
    eng = TrainEngine(cfg, device=cuda, seed=3)
    ref = dict(O.leaves(init_state(instantiate(cfg), root_key(3))))
    got = dict(O.leaves(eng.state_numpy()))
    assert set(ref) == set(got)
    for k in ref:
        assert np.array_equal(got[k], ref[k].astype(np.float32).astype(np.float64)), k


def test_embedding_bwd_deterministic(cuda):
    from paper_2507_05411_b200 import ops

    V, dim, n = 500, 64, 4000
    g = torch.Generator().manual_seed(1)
    ids = torch.randint(0, V, (n,), generator=g).to(cuda)
    dout = torch.randn(n, dim, generator=g).to(cuda)
    outs = []
    for _ in range(2):
        off, perm = ops.sort_ids(ids, V)
        dt = torch.zeros(V, dim, device=cuda)
        ops.embedding_bwd(off, perm, dout, dt)
        outs.append(dt)
    assert torch.equal(outs[0], outs[1])
    ref = torch.zeros(V, dim, dtype=torch.float64, device=cuda).index_add_(0, ids, dout.double())
    assert _rel(outs[0], ref) < 1e-6
    # stability: perm is sorted by (id, position)
    p = perm.cpu().numpy()
    keys = ids.cpu().numpy()[p]
    assert np.all(np.diff(keys) >= 0)
    same = np.diff(keys) == 0
    assert np.all(np.diff(p)[same] > 0)


def test_moe_router_topk_bit_exact(cuda):
    """Identical router inputs give the reference's stable top-k assignment, ties included."""
    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import _lib, ops

    n, d, E, k = 4096, 64, 8, 2
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, d)).astype(np.float32)
    router = rng.standard_normal((d, E)).astype(np.float32) * 0.1
    router[:, 5] = router[:, 2]  # exact ties between experts 2 and 5
    xt, rt = torch.tensor(x, device=cuda), torch.tensor(router, device=cuda)
    idx = torch.empty(n, k, dtype=torch.int32, device=cuda)
    w = torch.empty(n, k, device=cuda)
    probs = torch.empty(n, E, device=cuda)
    _lib.call("cb_moe_route", n, d, E, k, xt.data_ptr(), d, 0, rt.data_ptr(), idx.data_ptr(), w.data_ptr(),
              probs.data_ptr(), ops.stream_ptr())
    p64 = torch.softmax(torch.tensor(x, dtype=torch.float64) @ torch.tensor(router, dtype=torch.float64), -1)
    ridx, rw, _, _ = O.route_tokens(p64, k)
    assert np.array_equal(idx.cpu().numpy(), ridx.numpy())
    assert np.allclose(w.cpu().numpy(), rw.numpy(), atol=1e-6)


@pytest.mark.parametrize("n,vocab", [(1024, 8), (1025, 8), (32768, 8), (50001, 33), (40000, 64), (3000, 500)])
def test_sort_ids_matches_stable_argsort(cuda, n, vocab):
    """cb_sort_ids (single CTA, or the chunked multi-CTA sort for <= 64 keys) = numpy's stable
    argsort: positions grouped by id in position order, offsets = the ids' exclusive counts."""
    from paper_2507_05411_b200 import ops

    rng = np.random.default_rng(n + vocab)
    ids = rng.integers(0, vocab, n)
    ids[: n // 3] = rng.integers(0, 2, n // 3)  # skewed like the init routing
    off, perm = ops.sort_ids(torch.tensor(ids, device=cuda), vocab)
    assert np.array_equal(perm.cpu().numpy()[:n], np.argsort(ids, kind="stable"))
    ref_off = np.concatenate([[0], np.cumsum(np.bincount(ids, minlength=vocab))])
    assert np.array_equal(off.cpu().numpy(), ref_off)


def test_moe_router_bf16_topk_bit_exact(cuda):
    """The bf16-input router (several tokens per warp, d = 2048 as in the MoE config): the
    reference's stable top-k on the f64 logits of the same bf16 inputs, ties and a ragged tail
    of tokens included."""
    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import _lib, ops

    n, d, E, k = 4099, 2048, 8, 2
    rng = np.random.default_rng(4)
    xb = torch.tensor(rng.standard_normal((n, d)), dtype=torch.float32).bfloat16()
    router = rng.standard_normal((d, E)).astype(np.float32) * 0.02
    router[:, 6] = router[:, 1]  # exact ties between experts 1 and 6
    xt, rt = xb.to(cuda), torch.tensor(router, device=cuda)
    idx = torch.empty(n, k, dtype=torch.int32, device=cuda)
    w = torch.empty(n, k, device=cuda)
    probs = torch.empty(n, E, device=cuda)
    _lib.call("cb_moe_route", n, d, E, k, xt.data_ptr(), d, 1, rt.data_ptr(), idx.data_ptr(), w.data_ptr(),
              probs.data_ptr(), ops.stream_ptr())
    p64 = torch.softmax(xb.double() @ torch.tensor(router, dtype=torch.float64), -1)
    ridx, rw, _, _ = O.route_tokens(p64, k)
    assert np.array_equal(idx.cpu().numpy(), ridx.numpy())
    assert np.allclose(w.cpu().numpy(), rw.numpy(), atol=1e-6)
    assert np.allclose(probs.cpu().numpy(), p64.numpy(), atol=1e-6)


@pytest.mark.parametrize("k,dy_bf16", [(2, True), (3, False), (1, True)])
def test_moe_combine_fwd_bwd(cuda, k, dy_bf16):
    """cb_moe_combine: out[t] = sum_j w[t,j] y[inv[t,j]] (slot order, layers.py:529-531) and its
    backward dy[inv[t,j]] = w[t,j] dout[t], dw[t,j] = dout[t] . y[inv[t,j]], against fp64 torch
    on rows scattered through a padded expert layout."""
    from paper_2507_05411_b200 import _lib, ops

    n, d = 3001, 512
    cap = n * k + 997  # padded expert layout: more rows than assignments
    g = torch.Generator().manual_seed(k)
    inv = torch.randperm(cap, generator=g)[: n * k].to(torch.int32)
    w = torch.rand(n, k, generator=g)
    y = torch.randn(cap, d, generator=g)
    dout = torch.randn(n, d, generator=g)
    Inv, W, Y, Dout = inv.to(cuda), w.to(cuda), y.to(cuda), dout.to(cuda)
    out = torch.empty(n, d, device=cuda)
    _lib.call("cb_moe_combine", n, d, k, Inv.data_ptr(), W.data_ptr(), Y.data_ptr(), d, 0, out.data_ptr(), d, 0,
              ops.stream_ptr())
    rows = y.double()[inv.long()].view(n, k, d)
    ref = (w.double().unsqueeze(-1) * rows).sum(1)
    assert _rel(out.cpu(), ref) < 1e-6
    # the residual-fused form: bit-identical to combine followed by the residual add
    res = torch.randn(n, d, generator=g).to(cuda)
    fused = torch.empty(n, d, device=cuda)
    _lib.call("cb_moe_combine_residual", n, d, k, Inv.data_ptr(), W.data_ptr(), Y.data_ptr(), d, res.data_ptr(), d,
              fused.data_ptr(), d, ops.stream_ptr())
    assert torch.equal(fused, out + res)
    dy = torch.zeros(cap, d, device=cuda, dtype=torch.bfloat16 if dy_bf16 else torch.float32)
    dw = torch.empty(n, k, device=cuda)
    _lib.call("cb_moe_combine_bwd", n, d, k, Inv.data_ptr(), W.data_ptr(), Y.data_ptr(), d, Dout.data_ptr(), d,
              dy.data_ptr(), d, ops.dt(dy), dw.data_ptr(), ops.stream_ptr())
    ref_dy = torch.zeros(cap, d, dtype=torch.float64)
    ref_dy[inv.long()] = (w.double().unsqueeze(-1) * dout.double().unsqueeze(1)).reshape(n * k, d)
    assert _rel(dy.cpu(), ref_dy) < (4e-3 if dy_bf16 else 1e-6)
    ref_dw = (rows * dout.double().unsqueeze(1)).sum(-1)
    assert _rel(dw.cpu(), ref_dw) < 1e-5


@pytest.mark.parametrize("E,bf16_x", [(8, True), (8, False), (4, True)])
def test_moe_router_bwd_gemms(cuda, E, bf16_x):
    """cb_moe_router_bwd_gemms: drouter += x^T dlogits (fixed token blocks, ordered reduction)
    and dx += dlogits router^T, against fp64 torch; bit-identical on a rerun."""
    from paper_2507_05411_b200 import _lib, ops

    n, d = 1000, 512
    g = torch.Generator().manual_seed(E)
    x = torch.randn(n, d, generator=g)
    if bf16_x:
        x = x.bfloat16()
    dlog = torch.randn(n, E, generator=g)
    router = torch.randn(d, E, generator=g) * 0.1
    dx0 = torch.randn(n, d, generator=g)
    X, Dl, R = x.to(cuda), dlog.to(cuda), router.to(cuda)
    outs = []
    for _ in range(2):
        dr = torch.full((d, E), 0.5, device=cuda)
        dx = dx0.to(cuda)
        ws = torch.empty(((n + 127) // 128) * d * E, device=cuda)
        _lib.call("cb_moe_router_bwd_gemms", n, d, E, X.data_ptr(), d, ops.dt(X), Dl.data_ptr(), R.data_ptr(),
                  dr.data_ptr(), dx.data_ptr(), d, ws.data_ptr(), ops.stream_ptr())
        outs.append((dr.cpu(), dx.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ref_dr = 0.5 + x.double().t() @ dlog.double()
    ref_dx = dx0.double() + dlog.double() @ router.double().t()
    assert _rel(outs[0][0], ref_dr) < 1e-5
    assert _rel(outs[0][1], ref_dx) < 1e-6


def test_adamw_kernel(cuda):
    from oracle import decoder_oracle as O
    from paper_2507_05411_b200 import ops

    n = 10007
    g = torch.Generator().manual_seed(5)
    p = torch.randn(n, generator=g)
    gr = torch.randn(n, generator=g) * 1e-2
    P, G = p.to(cuda), gr.to(cuda)
    M, Vv = torch.zeros(n, device=cuda), torch.zeros(n, device=cuda)
    bf = torch.empty(n, device=cuda, dtype=torch.bfloat16)
    pn, mn, vn = p.double().numpy(), np.zeros(n), np.zeros(n)
    for step in (1, 2, 3):
        ops.adamw(P, G, M, Vv, bf, 1e-3, 0.9, 0.999, 1e-8, 0.01, step)
        pn, mn, vn = O.adamw_update(pn, gr.double().numpy(), mn, vn, step, O.AdamW(1e-3, weight_decay=0.01))
    assert np.abs(P.cpu().double().numpy() - pn).max() < 1e-6
    assert torch.equal(bf, P.to(torch.bfloat16))


@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_sum_parts_in_order(cuda, nparts):
    """cb_sum_parts (local half of the FSDP reduce-scatter): scale * sum of the parts in list
    order, bit-identical to the same-order f32 sum."""
    import torch

    from paper_2507_05411_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(nparts)
    n = 1 << 20
    parts = [torch.randn(n, device="cuda", generator=g) for _ in range(nparts)]
    out = torch.empty(n, device="cuda")
    ops.sum_parts(parts, out, 1.0 / nparts)
    ref = parts[0].clone()
    for t in parts[1:]:
        ref += t
    ref *= 1.0 / nparts
    assert torch.equal(out, ref)
    with pytest.raises(Exception):
        ops.sum_parts(parts, torch.empty(n - 1, device="cuda"))


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_linear_with_bias_matches_reference(cuda, precision):
    """a15: Linear with bias (reference layers.py:130-170) through the module API on the GPU:
    forward equals the reference's invoke output and the gradients equal the reference's
    central finite differences (tests/golden: `linear`) and the f64 closed form."""
    import json
    import os

    from paper_2507_05411_b200 import default_config, instantiate, root_key
    from paper_2507_05411_b200.module import value_and_grad

    lg = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))["linear"]
    m = instantiate(default_config("Linear").set("input_dim", 16).set("output_dim", 24).set("bias", True))
    wdt = torch.float32 if precision == "f32" else torch.bfloat16
    x = np.array(lg["x"])
    W, b, dy = np.array(lg["weight"]), np.array(lg["bias"]), np.array(lg["dy"])
    state = {"weight": torch.tensor(W, dtype=wdt, device=cuda), "bias": torch.tensor(b, dtype=torch.float32, device=cuda)}
    grads = {"weight": torch.zeros(16, 24, device=cuda), "bias": torch.zeros(24, device=cuda)}
    xt = torch.tensor(x, dtype=torch.float32, device=cuda)
    y, _, dx = value_and_grad(m, state, grads, root_key(0), xt, seed_grad=torch.tensor(dy, dtype=torch.float32, device=cuda),
                              options={"precision": precision})
    torch.cuda.synchronize()
    tol = 1e-5 if precision == "f32" else 2e-2
    y = y.double().cpu().numpy()
    assert _rel(torch.tensor(y), torch.tensor(np.array(lg["y"]))) < tol
    gw, gb, gx = grads["weight"].double().cpu().numpy(), grads["bias"].double().cpu().numpy(), dx.double().cpu().numpy()
    x2, dy2 = x.reshape(-1, 16), dy.reshape(-1, 24)
    assert _rel(torch.tensor(gw), torch.tensor(x2.T @ dy2)) < tol
    assert _rel(torch.tensor(gb), torch.tensor(dy2.sum(0))) < tol
    assert _rel(torch.tensor(gx), torch.tensor(dy @ W.T)) < tol
    # the reference's central differences: elementwise in f32; in bf16 against the tensor's
    # rms (a single entry of a cancelling sum of bf16-rounded terms has no relative bound)
    fd = lg["fd"]
    for key, got, full in (("weight[3, 5]", gw[3, 5], gw), ("weight[15, 23]", gw[15, 23], gw), ("bias[7]", gb[7], gb),
                           ("x[1, 2, 9]", gx[1, 2, 9], gx)):
        scale = abs(fd[key]) if precision == "f32" else float(np.sqrt(np.mean(full ** 2)))
        assert abs(got - fd[key]) <= 1e-6 + tol * scale, key


@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_adamw_parts_is_sum_parts_then_adamw(cuda, nparts):
    """cb_adamw_parts (FSDP: the reduce-scatter's in-order sum fused into AdamW) is bit-identical
    to cb_sum_parts followed by cb_adamw, bf16 working copy included."""
    from paper_2507_05411_b200 import ops

    n = 4096 * 3
    g = torch.Generator(device="cpu").manual_seed(nparts)
    parts = [torch.randn(n, generator=g).to(cuda) * 1e-3 for _ in range(nparts)]
    p0, m0, v0 = (torch.randn(n, generator=g).to(cuda) for _ in range(3))
    v0 = v0.abs()
    outs = []
    for fused in (False, True):
        p, m, v = p0.clone(), m0.clone(), v0.clone()
        bf = torch.empty(n, device=cuda, dtype=torch.bfloat16)
        gs = torch.empty(n, device=cuda)
        if fused:
            ops.adamw_parts(parts, 1.0 / nparts, gs, p, m, v, bf, 1e-3, 0.9, 0.999, 1e-8, 0.01, 3)
        else:
            ops.sum_parts(parts, gs, 1.0 / nparts)
            ops.adamw(p, gs, m, v, bf, 1e-3, 0.9, 0.999, 1e-8, 0.01, 3)
        outs.append((p, m, v, bf, gs))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("B,T,H,KVH,rope", [(2, 256, 4, 4, False), (1, 384, 8, 2, True), (1, 1152, 4, 4, False),
                                           (2, 512, 4, 1, True)])
def test_attention_dq_gemm_matches_sweep(cuda, B, T, H, KVH, rope):
    """The dS path of the tcgen05 backward (dK/dV sweep storing dS^T + dQ as a GEMM over it,
    dq_gemm_k) against the two-sweep path on the same inputs: dK / dV bit-identical (the same
    sweep), dQ equal up to the rounding of dS to bf16 in one kernel or the other, and both
    against fp64 at the kernel tolerance; deterministic reruns."""
    from paper_2507_05411_b200 import ops
    from paper_2507_05411_b200.layers import rope_tables

    hd = 128
    g = torch.Generator().manual_seed(T * H + B)
    d, kvd = H * hd, KVH * hd
    qkv = torch.randn(B * T, d + 2 * kvd, generator=g).to(cuda, torch.bfloat16)
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    do = torch.randn(B * T, d, generator=g).to(cuda, torch.bfloat16)
    scale = 1 / math.sqrt(hd)
    cs, sn = rope_tables(T, hd, 10000.0, cuda)
    o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
    outs = []
    default = ops._DQ_GEMM
    for dq_gemm in (True, True, False):
        ops._DQ_GEMM = dq_gemm
        try:
            dqkv = torch.empty_like(qkv)
            args = (q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
            if rope:
                ops.attention_bwd_rope(*args, cs, sn, o_lo=o_lo)
            else:
                ops.attention_bwd(*args, o_lo=o_lo)
        finally:
            ops._DQ_GEMM = default
        outs.append(dqkv)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])  # deterministic
    gemm, sweep = outs[0], outs[2]
    assert torch.equal(gemm[:, d:], sweep[:, d:])  # dK, dV: the same sweep
    assert _rel(gemm[:, :d], sweep[:, :d]) < 2e-3
    if not rope:
        Q = q.double().view(B, T, H, hd).transpose(1, 2).requires_grad_(True)
        K = k.double().view(B, T, KVH, hd).transpose(1, 2)
        Vv = v.double().view(B, T, KVH, hd).transpose(1, 2)
        rep = H // KVH
        P = torch.softmax(Q @ K.repeat_interleave(rep, 1).transpose(-1, -2) * scale, -1)
        (P @ Vv.repeat_interleave(rep, 1)).backward(do.double().view(B, T, H, hd).transpose(1, 2))
        assert _rel(gemm[:, :d].view(B, T, H, hd).transpose(1, 2), Q.grad) < 5e-3


@pytest.mark.parametrize("B,T,H,KVH,rope", [(2, 256, 4, 4, False), (1, 512, 8, 2, True), (1, 1024, 4, 4, False),
                                           (2, 768, 4, 1, True)])
def test_attention_dq_pair_matches_sweep(cuda, B, T, H, KVH, rope):
    """The dQ and dK/dV sweeps on CTA pairs (cta_group::2 MMAs over 256 query / key rows,
    cb_attention_set_dq_pair / _dkdv_pair) against the single-CTA sweeps on the same inputs: the
    same MMAs in the same order, so dQ, dK and dV are bit-identical in every combination;
    deterministic reruns."""
    from paper_2507_05411_b200 import ops
    from paper_2507_05411_b200.layers import rope_tables

    hd = 128
    g = torch.Generator().manual_seed(T * H + B + 7)
    d, kvd = H * hd, KVH * hd
    qkv = torch.randn(B * T, d + 2 * kvd, generator=g).to(cuda, torch.bfloat16)
    q, k, v = qkv[:, :d], qkv[:, d:d + kvd], qkv[:, d + kvd:]
    do = torch.randn(B * T, d, generator=g).to(cuda, torch.bfloat16)
    scale = 1 / math.sqrt(hd)
    cs, sn = rope_tables(T, hd, 10000.0, cuda)
    o, lse, o_lo = ops.attention_fwd(q, k, v, B, T, H, KVH, hd, scale, want_lo=True)
    outs = []
    defaults = (ops._DQ_PAIR, ops._DKDV_PAIR)
    for dq_pair, dkdv_pair in ((1, 1), (1, 1), (0, 0), (1, 0), (0, 1)):
        ops.set_dq_pair(bool(dq_pair))
        ops.set_dkdv_pair(bool(dkdv_pair))
        try:
            dqkv = torch.empty_like(qkv)
            args = (q, k, v, o, lse, do, dqkv[:, :d], dqkv[:, d:d + kvd], dqkv[:, d + kvd:], B, T, H, KVH, hd, scale)
            if rope:
                ops.attention_bwd_rope(*args, cs, sn, o_lo=o_lo)
            else:
                ops.attention_bwd(*args, o_lo=o_lo)
        finally:
            ops.set_dq_pair(defaults[0])
            ops.set_dkdv_pair(defaults[1])
        outs.append(dqkv)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])  # deterministic
    for o_ in outs[2:]:  # the single-CTA sweeps' bits, with either sweep on pairs
        assert torch.equal(outs[0], o_)
