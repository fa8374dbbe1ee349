"""End-to-end parity of the B200 training step against the CPU oracle (which is itself
pinned to the reference, tests/test_oracle_golden.py).

Contract (BASELINE.json north_star): loss, gradients and updated parameters within 1e-5
relative error in the fp32 mode and 2e-2 in the bf16 mode (relative L2 per tensor).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import decoder_oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def _leaves(t, pre=""):
    for k in sorted(t):
        v = t[k]
        p = f"{pre}.{k}" if pre else k
        if isinstance(v, dict):
            yield from _leaves(v, p)
        else:
            yield p, v


def fp32_oracle_errors(st, toks, spec, opt, forced=None):
    """Per-tensor error of a plain fp32 restatement (the oracle run in torch float32) against
    the f64 oracle, for gradients and step-1 updated parameters: what fp32 arithmetic itself
    permits.  Step-1 AdamW is ~lr*sign(g): gradient entries with |g| ~ eps=1e-8 turn ulp-level
    differences into lr-sized parameter changes, so on some shapes fp32 itself misses 1e-5 on
    the updated parameters (profiles/r02_f32_oracle_error.txt)."""
    _, g64, _ = O.value_and_grad(st, toks, spec, forced)
    _, g32, _ = O.value_and_grad(st, toks, spec, forced, dtype=torch.float32)
    g64, g32, st0 = dict(_leaves(g64)), dict(_leaves(g32)), dict(_leaves(st))

    def upd(g, k):
        return O.adamw_update(st0[k], g, 0 * st0[k], 0 * st0[k], 1, opt)[0]

    return ({k: _rel(g32[k], g64[k]) for k in g64}, {k: _rel(upd(g32[k], k), upd(g64[k], k)) for k in g64})


def _bf16_operand_grads(st, toks, spec, forced=None):
    with O.bf16_operands():
        lo, g, summ = O.value_and_grad(st, toks, spec, forced)
    return lo, dict(_leaves(g)), summ


def run_parity(cfg, precision, B, T, tol, seed=0, check_update=True, loose=None, exact_routing=False, report=None):
    """Loss, every gradient and every updated parameter vs the f64 oracle (relative L2).

    f32 mode: every gradient is held to 1e-5, or — only where a plain fp32 restatement itself
    misses 1e-5 (fp32_oracle_errors) — to 3x that fp32 error; updated parameters to 1e-5 on
    the well-conditioned entries (see below).
    bf16 mode: 2e-2; MoE layers are compared at the GPU's expert choices (bf16 router inputs
    flip ~0.5% of top-k choices against the f64 oracle), unless exact_routing.
    exact_routing: the GPU's top-k indices must equal the oracle's bit for bit.
    loose: {substring: tol} for tensors with a documented, larger bf16 error."""
    import torch

    from paper_2507_05411_b200 import TrainEngine, init_state, instantiate, root_key, set_dtype_policy, synthetic_batch

    cfg = set_dtype_policy(cfg, precision)
    eng = TrainEngine(cfg, device="cuda:0", seed=seed)
    V = eng.cfg.get("model.vocab_size")
    toks = synthetic_batch(seed, 0, B, T, V)["tokens"]
    eng.options["record_routing"] = True
    loss, col = eng.compute_grads(toks)
    loss = float(loss.item())
    routing = {}
    for key, vals in col.flat_summaries().items():
        if key.endswith("/route_indices"):
            routing[int(key.split("layer[")[1].split("]")[0])] = np.asarray(vals[0]).astype(np.int64)
    grads = dict(_leaves(eng.grads_numpy()))
    eng.apply_update()
    params = dict(_leaves(eng.state_numpy()))

    m = instantiate(cfg)
    st = init_state(m, root_key(seed))
    spec = O.spec_from_config(m.config)
    opt = O.AdamW(lr=eng.lr, beta1=eng.beta1, beta2=eng.beta2)
    forced = routing if (precision == "bf16" and not exact_routing) else None
    oracle_routing = {}
    lo, go, po, _, _, summ = O.train_step(st, toks, spec, opt, forced_routing=forced or None, routing=oracle_routing)
    if exact_routing:
        assert set(routing) == set(oracle_routing)
        for i in routing:
            assert np.array_equal(routing[i], oracle_routing[i]), f"layer {i}: top-k differs from the oracle"
    go, po = dict(_leaves(go)), dict(_leaves(po))
    assert set(grads) == set(go)
    assert abs(loss - lo) / abs(lo) < tol, (loss, lo)
    loose = loose or {}
    gbound = {k: tol for k in go}
    pbound = dict(gbound)
    if precision == "f32":
        e_g, e_p = fp32_oracle_errors(st, toks, spec, opt, forced)
        gbound = {k: max(tol, 3 * e_g[k]) for k in go}
        pbound = {k: max(tol, 3 * e_p[k]) for k in go}
    else:
        # bf16: where the oracle with only its GEMM operands rounded to bf16 (the least
        # rounding any bf16 path does) already errs by more than tol / 1.5, the tensor is held
        # to 1.5x that intrinsic error instead (ReLU kinks, sigmoid's common mode)
        _, gb, _ = _bf16_operand_grads(st, toks, spec, forced)
        gbound = {k: max(tol, 1.5 * _rel(gb[k], go[k])) for k in go}
    for k in go:
        for sub, v in loose.items():
            if sub in k:
                gbound[k], pbound[k] = max(gbound[k], v), max(pbound[k], v)
    gerr = {k: _rel(grads[k], go[k]) for k in go}
    perr = {k: _rel(params[k], po[k]) for k in po}
    if precision == "f32" and check_update:
        # Step-1 AdamW is p - lr * g / (|g| + eps): for |g| >= 100 eps the update's relative
        # sensitivity to a relative gradient error is <= eps / |g| <= 1e-2, so those entries are
        # held end to end to 1e-5 (relative L2 over them).  Entries with |g| < 100 eps are
        # ill-conditioned — an f32 gradient within the 1e-5 contract can still move such an
        # update by up to lr (the element dumps of profiles/r02_f32_param_conditioning.txt) — and
        # are held instead to AdamW applied in f64 to the GPU's own gradients (1e-6 relative).
        st0 = dict(_leaves(st))
        cond = {}
        for k in po:
            well = np.abs(go[k]) >= 100 * opt.eps
            own = O.adamw_update(st0[k], grads[k], 0 * st0[k], 0 * st0[k], 1, opt)[0]
            cond[k] = (_rel(params[k][well], po[k][well]) if well.any() else 0.0,
                       _rel(params[k][~well], own[~well]) if (~well).any() else 0.0, int((~well).sum()))
        bad = sorted((c[0], k) for k, c in cond.items() if c[0] >= tol)
        assert not bad, f"param (well-conditioned entries) {bad[-3:]}"
        bad = sorted((c[1], k) for k, c in cond.items() if c[1] >= 1e-6)
        assert not bad, f"param (ill-conditioned entries vs AdamW on the GPU's gradients) {bad[-3:]}"
        if report is not None:
            report["param_conditioned"] = cond
        check_update = False
    if report is not None:
        report.update({"loss": abs(loss - lo) / abs(lo), "grad": gerr, "param": perr,
                       "arrays": {"gpu_grad": grads, "oracle_grad": go, "gpu_param": params, "oracle_param": po}})
    bad = sorted((gerr[k], gbound[k], k) for k in go if gerr[k] >= gbound[k])
    assert not bad, f"grad {bad[-3:]}"
    if check_update:
        bad = sorted((perr[k], pbound[k], k) for k in po if perr[k] >= pbound[k])
        assert not bad, f"param {bad[-3:]}"
    flat = col.flat_summaries()
    for k, v in summ.items():
        assert abs(flat[k][0] - v) <= max(tol, 1e-6) * abs(v), (k, flat[k], v)
    return loss, lo


@pytest.mark.parametrize("name", ["txf_base", "txf_rope", "txf_d16_l1_relu", "txf_d64_l3_swiglu", "txf_moe"])
def test_registry_step_f32(cuda, name):
    from paper_2507_05411_b200 import build_experiment

    run_parity(build_experiment(name), "f32", 4, 8, 1e-5)


def test_tiny_bench_config_f32(cuda):
    from paper_2507_05411_b200.experiments import bench_tiny

    loss, lo = run_parity(bench_tiny("f32"), "f32", 8, 256, 1e-5)
    assert abs(lo - GOLD["tiny"]["loss"]) < 1e-12


@pytest.mark.parametrize("name", ["txf_rope", "txf_moe", "txf_base"])
def test_registry_step_bf16(cuda, name):
    from paper_2507_05411_b200 import build_experiment

    run_parity(build_experiment(name), "bf16", 4, 8, 2e-2)


def test_bf16_relu_d32_characterization(cuda):
    """Known bf16 limit, shown to be intrinsic to bf16 operands: on the d=32 ReLU stack with 32
    tokens a few tensors sit above 2e-2 (pre-activations near ReLU's kink change sign when the
    GEMM operands are rounded to bf16).  The oracle with ONLY its GEMM operands rounded to bf16
    (O.bf16_operands: the least rounding any bf16 path does) has the same error (~7% on
    feed_forward.w1), so every tensor is held to 2e-2 or to 2x that bf16-operand oracle's own
    error, whichever is larger."""
    from paper_2507_05411_b200 import build_experiment, init_state, instantiate, root_key, synthetic_batch

    cfg = build_experiment("txf_d32_l2_relu")
    m = instantiate(cfg)
    st = init_state(m, root_key(0))
    spec = O.spec_from_config(m.config)
    toks = synthetic_batch(0, 0, 4, 8, m.config.get("model.vocab_size"))["tokens"]
    _, g64, _ = O.value_and_grad(st, toks, spec)
    with O.bf16_operands():
        _, gb, _ = O.value_and_grad(st, toks, spec)
    g64, gb = dict(_leaves(g64)), dict(_leaves(gb))
    emu = {k: _rel(gb[k], g64[k]) for k in g64}
    assert max(emu.values()) > 2e-2  # the limit is the operand rounding itself
    loose = {k: 2 * e for k, e in emu.items() if 2 * e > 2e-2}
    rep = {}
    run_parity(cfg, "bf16", 4, 8, 2e-2, loose=loose, report=rep)


def _mid(hd: int, kind="FeedForward"):
    """An aligned shape that exercises the fast engines: tcgen05 GEMMs + flash attention."""
    from paper_2507_05411_b200.experiments import transformer_trainer

    heads = 256 // hd
    cfg = transformer_trainer(256, 2, ("linear", "silu"), pos_kind="RoPE", heads=heads, vocab=512,
                              feed_forward_kind=kind, num_experts=4, top_k=2)
    for i in range(2):
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    return cfg


@pytest.mark.parametrize("hd", [64, 128])
def test_fast_path_step_bf16(cuda, hd):
    run_parity(_mid(hd), "bf16", 4, 256, 2e-2)


@pytest.fixture(params=[False, True], ids=["simt_gemm", "tcgen05_bf16x6"])
def f32_tc(request):
    """The f32 parity mode's GEMMs on the SIMT engine, or on the tcgen05 engine as six bf16
    products of three-term operand splits (ops.set_f32_tc)."""
    from paper_2507_05411_b200 import ops

    ops.set_f32_tc(request.param)
    yield request.param
    ops.set_f32_tc(False)


@pytest.mark.parametrize("hd", [64, 128])
def test_fast_path_shape_f32(cuda, hd, f32_tc):
    run_parity(_mid(hd), "f32", 2, 128, 1e-5)


def test_fast_path_moe_bf16(cuda):
    """bf16 router *inputs* flip the top-2 choice of ~0.5% of tokens relative to the f64
    oracle — a discontinuity, not an arithmetic error.  The bf16 parity run
    therefore records the GPU's expert choices (debug summary ``route_indices``) and the
    oracle evaluates the step at those choices (the reference's own forced-routing oracle,
    tests/test_layers.py:352-359); every tensor is then held to 2e-2.  Bit-exact routing on
    identical inputs is tested in test_kernels_gpu.py::test_moe_router_topk_bit_exact."""
    run_parity(_mid(128, "MoE"), "bf16", 4, 128, 2e-2)


def test_moe_f32_unforced_routing_t256(cuda, f32_tc):
    """f32 MoE at T=256 with the GPU's OWN routing: the top-2 expert choices of every token equal
    the f64 oracle's bit for bit (reference route_tokens, layers.py:432-443: stable argsort,
    ties -> lowest id), and every tensor is held to the f32 contract."""
    run_parity(_mid(128, "MoE"), "f32", 2, 256, 1e-5, exact_routing=True)


def _gqa(hd: int, heads: int, kv_heads: int, layers: int = 2):
    """GroupedQueryAttention (the 70B-layer kind) in a small trainer; d = heads * hd."""
    from paper_2507_05411_b200 import default_config
    from paper_2507_05411_b200.experiments import transformer_trainer

    d = heads * hd
    cfg = transformer_trainer(d, layers, ("linear", "silu"), pos_kind="RoPE", heads=heads, vocab=512)
    for i in range(layers):
        p = f"model.decoder.transformer.layer[{i}]"
        cfg = (cfg.set(f"{p}.self_attention", default_config("GroupedQueryAttention").set("num_kv_heads", kv_heads)
                       .set("num_heads", heads).set("pos_emb", default_config("RoPE")))
               .set(f"{p}.feed_forward.hidden_dim", 768))
    return cfg


@pytest.mark.parametrize("hd,heads,kv", [(64, 4, 1), (64, 8, 2), (128, 4, 1), (128, 4, 2), (128, 8, 2)])
@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_gqa_engine_step(cuda, hd, heads, kv, precision, f32_tc):
    if f32_tc and precision == "bf16":
        pytest.skip("the f32 GEMM switch does not apply to bf16")
    """N1: the GQA kind through TrainEngine against the oracle (which repeats each kv head over
    its group of query heads, oracle/decoder_oracle.py attention)."""
    T = 128 if precision == "f32" else 256
    run_parity(_gqa(hd, heads, kv), precision, 2, T, 1e-5 if precision == "f32" else 2e-2)


def test_gqa_with_kv_equal_heads_is_the_reference_attention(cuda):
    """GroupedQueryAttention with num_kv_heads == num_heads is exactly the reference's Attention
    (layers.py:282-348): same parameters (same init keys), bit-identical loss and gradients."""
    from paper_2507_05411_b200 import TrainEngine, synthetic_batch
    from paper_2507_05411_b200.experiments import transformer_trainer

    toks = synthetic_batch(0, 0, 2, 128, 512)["tokens"]
    mha = transformer_trainer(256, 2, ("linear", "silu"), pos_kind="RoPE", heads=2, vocab=512)
    for i in range(2):
        mha = mha.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    outs = []
    for cfg in (mha, _gqa(128, 2, 2)):
        eng = TrainEngine(cfg, device="cuda:0")
        loss, _ = eng.compute_grads(toks)
        outs.append((float(loss.item()), dict(_leaves(eng.grads_numpy()))))
    assert outs[0][0] == outs[1][0]
    assert set(outs[0][1]) == set(outs[1][1])
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k


@pytest.mark.parametrize("act", ["sigmoid", "tanh", "linear", ("tanh", "sigmoid"), ("relu", "linear")])
@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_activation_table_step(cuda, act, precision):
    """a11: every entry of the activation table (layers.py:55-77), plain and gated, end to end
    against the oracle."""
    from paper_2507_05411_b200.experiments import transformer_trainer

    cfg = transformer_trainer(256, 2, act, pos_kind="RoPE", heads=2, vocab=512)
    for i in range(2):
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    run_parity(cfg, precision, 2, 128, 1e-5 if precision == "f32" else 2e-2)


@pytest.mark.parametrize("policy", ["recompute_all", "save_qkvo_flash", "offload_dots"])
@pytest.mark.parametrize("precision", ["f32", "bf16"])
@pytest.mark.parametrize("kind", ["FeedForward", "MoE"])
def test_remat_policy_against_oracle(cuda, policy, precision, kind):
    """f2: a rematerialised step against the oracle directly (not only against no-remat)."""
    from paper_2507_05411_b200.remat import POLICY_ALIASES

    cfg = _mid(128, kind)
    for i in range(2):
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].remat_policy", POLICY_ALIASES[policy])
    run_parity(cfg, precision, 2, 128 if precision == "f32" else 256, 1e-5 if precision == "f32" else 2e-2)


def test_tiny_bench_config_bf16(cuda):
    from paper_2507_05411_b200.experiments import bench_tiny

    run_parity(bench_tiny("bf16"), "bf16", 8, 256, 2e-2)


def test_forward_loss_matches_reference_invoke(cuda):
    """engine.loss == the reference's invoke() loss for every registry experiment (f32 mode)."""
    from paper_2507_05411_b200 import TrainEngine, build_experiment

    for name, rec in sorted(GOLD["experiments"].items()):
        eng = TrainEngine(build_experiment(name), device="cuda:0")
        got = eng.loss(np.array(rec["tokens"], dtype=np.int64))
        assert abs(got - rec["loss"]) / rec["loss"] < 1e-5, (name, got, rec["loss"])


@pytest.mark.parametrize("policy", ["recompute_all", "save_qkvo_flash", "offload_dots",
                                    {"hidden": "recompute", "context": "offload"}, {"q_proj": "recompute"}])
def test_remat_policies_are_exact(cuda, policy):
    """Rematerialised tags rerun the same deterministic kernels and offloaded ones come back
    byte for byte: gradients are bit-identical to the save-everything step."""
    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
    from paper_2507_05411_b200.remat import POLICY_ALIASES

    base = set_dtype_policy(_mid(128), "bf16")
    remat = base
    for i in range(2):
        remat = remat.set(f"model.decoder.transformer.layer[{i}].remat_policy",
                          POLICY_ALIASES[policy] if isinstance(policy, str) else policy)
    toks = synthetic_batch(0, 0, 2, 256, 512)["tokens"]
    outs, fwd_bytes = [], []
    for cfg in (base, remat):
        eng = TrainEngine(cfg, device="cuda:0")
        loss, _ = eng.compute_grads(toks)
        outs.append((float(loss.item()), dict(_leaves(eng.grads_numpy()))))
        fwd_bytes.append(eng.last_forward_bytes)
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k
    # the forward leaves less on the device for the backward
    assert fwd_bytes[1] < fwd_bytes[0], fwd_bytes


def test_wgrad_stream_is_exact(cuda, monkeypatch):
    """Weight gradients on the side stream (CB_WGRAD_STREAM, layers._wgrad) run the same
    deterministic GEMMs: two AdamW steps give bit-identical losses and parameters."""
    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch

    cfg = set_dtype_policy(_mid(128), "bf16")
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("CB_WGRAD_STREAM", flag)
        eng = TrainEngine(cfg, device="cuda:0")
        assert (eng._wgrad_stream is not None) == (flag == "1")
        losses = [float(eng.step(synthetic_batch(0, s, 4, 256, 512)["tokens"])[0].item()) for s in range(2)]
        outs.append((losses, dict(_leaves(eng.state_numpy()))))
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k


def test_two_steps_train(cuda):
    """Multi-step: oracle and engine stay within tolerance after 3 AdamW steps (f32)."""
    from paper_2507_05411_b200 import TrainEngine, build_experiment, init_state, instantiate, root_key, synthetic_batch

    cfg = build_experiment("txf_rope")
    eng = TrainEngine(cfg, device="cuda:0")
    m = instantiate(cfg)
    st = init_state(m, root_key(0))
    spec = O.spec_from_config(m.config)
    mm = vv = None
    for step in range(3):
        toks = synthetic_batch(0, step, 4, 8)["tokens"]
        loss, _ = eng.step(toks)
        lo, _, st, mm, vv, _ = O.train_step(st, toks, spec, O.AdamW(lr=1e-3), mm, vv, step + 1)
        assert abs(float(loss.item()) - lo) / lo < 1e-5
    mine = dict(_leaves(eng.state_numpy()))
    for k, v in _leaves(st):
        assert _rel(mine[k], v) < 1e-5, k


def test_functional_train_step_api(cuda):
    """train_step / forward_loss on the reference's state trees (SURVEY §8(b) step entry):
    fresh state in, (loss, summaries, new_state, new_opt_state, grads) out, inputs untouched,
    two chained steps against the oracle; forward_loss equals the reference invoke loss."""
    from paper_2507_05411_b200 import (build_experiment, child_key, forward_loss, init_state, instantiate, root_key,
                                       synthetic_batch, train_step)

    m = instantiate(build_experiment("txf_moe"))
    st = st0 = init_state(m, root_key(0))
    before = {k: v.copy() for k, v in _leaves(st0)}
    spec = O.spec_from_config(m.config)
    opt = None
    ost, mm, vv = st, None, None
    for step in range(2):
        toks = synthetic_batch(0, step, 4, 8)["tokens"]
        key = child_key(root_key(0), "step", step)
        loss, summ, new_st, opt, grads = train_step(m, st, opt, key, {"tokens": toks}, return_grads=True)
        lo, go, ost, mm, vv, osum = O.train_step(ost, toks, spec, O.AdamW(lr=1e-3), mm, vv, step + 1)
        assert abs(loss - lo) / lo < 1e-5
        for k, v in _leaves(go):
            assert _rel(dict(_leaves(grads))[k], v) < 1e-5, k
        for k, ref in osum.items():
            assert abs(summ[k][0] - ref) / abs(ref) < 1e-5, k
        assert opt["step"] == step + 1
        mine = dict(_leaves(new_st))
        for k, v in _leaves(ost):
            assert _rel(mine[k], v) < 1e-5, k
        for k, v in _leaves(mm):
            assert _rel(dict(_leaves(opt["m"]))[k], v) < 1e-5, k
        st = new_st
    for k, v in _leaves(st0):
        assert np.array_equal(before[k], v)  # the caller's arrays were not mutated
    rec = GOLD["experiments"]["txf_moe"]
    loss, col = forward_loss(m, init_state(m, root_key(0)), child_key(root_key(0), "step", 0),
                             {"tokens": np.array(rec["tokens"], dtype=np.int64)})
    assert abs(loss - rec["loss"]) / rec["loss"] < 1e-5


def test_checkpoint_resume_is_bit_exact(cuda, tmp_path):
    """save -> fresh engine -> load -> the next step equals the uninterrupted run exactly;
    retention keeps the newest checkpoints only."""
    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
    from paper_2507_05411_b200.checkpoint import GcPolicy, list_steps, load_checkpoint, save_checkpoint

    cfg = set_dtype_policy(_mid(128), "bf16")
    toks = [synthetic_batch(0, s, 2, 256, 512)["tokens"] for s in range(4)]
    a = TrainEngine(cfg, device="cuda:0")
    root = str(tmp_path / "ck")
    for s in range(3):
        a.step(toks[s])
        save_checkpoint(a, root, gc=GcPolicy(keep_last_n=2))
    assert list_steps(root) == [2, 3]
    la, _ = a.step(toks[3])
    b = TrainEngine(cfg, device="cuda:0", init=False)
    assert load_checkpoint(b, root) == 3
    lb, _ = b.step(toks[3])
    assert float(la.item()) == float(lb.item())
    sa, sb = dict(_leaves(a.state_numpy())), dict(_leaves(b.state_numpy()))
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k


def test_full_size_1b_step_properties(cuda):
    """BASELINE configs[1] at full size (16 layers, d=2048, seq 4096, 8 sequences) — too large
    for the CPU oracle, so size-independent properties: two engines from the same init and
    batch produce bit-identical losses and updated parameters (deterministic reductions, no
    atomics); the training step's loss equals the forward-only loss; the initial loss is near
    ln(V) (reference init gives near-uniform predictions); three steps on one batch lower it
    (measured 10.54 -> 10.45)."""
    import math

    import torch

    from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, synthetic_batch

    cfg = BENCH_CONFIGS["1b"](dtype="bf16")
    toks = synthetic_batch(0, 0, 8, 4096, 32000)["tokens"]
    runs = []
    for _ in range(2):
        eng = TrainEngine(cfg, device=cuda)
        fwd = float(eng.loss(toks))
        losses = [float(eng.step(toks)[0].item()) for _ in range(3)]
        sums = [float(rec["master"].double().sum().item()) for rec in eng.bufs]
        runs.append((fwd, losses, sums))
        del eng
        torch.cuda.empty_cache()
    assert runs[0] == runs[1]
    fwd, losses, _ = runs[0]
    assert abs(losses[0] - fwd) / fwd < 2e-2
    assert abs(losses[0] - math.log(32000)) < 1.0
    assert losses[2] < losses[0] - 0.05


@pytest.mark.parametrize("B,T", [(3, 200), (1, 136), (5, 72)])
def test_ragged_fast_path_bf16(cuda, B, T):
    """Ragged shapes through the fast engines end to end: token counts that are not multiples
    of the 256-row GEMM tiles or the 128-row attention tiles (masked key tiles, rows crossing
    sequence boundaries, a single partial tile)."""
    run_parity(_mid(128), "bf16", B, T, 2e-2)


def test_north_star_layer_shape_bf16(cuda):
    """Oracle parity at the north-star width: one Llama2-7B-shaped layer (d=4096, 32 heads of
    128, SwiGLU ffn 11008, V=32000, tied head) through the bench's bf16 engines — the CTA-pair
    GEMMs at their full N / K, the tcgen05 attention over two key tiles — against the f64
    oracle (loss, every gradient, every updated parameter at 2e-2; ~25 s and ~20 GB of host
    memory for the oracle)."""
    from paper_2507_05411_b200 import BENCH_CONFIGS

    run_parity(BENCH_CONFIGS["7b"](batch=1, seq=256, layers=1), "bf16", 1, 256, 2e-2)


def test_70b_head_geometry_bf16(cuda):
    """Oracle parity at the 70B layer's attention geometry: d=8192, GQA 64 query / 8 kv heads of
    128 (the FFN narrowed to 2048 and V to 512 so the f64 oracle stays small) — the GQA
    attention kernels and the d=8192 projections against the oracle at 2e-2."""
    from paper_2507_05411_b200.experiments import _llama_trainer

    run_parity(_llama_trainer(8192, 1, 64, 2048, 512, 1, 256, kv_heads=8), "bf16", 1, 256, 2e-2)


@pytest.mark.parametrize("name,B", [("7b", 3), ("70b_layer", 2), ("moe", 4)])
def test_full_size_step_properties(cuda, name, B):
    """BASELINE configs[2..4] at full size (too large for the CPU oracle): a second engine from
    the same init gives a bit-identical loss and master weights after two steps (deterministic
    reductions everywhere, grouped MoE GEMMs included); the first loss is near ln(V) (the
    reference init predicts near-uniformly) and one update lowers the loss on its batch (at the
    reference's lr 1e-3 later steps on one batch oscillate at this scale: 7B at 3 sequences
    10.54 -> 10.25 -> 10.66 -> 10.49 -> 9.52, identical with and without the one-GPU gradient
    ring, profiles/r02_loss_traj.log)."""
    import math

    from paper_2507_05411_b200 import BENCH_CONFIGS, TrainEngine, synthetic_batch

    import gc

    cfg = BENCH_CONFIGS[name](batch=B, dtype="bf16")
    toks = synthetic_batch(0, 0, B, 4096, 32000)["tokens"]
    runs = []
    for _ in range(2):
        gc.collect()
        torch.cuda.empty_cache()
        eng = TrainEngine(cfg, device=cuda)
        losses = [float(eng.step(toks)[0].item()) for _ in range(3)]
        sums = [float(rec["master"].double().sum().item()) for rec in eng.bufs]
        runs.append((losses, sums))
        del eng
        torch.cuda.empty_cache()
    assert runs[0] == runs[1]
    losses = runs[0][0]
    assert abs(losses[0] - math.log(32000)) < 1.5
    assert losses[1] < losses[0]


def test_single_gpu_grad_ring_is_exact(cuda, monkeypatch):
    """The one-GPU two-slot gradient ring (CB_GRAD_RING; automatic above CB_GRAD_RING_MIN_GB, e.g.
    the 7B step) gives bit-identical losses and parameters to full per-layer gradient buffers,
    with less engine state; reading gradients after such a step raises instead of returning
    stale values."""
    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
    from paper_2507_05411_b200.errors import ComposerError

    from paper_2507_05411_b200.experiments import transformer_trainer

    cfg = transformer_trainer(256, 5, ("linear", "silu"), pos_kind="RoPE", heads=2, vocab=512)
    for i in range(5):  # five layers: both ring slots are reused within a step
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    cfg = set_dtype_policy(cfg, "bf16")
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("CB_GRAD_RING", flag)
        eng = TrainEngine(cfg, device="cuda:0")
        assert eng._grad_ring == (flag == "1")
        losses = [float(eng.step(synthetic_batch(0, s, 4, 256, 512)["tokens"])[0].item()) for s in range(3)]
        outs.append((losses, dict(_leaves(eng.state_numpy())), eng.state_bytes()))
        if flag == "1":
            with pytest.raises(ComposerError):
                eng.grads_numpy()
    assert outs[0][0] == outs[1][0]
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k]), k
    assert outs[1][2] < outs[0][2]


@pytest.mark.parametrize("kind", ["swiglu_5l", "gqa"])
def test_fused_adamw_in_wgrad_gemm_is_exact(cuda, monkeypatch, kind):
    """One-GPU step with AdamW fused into the weight-gradient GEMMs' epilogues (cb_gemm_adamw,
    opt-in CB_FUSED_ADAMW=1), and with the weight-gradient GEMMs overwriting instead of
    accumulating into cleared buffers (CB_WGRAD_OVERWRITE, default on), against the separate
    AdamW kernel on cleared, accumulated gradients: bit-identical losses, parameters and AdamW
    moments over three steps, with and without the gradient ring; every layer bucket of these
    dense configs takes the fused / overwrite path."""
    from paper_2507_05411_b200 import TrainEngine, set_dtype_policy, synthetic_batch
    from paper_2507_05411_b200.experiments import _llama_trainer, transformer_trainer

    if kind == "gqa":
        cfg = _llama_trainer(256, 2, 4, 768, 512, 4, 256, kv_heads=2)
    else:
        cfg = transformer_trainer(256, 5, ("linear", "silu"), pos_kind="RoPE", heads=2, vocab=512)
        for i in range(5):
            cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    cfg = set_dtype_policy(cfg, "bf16")
    outs = []
    for fused, ring, ow in (("0", "0", "0"), ("0", "0", "1"), ("0", "1", "1"), ("1", "0", "1"), ("1", "1", "1")):
        monkeypatch.setenv("CB_FUSED_ADAMW", fused)
        monkeypatch.setenv("CB_GRAD_RING", ring)
        monkeypatch.setenv("CB_WGRAD_OVERWRITE", ow)
        eng = TrainEngine(cfg, device="cuda:0")
        nf = len(eng.fused_update_buckets())
        assert nf == (0 if fused == "0" else len(eng.layer_order))
        losses = [float(eng.step(synthetic_batch(0, s, 4, 256, 512)["tokens"])[0].item()) for s in range(3)]
        opt = eng.opt_state_numpy()
        outs.append((losses, dict(_leaves(eng.state_numpy())), dict(_leaves(opt["m"])), dict(_leaves(opt["v"]))))
        del eng
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        for j in (1, 2, 3):
            for k in outs[0][j]:
                assert np.array_equal(o[j][k], outs[0][j][k]), k
