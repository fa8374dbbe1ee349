"""Pins the CPU oracle (oracle/decoder_oracle.py) to the reference's own outputs.

Fixtures in tests/golden/reference_goldens.json were produced by running the reference
(tests/golden/make_reference_goldens.py).  The oracle must reproduce the reference
step-0 loss of all 27 registry experiments and of the tiny bench config, the MoE
load-balance summaries, route_tokens / rope_apply known answers, and — for gradients,
which the reference cannot compute — central finite differences of the reference loss.
"""

import json
import os

import numpy as np
import pytest

from oracle import decoder_oracle as O
from paper_2507_05411_b200 import build_experiment, init_state, instantiate, root_key, synthetic_batch
from paper_2507_05411_b200.experiments import bench_tiny

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))


def _setup(name):
    m = instantiate(build_experiment(name))
    st = init_state(m, root_key(0))
    rec = GOLD["experiments"][name]
    toks = np.array(rec["tokens"], dtype=np.int64)
    return m, st, toks, rec


@pytest.mark.parametrize("name", sorted(GOLD["experiments"]))
def test_oracle_loss_matches_reference(name):
    m, st, toks, rec = _setup(name)
    spec = O.spec_from_config(m.config)
    summ = {}
    loss = float(O.forward_loss(O.to_torch(st), toks, spec, summ))
    assert abs(loss - rec["loss"]) <= 1e-12, (loss, rec["loss"])
    for k, v in rec["summaries"].items():
        if k == "loss":
            continue
        assert abs(summ[k] - v[0]) <= 1e-12, k


def test_synthetic_batch_matches_reference():
    for name in ("txf_base", "txf_moe"):
        rec = GOLD["experiments"][name]
        toks = synthetic_batch(0, 0, rec["batch_size"], rec["seq_len"])["tokens"]
        assert toks.tolist() == rec["tokens"]


def test_oracle_tiny_config_loss():
    m = instantiate(bench_tiny("f32"))
    st = init_state(m, root_key(0))
    toks = synthetic_batch(0, 0, 8, 256)["tokens"]
    loss = float(O.forward_loss(O.to_torch(st), toks, O.spec_from_config(m.config)))
    assert abs(loss - GOLD["tiny"]["loss"]) <= 1e-12


def test_oracle_two_steps_seed7_moe():
    m = instantiate(build_experiment("txf_moe"))
    st = init_state(m, root_key(7))
    spec = O.spec_from_config(m.config)
    for step, want in enumerate(GOLD["txf_moe_seed7_losses"]):
        toks = synthetic_batch(7, step, 4, 8)["tokens"]
        assert abs(float(O.forward_loss(O.to_torch(st), toks, spec)) - want) <= 1e-12


@pytest.mark.parametrize("name", sorted(GOLD["fd_grads"]))
def test_oracle_grads_match_reference_finite_differences(name):
    m, st, toks, _ = _setup(name)
    _, grads, _ = O.value_and_grad(st, toks, O.spec_from_config(m.config))
    for rec in GOLD["fd_grads"][name]:
        g = grads
        for seg in rec["path"].split("."):
            g = g[seg]
        got = g[tuple(rec["index"])]
        assert abs(got - rec["grad"]) <= 1e-7 + 1e-5 * abs(rec["grad"]), (rec, got)


def test_oracle_route_tokens_known_answer():
    import torch

    r = GOLD["route"]
    probs = torch.tensor(r["probs"], dtype=torch.float64)
    idx, w, disp, mp = O.route_tokens(probs, r["top_k"])
    assert idx.tolist() == r["indices"]
    assert np.allclose(w.numpy(), r["weights"], atol=1e-15, rtol=0)
    assert np.allclose(disp.numpy(), r["dispatch"], atol=0)
    assert np.allclose(mp.numpy(), r["mean_probs"], atol=1e-15)


def test_oracle_rope_known_answer():
    import torch

    r = GOLD["rope"]
    out = O.rope_apply(torch.tensor(r["x"], dtype=torch.float64), r["base"])
    assert np.allclose(out.numpy(), r["out"], atol=1e-14, rtol=0)


def test_oracle_adamw_first_step_sign():
    p = np.array([1.0, -2.0, 0.5])
    g = np.array([0.3, -1e-3, 0.0])
    newp, m, v = O.adamw_update(p, g, np.zeros(3), np.zeros(3), 1, O.AdamW(lr=1e-3))
    # step 1: update = g/(|g|+eps) -> ~sign(g)
    assert np.allclose(newp, p - 1e-3 * g / (np.abs(g) + 1e-8))
