"""Per-tensor parity table (GPU vs the f64 oracle, next to what a plain fp32 restatement and a
bf16-operand restatement of the oracle reach) for named cases; used to document tolerances.

    python scripts/parity_report.py CASE [CASE ...]      (cases: see CASES)
"""
import json
import os
import sys
import traceback

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import test_step_gpu as TS  # noqa: E402
from oracle import decoder_oracle as O  # noqa: E402


def _act(act):
    from paper_2507_05411_b200.experiments import transformer_trainer

    cfg = transformer_trainer(256, 2, act, pos_kind="RoPE", heads=2, vocab=512)
    for i in range(2):
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    return cfg


CASES = {
    "mid64_f32": (lambda: TS._mid(64), "f32", 2, 128),
    "mid128_f32": (lambda: TS._mid(128), "f32", 2, 128),
    "moe_f32_t256": (lambda: TS._mid(128, "MoE"), "f32", 2, 256),
    "linear_f32": (lambda: _act("linear"), "f32", 2, 128),
    "sigmoid_f32": (lambda: _act("sigmoid"), "f32", 2, 128),
    "sigmoid_bf16": (lambda: _act("sigmoid"), "bf16", 2, 128),
    "tanh_sigmoid_bf16": (lambda: _act(("tanh", "sigmoid")), "bf16", 2, 128),
    "tanh_bf16": (lambda: _act("tanh"), "bf16", 2, 128),
    "swiglu_bf16": (lambda: _act(("linear", "silu")), "bf16", 2, 128),
    "relu_d32_bf16": (lambda: __import__("paper_2507_05411_b200").build_experiment("txf_d32_l2_relu"), "bf16", 4, 8),
}


def yardsticks(cfg, B, T, precision):
    from paper_2507_05411_b200 import init_state, instantiate, root_key, set_dtype_policy, synthetic_batch

    m = instantiate(set_dtype_policy(cfg, precision))
    st = init_state(m, root_key(0))
    spec = O.spec_from_config(m.config)
    toks = synthetic_batch(0, 0, B, T, m.config.get("model.vocab_size"))["tokens"]
    _, g64, _ = O.value_and_grad(st, toks, spec)
    _, g32, _ = O.value_and_grad(st, toks, spec, dtype=torch.float32)
    with O.bf16_operands():
        _, gb, _ = O.value_and_grad(st, toks, spec)
    g64, g32, gb = dict(O.leaves(g64)), dict(O.leaves(g32)), dict(O.leaves(gb))
    return {k: TS._rel(g32[k], g64[k]) for k in g64}, {k: TS._rel(gb[k], g64[k]) for k in g64}


def element_dump(cfg, B, T, precision, key, rep, top=8):
    """The entries of tensor `key` whose updated values differ most from the oracle's."""
    g = rep["arrays"]
    d = np.abs(g["gpu_param"][key] - g["oracle_param"][key]).ravel()
    idx = np.argsort(-d)[:top]
    return [{"i": int(i), "dparam": float(d[i]), "g_oracle": float(g["oracle_grad"][key].ravel()[i]),
             "g_gpu": float(g["gpu_grad"][key].ravel()[i])} for i in idx]


def main():
    out = {}
    for name in sys.argv[1:] or list(CASES):
        mk, prec, B, T = CASES[name]
        rep = {}
        err = None
        try:
            TS.run_parity(mk(), prec, B, T, 1e-5 if prec == "f32" else 2e-2, report=rep, exact_routing="moe" in name)
        except AssertionError as e:
            err = str(e)[:400]
        except Exception:  # noqa: BLE001
            err = traceback.format_exc()[-800:]
        e32, ebf = yardsticks(mk(), B, T, prec)
        rows = []
        for k in sorted(rep.get("grad", {}), key=lambda k: -rep["grad"][k])[:8]:
            rows.append({"tensor": k, "gpu_grad": rep["grad"][k], "gpu_param": rep["param"][k], "fp32_grad": e32[k],
                         "bf16_operand_grad": ebf[k]})
        if rep.get("param"):
            wk = max(rep["param"], key=lambda k: rep["param"][k])
            out_el = element_dump(mk(), B, T, prec, wk, rep)
        else:
            out_el = None
        out[name] = {"precision": prec, "B": B, "T": T, "loss_rel": rep.get("loss"), "assert": err,
                     "worst_param_elements": out_el,
                     "worst_param": max(rep.get("param", {0: 0}).values()), "rows": rows}
        print(json.dumps({name: out[name]}), flush=True)


if __name__ == "__main__":
    main()
