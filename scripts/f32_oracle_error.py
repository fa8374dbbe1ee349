"""fp32 restatement vs the f64 oracle (gradients and step-1 AdamW updates) on the f32 parity-test
shapes: what plain fp32 arithmetic reaches (profiles/r02_f32_param_conditioning.txt)."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from oracle import decoder_oracle as O
from paper_2507_05411_b200 import build_experiment, init_state, instantiate, root_key, set_dtype_policy, synthetic_batch
from paper_2507_05411_b200.experiments import bench_tiny, transformer_trainer

def mid(hd, kind="FeedForward"):
    heads = 256 // hd
    cfg = transformer_trainer(256, 2, ("linear", "silu"), pos_kind="RoPE", heads=heads, vocab=512, feed_forward_kind=kind, num_experts=4, top_k=2)
    for i in range(2):
        cfg = cfg.set(f"model.decoder.transformer.layer[{i}].feed_forward.hidden_dim", 768)
    return cfg

def run(dt, st, toks, spec):
    O.F64 = dt
    def tt(tree):
        if isinstance(tree, dict): return {k: tt(v) for k, v in tree.items()}
        return torch.tensor(np.asarray(tree), dtype=dt).requires_grad_(True)
    p = tt(st)
    loss = O.forward_loss(p, toks, spec, {})
    loss.backward()
    g = {k: v.grad.double().numpy() for k, v in O.leaves(p)}
    return float(loss), g

cases = [(build_experiment(n), 4, 8, n) for n in ["txf_base","txf_rope","txf_d16_l1_relu","txf_d64_l3_swiglu","txf_moe"]]
cases += [(bench_tiny("f32"), 8, 256, "tiny"), (mid(64), 2, 128, "mid64"), (mid(128), 2, 128, "mid128")]
opt = O.AdamW(lr=1e-3)
for cfg, B, T, name in cases:
    m = instantiate(set_dtype_policy(cfg, "f32")); st = init_state(m, root_key(0)); spec = O.spec_from_config(m.config)
    toks = synthetic_batch(0, 0, B, T, m.config.get("model.vocab_size"))["tokens"]
    l64, g64 = run(torch.float64, st, toks, spec)
    l32, g32 = run(torch.float32, st, toks, spec)
    st0 = dict(O.leaves(st))
    worst_g = max((np.linalg.norm(g32[k]-g64[k])/max(np.linalg.norm(g64[k]),1e-30), k) for k in g64)
    def upd(g, k): return O.adamw_update(st0[k], g, 0*st0[k], 0*st0[k], 1, opt)[0]
    # f32 params: round master to f32 then update in f32-ish
    worst_p = max((np.linalg.norm(upd(g32[k],k)-upd(g64[k],k))/np.linalg.norm(upd(g64[k],k)), k) for k in g64)
    print(f"{name:22s} loss {abs(l32-l64)/l64:.1e} grad {worst_g[0]:.2e} {worst_g[1]} param {worst_p[0]:.2e} {worst_p[1]}")
