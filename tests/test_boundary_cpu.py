"""C-ABI boundary and host-API tests that run without a GPU.

* the shared library loads and exports every CB_API symbol include/composer_b200.h declares
  (no compute calls: there is no device here);
* the ctypes signature table covers exactly the declared API;
* status codes map onto the reference's error classes;
* the config / module API behaves like the reference's (reference tests test_config.py,
  test_module.py): value semantics, REQUIRED, fn: resolution, errors, init determinism,
  golden round trips.
"""

import os

import numpy as np
import pytest

import paper_2507_05411_b200 as cb
from paper_2507_05411_b200 import _lib
from paper_2507_05411_b200.errors import (
    BadPathError,
    BadTopKError,
    KernelError,
    OddDimError,
    ShapeError,
    TypeMismatchError,
    UnknownActivationError,
    UnsetFieldError,
)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.cb_abi_version() == 1


def test_signature_table_matches_header():
    declared = set(_lib.declared_symbols())
    special = {"cb_last_error", "cb_launch_count"}
    assert set(_lib.SIGNATURES) | special == declared


def test_sort_scratch_sizes():
    """cb_sort_ids' scratch: one count per key and 1024-position chunk for the multi-CTA
    small-vocabulary sort (MoE expert ids), else one cursor per key (host-only query)."""
    lib = _lib.load()
    assert lib.cb_sort_ids_scratch(32768, 8) == 32 * 8
    assert lib.cb_sort_ids_scratch(1000, 8) == 8
    assert lib.cb_sort_ids_scratch(32768, 32000) == 32000


def test_status_mapping():
    _lib.load()
    with pytest.raises(ShapeError):
        _lib.check(_lib.CB_ERR_SHAPE)
    with pytest.raises(TypeMismatchError):
        _lib.check(_lib.CB_ERR_UNSUPPORTED)
    with pytest.raises(KernelError):
        _lib.check(_lib.CB_ERR_CUDA)


def test_shape_errors_raised_before_launch():
    """Argument validation happens in the library before any device work (no GPU needed)."""
    _lib.load()
    with pytest.raises(ShapeError):
        _lib.call("cb_gemm", -1, 4, 4, 1, None, 4, 0, None, 4, 0, 1, 4, 0, None, 0, 0, 1.0, 0, None)
    with pytest.raises(ShapeError):
        _lib.call("cb_rope", 4, 4, 1, 7, None, 7, 0, None, None, 0, None)
    with pytest.raises(ShapeError):
        _lib.call("cb_moe_route", 4, 8, 4, 5, None, 8, 0, None, None, None, None, None)
    with pytest.raises(ShapeError):
        _lib.call("cb_xent_fwd_bwd", 2, 1, 8, None, 8, 0, None, None, None, 0, 0, 1.0, None, None, None)


# ----------------------------------------------------------------------- config API
def test_value_semantics_and_paths():
    base = cb.default_config("Trainer")
    a = base.set("model.dim", 64)
    assert base.get("model.dim") is cb.REQUIRED and a.get("model.dim") == 64
    layer = cb.default_config("TransformerLayer").set("self_attention.num_heads", 4)
    b = a.set("model.decoder.transformer.layer", (layer, layer))
    c = b.set("model.decoder.transformer.layer[1].self_attention.num_heads", 8)
    assert b.get("model.decoder.transformer.layer[1].self_attention.num_heads") == 4
    assert c.get("model.decoder.transformer.layer[1].self_attention.num_heads") == 8
    with pytest.raises(BadPathError):
        a.set("model.nope", 1)
    with pytest.raises(TypeMismatchError):
        a.set("model.dim", "x")


def test_instantiate_propagates_and_resolves():
    cfg = cb.build_experiment("txf_rope")
    m = cb.instantiate(cfg)
    att = m.child("model.decoder.transformer.layer[0].self_attention")
    assert att.config.get("input_dim") == 32
    assert att.config.get("pos_emb.dim") == 8
    ff = m.child("model.decoder.transformer.layer[0].feed_forward")
    assert ff.config.get("hidden_dim") == 85  # floor(32 * 8/3 + 0.5)
    with pytest.raises(UnsetFieldError):
        cb.instantiate(cb.default_config("Trainer"))


def test_layer_validation_errors():
    with pytest.raises(ShapeError):
        cb.instantiate(cb.build_experiment("txf_base").set("model.dim", 30))
    with pytest.raises(OddDimError):
        cb.instantiate(cb.experiments.transformer_trainer(48, 1, "relu", pos_kind="RoPE", heads=16))
    with pytest.raises(UnknownActivationError):
        cb.instantiate(cb.build_experiment("txf_base").set("model.decoder.transformer.layer[0].feed_forward.activation",
                                                           "gelu"))
    with pytest.raises(BadTopKError):
        cb.instantiate(cb.build_experiment("txf_moe").set("model.decoder.transformer.layer[0].feed_forward.top_k", 9))


def test_init_state_deterministic_and_path_local():
    m = cb.instantiate(cb.build_experiment("txf_d16_l2_relu"))
    s1 = cb.init_state(m, cb.root_key(0))
    s2 = cb.init_state(m, cb.root_key(0))
    l0a = s1["model"]["decoder"]["transformer"]["layer[0]"]["self_attention"]["wq"]
    assert np.array_equal(l0a, s2["model"]["decoder"]["transformer"]["layer[0]"]["self_attention"]["wq"])
    l1a = s1["model"]["decoder"]["transformer"]["layer[1]"]["self_attention"]["wq"]
    assert not np.array_equal(l0a, l1a)


def test_flops_and_remat_metadata_match_reference_formulas():
    m = cb.instantiate(cb.build_experiment("txf_moe"))
    att = m.child("model.decoder.transformer.layer[0].self_attention")
    assert att.behavior.own_flops(att.config, 4, 8) == 8 * 32 * 32 * 32 + 4 * 32 * 8 * 32
    moe = m.child("model.decoder.transformer.layer[0].feed_forward")
    d, h, e, k, rows = 32, 85, 4, 2, 32
    assert moe.behavior.own_flops(moe.config, 4, 8) == 2 * rows * d * e + k * (2 * 2 * rows * d * h + 2 * rows * h * d)
    assert [t.name for t in moe.behavior.remat_tags(moe.config, 4, 8)] == ["router_logits", "expert_hidden",
                                                                             "expert_output"]


REF_GOLDENS = "/root/reference/pkg/tests/goldens"


@pytest.mark.skipif(not os.path.isdir(REF_GOLDENS), reason="reference goldens not present (GPU box)")
def test_reference_golden_configs_round_trip_and_instantiate():
    for f in sorted(os.listdir(REF_GOLDENS)):
        text = open(os.path.join(REF_GOLDENS, f)).read()
        cfg = cb.parse_golden(text)
        assert cb.serialize_golden(cfg) == text, f
        cb.instantiate(cfg)


def test_engine_layout_fuses_and_aligns():
    from paper_2507_05411_b200.engine import ALIGN, build_layout

    m = cb.instantiate(cb.BENCH_CONFIGS["1b"](batch=1, seq=128, layers=2))
    buckets = build_layout(m)
    names = [b.name for b in buckets]
    assert names[0] == "root" and names[-1] == "replicated"
    assert names[1] == "model.decoder.transformer.layer[0]"
    layer = buckets[1]
    att = {e.name: e for e in layer.entries if e.path.endswith("self_attention")}
    assert att["wq"].ld == att["wk"].ld == 3 * 2048 and att["wk"].col0 == 2048
    for b in buckets:
        for e in b.entries:
            assert e.offset % ALIGN == 0
    rep = buckets[-1]
    assert all(e.name == "scale" for e in rep.entries)


def test_checkpoint_plan_and_retention():
    """Checkpoint planning / retention restated from reference runtime_sim.py:22-157:
    exact partition, replicated shards round-robin, owned shards stay with their owner."""
    import pytest

    from paper_2507_05411_b200.checkpoint import GcPolicy, Shard, ShardManifest, gc_retained, plan_checkpoint

    shards = (Shard("a", 10), Shard("b", 20), Shard("c", 30, replicated=False, owner=1), Shard("d", 5),
              Shard("e", 7, replicated=False, owner=0), Shard("f", 1))
    plan = plan_checkpoint(ShardManifest(shards, replicas=2))
    assert [s.name for s in plan[0]] == ["a", "d", "e"] and [s.name for s in plan[1]] == ["b", "c", "f"]
    assert sorted(s.name for r in plan.values() for s in r) == sorted(s.name for s in shards)
    single = plan_checkpoint(ShardManifest(shards[:2], replicas=1))
    assert [s.name for s in single[0]] == ["a", "b"]
    with pytest.raises(ValueError):
        ShardManifest((Shard("x", 1), Shard("x", 2)))
    with pytest.raises(ValueError):
        ShardManifest((Shard("x", 1, replicated=False, owner=3),), replicas=2)
    assert gc_retained([1, 2, 3, 4, 5, 6], GcPolicy(keep_last_n=2, keep_every_k=3)) == {3, 5, 6}
    with pytest.raises(ValueError):
        GcPolicy()


def _reference_package():
    """The unmodified reference (oracle/_ref, or /root/reference in the build container)."""
    import sys

    for p in (os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "composer")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import composer

            return composer
    pytest.skip("reference package not available")


@pytest.mark.parametrize("name,devices,policy", [("7b", 1, None), ("7b", 4, None), ("1b", 8, "save_qkvo_flash"),
                                                 ("moe", 2, "recompute_all"), ("1b", 2, "offload_dots")])
def test_memory_plan_matches_reference_aot_analyze(name, devices, policy):
    """memory.aot_device_bytes == the reference's aot_analyze (mesh.py:563-686) on the bench
    configs: same golden text parsed by the reference, a catalog row with `devices` GPUs."""
    R = _reference_package()
    from composer.mesh import DeviceSpec, aot_analyze

    from paper_2507_05411_b200 import BENCH_CONFIGS, instantiate, serialize_golden
    from paper_2507_05411_b200.memory import aot_device_bytes
    from paper_2507_05411_b200.remat import POLICY_ALIASES

    cfg = BENCH_CONFIGS[name]()
    if policy:
        for i in range(len(cfg.get("model.decoder.transformer.layer"))):
            cfg = cfg.set(f"model.decoder.transformer.layer[{i}].remat_policy", POLICY_ALIASES[policy])
    cfg = cfg.set("mesh_shape", (devices,)).set("mesh_axis_names", ("fsdp",)).set("mesh_rules", ())
    B, T = cfg.get("batch_size") * devices, cfg.get("seq_len")
    cat = {"b200": DeviceSpec("b200", devices=devices, hbm_bytes=180_000_000_000, peak_flops=2.25e15,
                              interconnect_bps=9e11, hostlink_bps=6.4e10)}
    rep = aot_analyze(R.parse_golden(serialize_golden(cfg)), "b200", B, T, catalog=cat)
    mine = aot_device_bytes(instantiate(cfg), B, T, devices)
    assert mine["param_bytes"] == rep.param_bytes
    assert mine["optimizer_bytes"] == rep.optimizer_bytes
    assert mine["saved_activation_bytes"] == rep.saved_activation_bytes
    assert mine["per_device_bytes"] == rep.per_device_bytes


def test_remat_decisions_match_reference():
    """remat.resolve_policy / decide_tag (what every behavior's remat_decision applies) give the
    reference's decisions (mesh.py:204-252) for its named policies and mixed exact / glob maps."""
    _reference_package()
    from composer.mesh import decide_tag as ref_decide
    from composer.mesh import resolve_policy as ref_resolve

    from paper_2507_05411_b200.remat import decide_tag, resolve_policy

    tags = ["q_proj", "k_proj", "v_proj", "context", "o_proj", "hidden", "output", "router_logits", "expert_hidden",
            "expert_output", "logits", "unknown_tag"]
    policies = ["save_all", "recompute_all", "offload_dots", "save_qkvo_flash",
                {"hidden": "recompute", "*_proj": "offload"}, {"*": "save", "expert_*": "recompute", "expert_output": "save"},
                {"?_proj": "recompute", "*": "offload"}]
    for pol in policies:
        mine, ref = resolve_policy(pol), ref_resolve(pol)
        assert mine == ref
        for t in tags:
            assert decide_tag(t, mine) == ref_decide(t, ref), (pol, t)
