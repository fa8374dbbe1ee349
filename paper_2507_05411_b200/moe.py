"""MoE kind: token-choice top-k experts (reference layers.py:452-533), executed sparsely.

The reference evaluates every expert on every token (dense einsum, layers.py:519-525)
and then picks; the result only depends on the k selected experts, so the GPU path
computes exactly those: route (f64 router, stable top-k, renorm) -> stable
expert-sorted dispatch -> per-expert GEMMs on contiguous row blocks -> slot-order
combine.  FLOPs match the reference's own accounting, which already counts only the k
experts (layers.py:494-499).  ``load_balance_loss`` is recorded as a summary and, as in
the reference, is not part of the loss (layers.py:532 vs 649-651).

bf16 (the benchmark path): the dispatch writes each expert's rows at a 256-row boundary
(cb_moe_dispatch_padded, zero pad rows) and every expert projection — forward and backward,
weight gradients included — is ONE grouped CTA-pair GEMM launch that reads the expert
offsets on the GPU (cb_gemm_grouped / cb_gemm_gated_*_grouped): no host round trip and no
per-expert launch loop.  f32 (the parity mode) runs per-expert SIMT GEMMs sized from the E+1
offsets read back to the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, ops
from .errors import BadTopKError, ShapeError
from .module import Behavior, RematTag, add_summary, param, param_grad, param_key, save, saved


def _layers():
    from . import layers

    return layers


class MoEBehavior(Behavior):
    def validate(self, cfg):
        L = _layers()
        experts, top_k = cfg.get("num_experts"), cfg.get("top_k")
        if experts < 1 or not 1 <= top_k <= experts:
            raise BadTopKError(f"top_k={top_k} must lie in [1, {experts}]")
        pair = L.activation_pair(cfg.get("activation"))
        for n in pair if pair else (cfg.get("activation"),):
            L.check_activation(n)

    def param_shapes(self, cfg):
        d, h, e = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts")
        shapes = {"router": (d, e), "w1": (e, d, h), "w2": (e, h, d)}
        if _layers().activation_pair(cfg.get("activation")):
            shapes["w1_gate"] = (e, d, h)
        return shapes

    def param_specs(self, cfg):
        spec = tuple(cfg.get("param_partition_spec"))
        rev = tuple(reversed(spec))
        specs = {"router": (spec[0], None), "w1": (None,) + spec, "w2": (None,) + rev}
        if _layers().activation_pair(cfg.get("activation")):
            specs["w1_gate"] = (None,) + spec
        return specs

    def init_params(self, cfg, key):
        L = _layers()
        d, h, e = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts")
        out = {"router": L.fan_in_uniform(param_key(key, "router"), (d, e), d),
               "w1": L.fan_in_uniform(param_key(key, "w1"), (e, d, h), d),
               "w2": L.fan_in_uniform(param_key(key, "w2"), (e, h, d), h)}
        if L.activation_pair(cfg.get("activation")):
            out["w1_gate"] = L.fan_in_uniform(param_key(key, "w1_gate"), (e, d, h), d)
        return out

    def param_init(self, cfg):
        L = _layers()
        d, h = cfg.get("input_dim"), cfg.get("hidden_dim")
        out = {"router": L.uniform_spec(d), "w1": L.uniform_spec(d), "w2": L.uniform_spec(h)}
        if L.activation_pair(cfg.get("activation")):
            out["w1_gate"] = L.uniform_spec(d)
        return out

    def own_flops(self, cfg, batch, seq_len):
        d, h, e, k = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts"), cfg.get("top_k")
        rows = batch * seq_len
        br = 2 if _layers().activation_pair(cfg.get("activation")) else 1
        return 2 * rows * d * e + k * (br * 2 * rows * d * h + 2 * rows * h * d)

    def remat_tags(self, cfg, batch, seq_len):
        d, h, e, k = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts"), cfg.get("top_k")
        rows = batch * seq_len
        nb = _layers().DTYPE_BYTES[cfg.get("dtype")]
        br = 2 if _layers().activation_pair(cfg.get("activation")) else 1
        return [RematTag("router_logits", rows * e * nb, 2 * rows * d * e),
                RematTag("expert_hidden", k * br * rows * h * nb, k * br * 2 * rows * d * h),
                RematTag("expert_output", k * rows * d * nb, k * 2 * rows * h * d)]

    # ------------------------------------------------------------------ execution
    fuses_residual = True  # forward(x, residual=r) returns r + moe(x) from the combine kernel

    def forward(self, module, x, residual=None):
        L = _layers()
        cfg = module.config
        d, h, E, k = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts"), cfg.get("top_k")
        B, T = L._checked_3d(x, d, "MoE")
        adt = L.act_dtype()
        dev = x.device
        x2 = ops.cast(ops.rows2d(x), adt)
        n = x2.shape[0]
        router = L._f32(param("router"))
        idx = torch.empty((n, k), device=dev, dtype=torch.int32)
        w = torch.empty((n, k), device=dev, dtype=torch.float32)
        probs = torch.empty((n, E), device=dev, dtype=torch.float32)
        _lib.call("cb_moe_route", n, d, E, k, x2.data_ptr(), ops.ld(x2), ops.dt(x2), router.data_ptr(),
                  idx.data_ptr(), w.data_ptr(), probs.data_ptr(), ops.stream_ptr())
        stats = torch.empty((1 + 2 * E,), device=dev, dtype=torch.float64)
        _lib.call("cb_moe_stats", n, E, k, idx.data_ptr(), probs.data_ptr(), stats.data_ptr(), ops.stream_ptr())
        grp = L.option("dp_group")
        if grp is not None:
            # data parallel: f_e and p_e are global-batch statistics, so the per-expert counts
            # and probability sums are all-reduced before forming E * sum_e f_e p_e (SURVEY
            # §8(e) C3); a (1 + 2E)-double collective on the compute stream
            import torch.distributed as dist

            raw = stats[1:].clone()
            raw[E:] *= n
            dist.all_reduce(raw, group=grp)
            n_glob = n * dist.get_world_size(grp)
            f = raw[:E] / (n_glob * k)
            p = raw[E:] / n_glob
            stats = torch.cat([(E * (f * p).sum()).view(1), raw[:E], p])
        add_summary("load_balance_loss", stats[0:1] if L.is_recording() else float(stats[0].item()))
        if L.option("moe_balanced_routing", False):
            # BENCHMARK KNOB ONLY (bench.py --moe-routing balanced): token t's slot j goes to
            # expert (t*k + j) % E, so every expert gets n*k/E rows — the dispatch, grouped
            # GEMMs and combine measured off the reference init's degenerate routing
            idx.copy_((torch.arange(n * k, device=dev, dtype=torch.int32) % E).view(n, k))
        if L.option("record_routing", False):  # debug summary: the chosen experts per token
            add_summary("route_indices", idx.view(B, T, k))
        # stable expert-sorted dispatch of the n*k assignments
        ids64 = torch.empty((n * k,), device=dev, dtype=torch.int64)
        _lib.call("cb_widen_i32", n * k, idx.data_ptr(), ids64.data_ptr(), ops.stream_ptr())
        offsets, perm = ops.sort_ids(ids64, E)
        if self._grouped_ok(module, adt):
            # all experts in one grouped launch per projection, expert offsets read on the GPU:
            # each expert's rows padded to a 256-row boundary (zero rows), no host round trip
            cap = (n * k + 255 * E + 255) // 256 * 256
            xe = torch.empty((cap, d), device=dev, dtype=adt)
            poff = torch.empty((E + 1,), device=dev, dtype=torch.int32)
            inv = torch.empty((n * k,), device=dev, dtype=torch.int32)  # assignment -> padded row
            _lib.call("cb_moe_dispatch_padded", n * k, d, E, k, offsets.data_ptr(), perm.data_ptr(), x2.data_ptr(),
                      ops.ld(x2), ops.dt(x2), poff.data_ptr(), inv.data_ptr(), xe.data_ptr(), ops.ld(xe), cap,
                      ops.stream_ptr())
            off = ("grouped", offsets, poff, n * k)
        else:
            # per-expert GEMMs sized on the host: the E+1 offsets are copied out right after
            # the sort, so the host waits only for the sort while the gather below still runs
            off_host = _pinned_offsets(E + 1)
            off_host.copy_(offsets, non_blocking=True)
            off_ready = torch.cuda.Event()
            off_ready.record()
            inv = torch.empty((n * k,), device=dev, dtype=torch.int32)
            _lib.call("cb_invert_perm", n * k, perm.data_ptr(), inv.data_ptr(), ops.stream_ptr())
            xe = torch.empty((n * k, d), device=dev, dtype=adt)
            _lib.call("cb_gather_rows", n * k, d, perm.data_ptr(), k, x2.data_ptr(), ops.ld(x2), xe.data_ptr(),
                      ops.ld(xe), ops.dt(xe), ops.stream_ptr())
            off_ready.synchronize()
            off = off_host.numpy().astype(np.int64)
        pre, hid = self._experts_up(module, xe, off)
        ye = self._experts_down(module, hid, off)
        out = torch.empty((n, d), device=dev, dtype=torch.float32)
        res = None if residual is None else ops.rows2d(residual)
        if not (res is not None and ye.dtype == torch.float32 and res.dtype == torch.float32 and _lib.try_call(
                "cb_moe_combine_residual", n, d, k, inv.data_ptr(), w.data_ptr(), ye.data_ptr(), ops.ld(ye),
                res.data_ptr(), ops.ld(res), out.data_ptr(), ops.ld(out), ops.stream_ptr())):
            _lib.call("cb_moe_combine", n, d, k, inv.data_ptr(), w.data_ptr(), ye.data_ptr(), ops.ld(ye), ops.dt(ye),
                      out.data_ptr(), ops.ld(out), 0, ops.stream_ptr())
            if res is not None:
                ops.add_(out, res)
        if L.is_recording():
            # remat tags (reference layers.py:501-511): router_logits = the router
            # probabilities, expert_hidden = the experts' up-projections, expert_output = the
            # experts' outputs (read by the combine backward for the routing-weight gradient)
            save(x2=x2, idx=idx, w=w, probs=L.keep(probs, L.remat_plan("router_logits")), perm=perm, inv=inv,
                 off=off, xe=xe, pre=L.keep(pre, L.remat_plan("expert_hidden")),
                 hid=L.keep(hid, L.remat_plan("expert_hidden")), ye=L.keep(ye, L.remat_plan("expert_output")),
                 geom=(B, T, d, h, E, k))
        return out.view(B, T, d)

    @staticmethod
    def _stacked(module):
        """Every expert's [W1|Wg] as one [E*d, 2h] matrix and W2 as [E*h, d] (views of the
        bucket), or None when the layout is not the engine's fused one."""
        L = _layers()
        cfg = module.config
        d, h, E = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts")
        w1, wg, w2 = param("w1"), param("w1_gate"), param("w2")
        es = w1.element_size()
        if (w1.stride() != (d * 2 * h, 2 * h, 1) or wg.stride() != w1.stride()
                or wg.data_ptr() != w1.data_ptr() + h * es or not w2.is_contiguous()):
            return None
        return torch.as_strided(w1, (E * d, 2 * h), (2 * h, 1)), w2.view(E * h, d)

    @staticmethod
    def _stacked_grads(module):
        cfg = module.config
        d, h, E = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts")
        g1, gg, g2 = param_grad("w1"), param_grad("w1_gate"), param_grad("w2")
        if (g1.stride() != (d * 2 * h, 2 * h, 1) or gg.data_ptr() != g1.data_ptr() + h * g1.element_size()
                or not g2.is_contiguous()):
            return None
        return torch.as_strided(g1, (E * d, 2 * h), (2 * h, 1)), g2.view(E * h, d)

    def _grouped_ok(self, module, adt) -> bool:
        L = _layers()
        cfg = module.config
        pair = L.activation_pair(cfg.get("activation"))
        return (adt == torch.bfloat16 and pair is not None and L.option("fuse_glu", True)
                and L.option("moe_grouped", True) and cfg.get("hidden_dim") % 128 == 0
                and cfg.get("input_dim") % 64 == 0 and cfg.get("num_experts") <= 64
                and self._stacked(module) is not None)

    def _experts_up(self, module, xe, off):
        """pre / hid of every expert's rows (gate/up GEMM with the gated activation in its
        epilogue): one grouped launch over the padded layout, or per expert on its rows."""
        L = _layers()
        cfg = module.config
        h, E = cfg.get("hidden_dim"), cfg.get("num_experts")
        adt = L.act_dtype()
        dev = xe.device
        nk = xe.shape[0]
        pair = L.activation_pair(cfg.get("activation"))
        if isinstance(off, tuple):
            w1s, _ = self._stacked(module)
            pre = torch.empty((nk, 2 * h), device=dev, dtype=adt)
            hid = torch.empty((nk, h), device=dev, dtype=adt)
            ops.gemm_gated_fwd_grouped(xe, w1s, off[2], E, pair[0], pair[1], pre, hid, rows=off[3])
            return pre, hid
        w1 = param("w1")
        wg = param("w1_gate") if pair else None
        width = 2 * h if pair else h
        pre = torch.empty((nk, width), device=dev, dtype=adt)
        hid = torch.empty((nk, h), device=dev, dtype=adt)
        fused_all = pair is not None and L.option("fuse_glu", True)
        unfused = []
        for e in range(E):
            r0, r1 = int(off[e]), int(off[e + 1])
            if r1 == r0:
                continue
            xs = xe[r0:r1]
            wcat = L.fused_columns(w1[e], wg[e]) if fused_all else None
            if wcat is not None and ops.gemm_gated_fwd(xs, wcat, pair[0], pair[1], pre=pre[r0:r1],
                                                       hidden=hid[r0:r1]) is not None:
                continue
            ops.gemm(xs, w1[e], pre[r0:r1, :h])
            if pair:
                ops.gemm(xs, wg[e], pre[r0:r1, h:])
            unfused.append((r0, r1))
        for r0, r1 in unfused:
            if pair:
                ops.act_fwd(pre[r0:r1, :h], pre[r0:r1, h:], pair[0], pair[1], out=hid[r0:r1])
            else:
                ops.act_fwd(pre[r0:r1], None, cfg.get("activation"), out=hid[r0:r1])
        return pre, hid

    def _experts_down(self, module, hid, off):
        cfg = module.config
        d, E = cfg.get("input_dim"), cfg.get("num_experts")
        w2 = param("w2")
        ye = torch.empty((hid.shape[0], d), device=hid.device, dtype=torch.float32)
        if isinstance(off, tuple):
            ops.gemm_grouped_rows(hid, self._stacked(module)[1], ye, off[2], E, rows=off[3])
            return ye
        for e in range(E):
            r0, r1 = int(off[e]), int(off[e + 1])
            if r1 > r0:
                ops.gemm(hid[r0:r1], w2[e], ye[r0:r1])
        return ye

    def backward(self, module, dout):
        L = _layers()
        cfg = module.config
        s = saved()
        B, T, d, h, E, k = s["geom"]
        adt = L.act_dtype()
        dev = dout.device
        n = B * T
        off, xe = s["off"], s["xe"]
        pre, hid = L.restore(s["pre"]), L.restore(s["hid"])
        if pre is None:  # expert_hidden rematerialised
            pre, hid = self._experts_up(module, xe, off)
        ye = L.restore(s["ye"])
        if ye is None:  # expert_output rematerialised
            ye = self._experts_down(module, hid, off)
        probs = L.restore(s["probs"])
        if probs is None:  # router_logits rematerialised (same deterministic kernel: same top-k)
            probs = torch.empty((n, E), device=dev, dtype=torch.float32)
            i2 = torch.empty((n, k), device=dev, dtype=torch.int32)
            w2_ = torch.empty((n, k), device=dev, dtype=torch.float32)
            x2 = s["x2"]
            _lib.call("cb_moe_route", n, d, E, k, x2.data_ptr(), ops.ld(x2), ops.dt(x2), L._f32(param("router")).data_ptr(),
                      i2.data_ptr(), w2_.data_ptr(), probs.data_ptr(), ops.stream_ptr())
        g = ops.rows2d(dout).contiguous() if dout.dtype == torch.float32 else ops.cast(ops.rows2d(dout), torch.float32)
        grouped = isinstance(off, tuple)
        dye = torch.empty((xe.shape[0], d), device=dev, dtype=adt)
        if grouped:  # the pad rows feed the grouped weight-gradient GEMMs: zero
            _lib.call("cb_moe_zero_pad_rows", xe.shape[0], d, E, off[1].data_ptr(), off[2].data_ptr(), dye.data_ptr(),
                      ops.ld(dye), ops.dt(dye), ops.stream_ptr())
        dw = torch.empty((n, k), device=dev, dtype=torch.float32)
        _lib.call("cb_moe_combine_bwd", n, d, k, s["inv"].data_ptr(), s["w"].data_ptr(), ye.data_ptr(),
                  ops.ld(ye), g.data_ptr(), ops.ld(g), dye.data_ptr(), ops.ld(dye), ops.dt(dye), dw.data_ptr(),
                  ops.stream_ptr())
        pair = L.activation_pair(cfg.get("activation"))
        if grouped:
            dxe = self._experts_bwd_grouped(module, xe, pre, hid, dye, off[2], pair, off[3])
        else:
            dxe = self._experts_bwd(module, xe, pre, hid, dye, off, pair)
        dx = torch.empty((n, d), device=dev, dtype=torch.float32)
        _lib.call("cb_moe_combine", n, d, k, s["inv"].data_ptr(), None, dxe.data_ptr(), ops.ld(dxe), ops.dt(dxe),
                  dx.data_ptr(), ops.ld(dx), 0, ops.stream_ptr())
        # router: w = renorm(topk(softmax(x @ router)))
        dlog = torch.empty((n, E), device=dev, dtype=torch.float32)
        _lib.call("cb_moe_router_bwd", n, E, k, probs.data_ptr(), s["idx"].data_ptr(), s["w"].data_ptr(),
                  dw.data_ptr(), dlog.data_ptr(), ops.stream_ptr())
        router = L._f32(param("router"))
        x2 = s["x2"]
        ws = torch.empty(((n + 127) // 128) * d * E, device=dev, dtype=torch.float32)
        _lib.call("cb_moe_router_bwd_gemms", n, d, E, x2.data_ptr(), ops.ld(x2), ops.dt(x2), dlog.data_ptr(),
                  router.data_ptr(), param_grad("router").data_ptr(), dx.data_ptr(), ops.ld(dx), ws.data_ptr(),
                  ops.stream_ptr())
        return dx.view(B, T, d)

    def _experts_bwd_grouped(self, module, xe, pre, hid, dye, poff, pair, rows):
        """The experts' backward in four grouped launches: dpre (dhidden = dye @ W2^T formed
        and consumed by the gated-activation backward in the epilogue), dW2 += hid^T dye,
        d[W1|Wg] += xe^T dpre (grouped over K: each expert's own rows), dxe = dpre @ [W1|Wg]^T."""
        cfg = module.config
        d, E = cfg.get("input_dim"), cfg.get("num_experts")
        w1s, w2s = self._stacked(module)
        g1s, g2s = self._stacked_grads(module)
        dpre = torch.empty_like(pre)
        ops.gemm_gated_bwd_grouped(dye, w2s, poff, E, pre, pair[0], pair[1], dpre, rows=rows)
        ops.gemm_grouped_k(hid, dye, g2s, poff, E, rows=rows)
        ops.gemm_grouped_k(xe, dpre, g1s, poff, E, rows=rows)
        dxe = torch.empty((xe.shape[0], d), device=xe.device, dtype=torch.float32)
        ops.gemm_grouped_rows(dpre, w1s, dxe, poff, E, trans_b=True, rows=rows)
        return dxe

    def _experts_bwd(self, module, xe, pre, hid, dye, off, pair):
        L = _layers()
        cfg = module.config
        d, h, E = cfg.get("input_dim"), cfg.get("hidden_dim"), cfg.get("num_experts")
        dev = xe.device
        n_k = xe.shape[0]
        w1, w2 = param("w1"), param("w2")
        gw1, gw2 = param_grad("w1"), param_grad("w2")
        wg = param("w1_gate") if pair else None
        gwg = param_grad("w1_gate") if pair else None
        dpre = torch.empty_like(pre)
        dhid = None
        fuse = pair is not None and L.option("fuse_glu", True)
        for e in range(E):
            r0, r1 = int(off[e]), int(off[e + 1])
            if r1 == r0:
                continue
            ops.gemm(hid[r0:r1], dye[r0:r1], gw2[e], trans_a=True, accumulate=True)
            # dhidden = dye @ w2^T consumed by the gated-activation backward in the epilogue
            if fuse and ops.gemm_gated_bwd(dye[r0:r1], w2[e], pre[r0:r1], pair[0], pair[1],
                                           dpre=dpre[r0:r1]) is not None:
                continue
            if dhid is None:
                dhid = torch.empty_like(hid)
            ops.gemm(dye[r0:r1], w2[e], dhid[r0:r1], trans_b=True)
            if pair:
                ops.act_bwd(pre[r0:r1, :h], pre[r0:r1, h:], dhid[r0:r1], dpre[r0:r1, :h], dpre[r0:r1, h:], pair[0],
                            pair[1])
            else:
                ops.act_bwd(pre[r0:r1], None, dhid[r0:r1], dpre[r0:r1], None, cfg.get("activation"))
        dxe = torch.empty((n_k, d), device=dev, dtype=torch.float32)
        for e in range(E):
            r0, r1 = int(off[e]), int(off[e + 1])
            if r1 == r0:
                continue
            xs = xe[r0:r1]
            ops.gemm(xs, dpre[r0:r1, :h], gw1[e], trans_a=True, accumulate=True)
            ops.gemm(dpre[r0:r1, :h], w1[e], dxe[r0:r1], trans_b=True)
            if pair:
                ops.gemm(xs, dpre[r0:r1, h:], gwg[e], trans_a=True, accumulate=True)
                ops.gemm(dpre[r0:r1, h:], wg[e], dxe[r0:r1], trans_b=True, accumulate=True)
        return dxe


_PINNED: dict = {}


def _pinned_offsets(n: int) -> torch.Tensor:
    """A reusable pinned int32 host buffer for the expert offsets (read before the next use)."""
    t = _PINNED.get(n)
    if t is None:
        t = _PINNED[n] = torch.empty((n,), dtype=torch.int32, pin_memory=True)
    return t
