"""The training-step engine: parameter layout in HBM, FSDP, optimizer, step driver.

``TrainEngine(cfg)`` instantiates a reference-style Trainer config and owns:

* a **flat bucketed parameter layout** — one bucket per ``TransformerStack`` layer plus a
  root bucket (embedding, final norm, ...) and a small replicated bucket for f32-pinned
  tensors (norm scales, MoE router).  Inside a bucket an attention block's wq|wk|wv and a
  gated FFN's w1|w1_gate are laid out as column slices of one matrix so the behaviors
  issue one wide GEMM; every block is 64-element aligned (TMA needs 16 B).
* per bucket: f32 master shard, bf16 (or f32) working copy, f32 gradient, AdamW m/v shards.
  With world size 1 the shard is the whole bucket; large models keep the layers' gradients in
  a two-slot ring (``CB_GRAD_RING``), each layer updated right after its backward, inline on
  the compute stream.  Dense layers' weight-gradient GEMMs write their gradient buffers instead
  of accumulating into cleared ones (``overwrite_buckets``).
* **FSDP / ZeRO-3** (world size N > 1, one process per GPU, single node): parameters,
  gradients and optimizer state sharded 1/N; layer p's working copy is gathered into ring slot
  p % 2 on the comm stream (copy-engine reads of the peers' symmetric-memory shards, or NCCL)
  while the previous layer computes, again before its backward; its gradient is
  reduce-scattered right after its backward and AdamW runs on the in-order sum of the slices
  (``cb_adamw_parts``).  Sequences are independent, so the data path is plain data parallelism
  over the batch and the loss is the all-reduced mean (reference SPEC.md:445: numerics do not
  depend on partitioning).

The step itself is ``module.value_and_grad`` over the behaviors in ``layers.py``: no
PyTorch arithmetic, only C-ABI kernel launches.  PyTorch provides memory, streams and
``torch.distributed``.
"""

from __future__ import annotations

import os

import math
import re
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, ops
from .config import ConfigNode, visit
from .errors import MeshError, ShapeError, TypeMismatchError
from .module import Module, ParamProvider, instantiate, invoke, iter_param_specs, value_and_grad
from .prng import child_key, root_key

ALIGN = 64
_F32_KINDS = {("RMSNorm", "scale"), ("MoE", "router")}
_LAYER_RE = re.compile(r"^(.*\.transformer\.layer\[\d+\])(\.|$)")


def model_precision(cfg: ConfigNode) -> str:
    """The uniform compute dtype of every dtype-bearing node (the reference's DtypePolicy hook)."""
    tags = set()

    def enter(path, node):
        if node.has_field("dtype"):
            tags.add(node.get("dtype"))

    visit(cfg, enter_fn=enter)
    if not tags:
        return "f32"
    if len(tags) > 1:
        raise TypeMismatchError(f"mixed dtype policies are not supported: {sorted(tags)}")
    tag = tags.pop()
    if tag not in ("f32", "bf16"):
        raise TypeMismatchError(f"dtype {tag!r} has no B200 kernel path (supported: f32, bf16)")
    return tag


def set_dtype_policy(cfg: ConfigNode, tag: str) -> ConfigNode:
    """Sets `dtype` on every matmul-bearing node (what the reference's DtypePolicyModifier does)."""
    targets = []

    def enter(path, node):
        if node.has_field("dtype"):
            targets.append(path)

    visit(cfg, enter_fn=enter)
    for p in targets:
        cfg = cfg.set(f"{p}.dtype" if p else "dtype", tag)
    return cfg


DP_AXES = ("data", "fsdp")


def check_mesh(cfg: ConfigNode) -> None:
    """The step is data-parallel (FSDP over the batch): a mesh axis other than data/fsdp
    with a size other than 1 — e.g. the reference's gpu-H100 rule fsdp=-1, model=8
    (experiments.py:48) — would need tensor/expert parallelism, which this path does not
    implement, so it is rejected instead of silently running as data parallelism."""
    if not (cfg.has_field("mesh_axis_names") and cfg.has_field("mesh_shape")):
        return
    names, sizes = tuple(cfg.get("mesh_axis_names")), tuple(cfg.get("mesh_shape"))
    if len(names) != len(sizes):
        raise MeshError(f"mesh_shape {sizes} does not match mesh_axis_names {names}")
    for n, sz in zip(names, sizes):
        if n not in DP_AXES and int(sz) != 1:
            raise MeshError(f"mesh axis {n!r} of size {sz}: only data/fsdp axes are supported on this path "
                            f"(tensor/expert parallelism is not implemented)")


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


@dataclass
class Entry:
    path: str  # module path ("model.decoder.emb")
    name: str  # param name ("weight")
    shape: tuple
    offset: int  # element offset of the (group) block in the bucket
    col0: int = 0  # column offset inside a fused group
    ld: int = 0  # row stride inside a fused group (0 = contiguous)
    module_kind: str = ""


@dataclass
class Bucket:
    name: str
    entries: list = field(default_factory=list)
    numel: int = 0
    replicated: bool = False


def build_layout(module: Module) -> list[Bucket]:
    root = Bucket("root")
    rep = Bucket("replicated", replicated=True)
    layers: dict[str, Bucket] = {}
    order: list[Bucket] = []
    grouped = {}
    for path, mod, pname, shape in iter_param_specs(module):
        if (mod.kind, pname) in _F32_KINDS:
            b = rep
        else:
            m = _LAYER_RE.match(path)
            if m:
                key = m.group(1)
                if key not in layers:
                    layers[key] = Bucket(key)
                    order.append(layers[key])
                b = layers[key]
            else:
                b = root
        grouped.setdefault((id(b), path), (b, mod, []))[2].append((pname, shape))
    for (_, path), (b, mod, plist) in grouped.items():
        names = dict(plist)
        fuse = None
        if mod.kind in ("Attention", "GroupedQueryAttention") and {"wq", "wk", "wv"} <= set(names):
            fuse = ["wq", "wk", "wv"]
        elif mod.kind in ("FeedForward", "MoE") and {"w1", "w1_gate"} <= set(names):
            # gate and up projections side by side ([.., d, 2h]; per expert for MoE): one wide
            # GEMM with the gated activation in its epilogue
            fuse = ["w1", "w1_gate"]
        done = set()
        if fuse:
            rows = int(np.prod(names[fuse[0]][:-1]))
            width = sum(names[n][-1] for n in fuse)
            off = b.numel
            col = 0
            for n in fuse:
                b.entries.append(Entry(path, n, tuple(names[n]), off, col, width, mod.kind))
                col += names[n][-1]
                done.add(n)
            b.numel = _align(off + rows * width)
        for pname, shape in plist:
            if pname in done:
                continue
            b.entries.append(Entry(path, pname, tuple(shape), b.numel, 0, 0, mod.kind))
            b.numel = _align(b.numel + int(np.prod(shape)))
    out = [root] + order
    if rep.entries:
        out.append(rep)
    return [b for b in out if b.entries]


def _rc(e: Entry) -> tuple[int, int]:
    """(rows, cols) of an entry seen as a row-major matrix (leading dims folded into rows)."""
    return int(np.prod(e.shape[:-1])), int(e.shape[-1])


def _view(buf: torch.Tensor, e: Entry) -> torch.Tensor:
    if e.ld:
        # column block of a fused group: row stride ld; a leading expert dim folds into rows
        strides, acc = [1], e.ld
        for dim in reversed(e.shape[:-1]):
            strides.insert(0, acc)
            acc *= dim
        return buf.as_strided(tuple(e.shape), tuple(strides), buf.storage_offset() + e.offset + e.col0)
    n = int(np.prod(e.shape))
    return buf[e.offset:e.offset + n].view(e.shape)


def _tree_set(tree: dict, path: str, name: str, value):
    from .module import state_segments

    node = tree
    for seg in state_segments(path) if path else []:
        node = node.setdefault(seg, {})
    node[name] = value


def _tree_get(tree: dict, path: str, name: str):
    from .module import state_segments

    node = tree
    for seg in state_segments(path) if path else []:
        node = node[seg]
    return node[name]


def _skeleton(module: Module) -> dict:
    """Empty nested dicts for every module path (so state/grads trees mirror the reference)."""
    tree: dict = {}
    for name, c in module.children.items():
        tree[name] = _skeleton(c)
    return tree


def _on_device(fn):
    """Runs an engine entry point with its device current, so ops.stream_ptr() (the current
    device's current stream) and every launch target the engine's GPU even when it is not
    the caller's current device."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        if self.device.type != "cuda":
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self.device):
            return fn(self, *args, **kwargs)

    return wrapper


class _Dist:
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.group = group
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0


class TrainEngine:
    """Owns device state for one Trainer config and runs training steps on one GPU (rank)."""

    def __init__(self, cfg: ConfigNode, device=None, precision: str | None = None, seed: int = 0,
                 eps: float = 1e-8, weight_decay: float = 0.0, group=None, init: bool = True):
        self.cfg = cfg
        self.module = instantiate(cfg)
        self.cfg = self.module.config
        check_mesh(self.cfg)
        self.precision = precision or model_precision(self.cfg)
        if self.precision not in ("f32", "bf16"):
            raise TypeMismatchError(f"precision {self.precision!r} unsupported")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.work_dtype = torch.bfloat16 if self.precision == "bf16" else torch.float32
        learner = self.module.children.get("learner")
        spec = learner.impl if learner is not None else None
        self.lr = spec.lr if spec else 1e-3
        self.beta1 = spec.beta1 if spec else 0.9
        self.beta2 = spec.beta2 if spec else 0.999
        self.eps, self.weight_decay = eps, weight_decay
        self.seed = seed
        self.step_count = 0
        # FSDP + copy-engine reduce-scatter: step() sums the gradient slices inside AdamW; set
        # True to also store the summed gradient shards (grads_numpy() after step())
        self.keep_grad_shards = False
        self._grad_shards_stale = False
        self.d = _Dist(group)
        self.buckets = build_layout(self.module)
        self._alloc()
        # split-K is opt-in: measured on the 1B and MoE steps its partial round trip cost
        # more than the wave-quantization time it recovers (CB_GEMM_SPLITK=1 enables it)
        if os.environ.get("CB_GEMM_SPLITK", "0") == "1":
            ops.ensure_gemm_workspace(self.device)
        # epilogue staging mask of the CTA-pair GEMM (cb_gemm_set_staged_epilogue; A/B runs)
        if "CB_GEMM_STAGED_EPILOGUE" in os.environ and self.device.type == "cuda":
            _lib.call("cb_gemm_set_staged_epilogue", int(os.environ["CB_GEMM_STAGED_EPILOGUE"]))
        if "CB_GEMM_RASTER" in os.environ and self.device.type == "cuda":  # raster A/B
            _lib.call("cb_gemm_set_raster", int(os.environ["CB_GEMM_RASTER"]))
        self.options = {"precision": self.precision, "validate_ids": False,
                        "fuse_glu": os.environ.get("CB_FUSE_GLU", "1") != "0"}
        # weight-gradient GEMMs on their own stream (layers._wgrad), at most CB_WGRAD_STREAM of
        # them in flight; 0 keeps them on the compute stream
        self._wgrad_stream = None
        depth = int(os.environ.get("CB_WGRAD_STREAM", "4"))
        if self.device.type == "cuda" and depth > 0:
            self._wgrad_stream = torch.cuda.Stream(self.device)
            self.options["wgrad_stream"] = self._wgrad_stream
            self.options["wgrad_depth"] = depth
            self.options["wgrad_wave_eff"] = float(os.environ.get("CB_WGRAD_WAVE_EFF", "0.9"))
            self.options["wgrad_pending"] = self._wgrad_pending = []
        if self.d.world > 1:  # summaries that are global-batch statistics reduce over this group
            self.options["dp_group"] = self.d.group if self.d.group is not None else self.d.dist.group.WORLD
        if init:
            self.init_params(root_key(seed))

    # ------------------------------------------------------------------ memory
    def _alloc(self):
        N, dev = self.d.world, self.device
        # parameter all-gather as copy-engine peer reads of symmetric-memory working copies
        # (FSDPProvider._ag; 7B step +2.5% and MoE +1.3% at 4 GPUs, 1B neutral,
        # profiles/r01s3_ce_gather_ab/); CB_FSDP_CE_GATHER=0 gathers with NCCL
        self._ce_gather = (N > 1 and dev.type == "cuda" and self.d.world > 1
                           and os.environ.get("CB_FSDP_CE_GATHER", "1") == "1")
        # gradient reduce-scatter as copy-engine reads of the peers' slices + a local in-order
        # sum (cb_sum_parts); CB_FSDP_CE_REDUCE=0 reduce-scatters with NCCL
        self._ce_reduce = self._ce_gather and N <= 8 and os.environ.get("CB_FSDP_CE_REDUCE", "1") == "1"
        if self._ce_gather and int(os.environ.get("LOCAL_WORLD_SIZE", N)) != N:
            self._ce_gather = self._ce_reduce = False  # peers on another node: no peer mapping
        if self._ce_gather:
            # probe once, then agree: every rank takes the same collective path (a rank whose
            # driver cannot map peer memory would otherwise sit in NCCL while its peers spin
            # in a symmetric-memory barrier)
            ok = 1
            try:
                group = self.d.group if self.d.group is not None else self.d.dist.group.WORLD
                probe = _symm_mem().empty(16, dtype=torch.float32, device=dev)
                _symm_mem().rendezvous(probe, group)
            except Exception as exc:  # noqa: BLE001
                import warnings

                warnings.warn(f"symmetric memory unavailable on rank {self.d.rank} ({exc})")
                ok = 0
            flag = torch.tensor([ok], device=dev, dtype=torch.int32)
            self.d.dist.all_reduce(flag, op=self.d.dist.ReduceOp.MIN, group=self.d.group)
            if int(flag.item()) == 0:
                import warnings

                warnings.warn("symmetric memory unavailable on some rank; FSDP collectives use NCCL")
                self._ce_gather = self._ce_reduce = False
        # ZeRO-3 (N > 1): a layer's full bf16 working copy exists only in a ring of two gather
        # buffers (gathered before its forward and again before its backward), and its full f32
        # gradient only in a ring of two gradient buffers (reduce-scattered into the shard right
        # after its backward); the root bucket (embedding / final norm, used at both ends of the
        # step) stays gathered.  CB_FSDP_RESHARD=0 / CB_FSDP_GRAD_RING=0 keep full per-bucket
        # buffers instead.
        self.layer_order = [i for i, b in enumerate(self.buckets) if b.name != "root" and not b.replicated]
        self._pos = {i: p for p, i in enumerate(self.layer_order)}
        self._reshard = N > 1 and bool(self.layer_order) and os.environ.get("CB_FSDP_RESHARD", "1") == "1"
        self._grad_ring = N > 1 and bool(self.layer_order) and os.environ.get("CB_FSDP_GRAD_RING", "1") == "1"
        # one GPU: the same two-slot gradient ring when the layers' full f32 gradients would be
        # large (> CB_GRAD_RING_MIN_GB, default 16: the 7B step's 26 GB; not the 1B, MoE or 70B-layer
        # steps' 3.5 / 9.7 / 14.7 GB, which fit comfortably and run ~1% faster without it) —
        # each layer's AdamW runs right after its backward, so only two layers' gradients are ever
        # live; CB_GRAD_RING=0 / 1 forces it off / on
        if N == 1 and self.layer_order and self.device.type == "cuda":
            gbytes = 4 * sum(_align(self.buckets[i].numel) for i in self.layer_order)
            flag = os.environ.get("CB_GRAD_RING", "auto")
            self._grad_ring = flag == "1" or (flag == "auto" and gbytes > float(
                os.environ.get("CB_GRAD_RING_MIN_GB", "16")) * 1e9)
        ring_total = max([_align(self.buckets[i].numel, ALIGN * N) for i in self.layer_order] or [0])

        def symm_or_zeros(n, dtype, symm):
            if symm:
                return _symm_mem().empty(n, dtype=dtype, device=dev).zero_()
            return torch.zeros(n, device=dev, dtype=dtype)

        self._wring = [torch.zeros(ring_total, device=dev, dtype=self.work_dtype) for _ in range(2)] \
            if self._reshard else []
        self._gring = [symm_or_zeros(ring_total, torch.float32, self._ce_reduce) for _ in range(2)] \
            if self._grad_ring else []
        self.bufs = []
        for i, b in enumerate(self.buckets):
            if b.replicated:
                total = b.numel
                master = torch.zeros(total, device=dev, dtype=torch.float32)
                rec = dict(total=total, shard=total, master=master, work=master, wshard=master,
                           grad=torch.zeros(total, device=dev, dtype=torch.float32))
                rec["grad_shard"] = rec["grad"]
            else:
                total = _align(b.numel, ALIGN * N)
                shard = total // N
                r0 = self.d.rank * shard
                ringed = i in self._pos
                master = torch.zeros(shard, device=dev, dtype=torch.float32)
                if N == 1 and self.work_dtype == torch.float32:
                    work = wshard = master
                elif self._reshard and ringed:
                    work = self._wring[self._pos[i] % 2][:total]
                    wshard = symm_or_zeros(shard, self.work_dtype, self._ce_gather)
                else:
                    work = symm_or_zeros(total, self.work_dtype, self._ce_gather)
                    wshard = work[r0:r0 + shard]
                if N == 1:
                    grad = (self._gring[self._pos[i] % 2][:total] if (self._grad_ring and ringed)
                            else torch.zeros(total, device=dev, dtype=torch.float32))
                    grad_shard = grad
                else:
                    grad = (self._gring[self._pos[i] % 2][:total] if (self._grad_ring and ringed)
                            else symm_or_zeros(total, torch.float32, self._ce_reduce))
                    grad_shard = torch.zeros(shard, device=dev, dtype=torch.float32)
                rec = dict(total=total, shard=shard, master=master, work=work, wshard=wshard, grad=grad,
                           grad_shard=grad_shard, ringed=ringed)
            rec["m"] = torch.zeros(rec["shard"], device=dev, dtype=torch.float32)
            rec["v"] = torch.zeros(rec["shard"], device=dev, dtype=torch.float32)
            self.bufs.append(rec)
        if self._ce_gather:  # collective: every rank maps every peer's shards / gradient buffers
            group = self.d.group if self.d.group is not None else self.d.dist.group.WORLD
            for b, rec in zip(self.buckets, self.bufs):
                if b.replicated:
                    continue
                if self._reshard and rec["ringed"]:
                    rec["symm"] = _symm_mem().rendezvous(rec["wshard"], group)  # peers read the whole shard
                else:
                    rec["symm"] = _symm_mem().rendezvous(rec["work"], group)  # peers read slice p of it
                if self._ce_reduce and not (self._grad_ring and rec["ringed"]):
                    rec["gsymm"] = _symm_mem().rendezvous(rec["grad"], group)
            self._gring_symm = [_symm_mem().rendezvous(g, group) for g in self._gring] if self._ce_reduce else []
            if os.environ.get("CB_FSDP_MEMOP_BARRIER", "1") == "1":
                self._memop_barrier = _MemopBarrier(self, group)
            if self._ce_reduce:  # the peers' slices of one bucket's gradient, read before the sum
                big = max(r["shard"] for b, r in zip(self.buckets, self.bufs) if not b.replicated)
                self._rs_stage = torch.empty((N - 1) * big, device=dev, dtype=torch.float32)
        self.state = _skeleton(self.module)
        self.grads = _skeleton(self.module)
        for b, rec in zip(self.buckets, self.bufs):
            for e in b.entries:
                _tree_set(self.state, e.path, e.name, _view(rec["work"], e))
                _tree_set(self.grads, e.path, e.name, _view(rec["grad"], e))

    def _barrier(self, h) -> None:
        """A cross-rank barrier on the current (comm) stream: by default stream memory operations
        on the engine's own signal slots (cb_stream_signal / _wait: the GPU front end waits, no
        SM spins while a peer is late — 70B layer at 4 GPUs +1.5%, profiles/r02_memop_barrier_4gpu;
        a dead peer is caught by the NCCL watchdog on the step's loss all-reduce), or —
        CB_FSDP_MEMOP_BARRIER=0 — torch symmetric memory's barrier kernel on handle h, bounded by
        CB_SYMM_BARRIER_TIMEOUT_MS."""
        mb = getattr(self, "_memop_barrier", None)
        if mb is not None:
            mb()
        else:
            h.barrier(channel=0, timeout_ms=_BARRIER_TIMEOUT_MS)

    def _refresh_work(self, i: int) -> None:
        """This rank's slice of bucket i's working copy <- its f32 master shard."""
        self._gather_synced = False
        rec = self.bufs[i]
        if rec["wshard"].data_ptr() != rec["master"].data_ptr():
            ops.copy2d(rec["master"].view(1, -1), rec["wshard"].view(1, -1))

    def state_bytes(self) -> int:
        """Bytes of every persistent per-rank buffer the engine owns (master/work/grad/m/v,
        shard and staging buffers; each storage counted once)."""
        seen, total = set(), 0
        tensors = [t for rec in self.bufs for t in rec.values() if isinstance(t, torch.Tensor)]
        tensors += [t for t in (getattr(self, "_rs_stage", None),) if t is not None]
        tensors += list(getattr(self, "_gring", [])) + list(getattr(self, "_wring", []))
        for t in tensors:
            key = t.untyped_storage().data_ptr()
            if key not in seen:
                seen.add(key)
                total += t.untyped_storage().nbytes()
        return total

    def param_count(self) -> int:
        return sum(int(np.prod(e.shape)) for b in self.buckets for e in b.entries)

    # -------------------------------------------------------------- parameters
    def _host_bucket(self, b: Bucket, rec, values) -> None:
        """values(entry) -> np.ndarray; writes this rank's shard of the bucket's master + work."""
        self._gather_synced = False
        host = np.zeros(rec["total"], dtype=np.float32)
        for e in b.entries:
            arr = np.asarray(values(e), dtype=np.float64)
            if tuple(arr.shape) != tuple(e.shape):
                raise ShapeError(f"{e.path}.{e.name}: shape {arr.shape} != {e.shape}")
            if e.ld:
                rows, cols = _rc(e)
                blk = host[e.offset:e.offset + rows * e.ld].reshape(rows, e.ld)
                blk[:, e.col0:e.col0 + cols] = arr.reshape(rows, cols)
            else:
                host[e.offset:e.offset + arr.size] = arr.reshape(-1)
        r0 = 0 if b.replicated else self.d.rank * rec["shard"]
        t = torch.from_numpy(host[r0:r0 + rec["shard"]]).to(self.device)
        rec["master"].copy_(t)
        self._refresh_work(self.buckets.index(b))

    @_on_device
    def init_params(self, key) -> None:
        """Reference-identical init, generated on the device (init.cu: numpy's PCG64 stream
        reproduced bit-exactly from each tensor's key).  Kinds without a declarative
        ``param_init`` fall back to their host ``init_params``."""
        from . import _lib
        from .module import param_key
        from .prng import pcg64_state

        fallback = False
        for bi, (b, rec) in enumerate(zip(self.buckets, self.bufs)):
            if b.replicated:
                m0, m1 = 0, rec["total"]
            else:
                m0, m1 = self.d.rank * rec["shard"], (self.d.rank + 1) * rec["shard"]
            # one rank holds the whole bucket: master and working copy in one pass; under FSDP
            # only the own slice is written (from the master below) and peers gather it
            work = None if (rec["work"] is rec["master"] or self.d.world > 1) else rec["work"]
            wdt = ops.dt(rec["work"])
            for e in b.entries:
                mod = self.module.child(e.path) if e.path else self.module
                spec = mod.behavior.param_init(mod.config)
                if spec is None or e.name not in spec:
                    fallback = True
                    continue
                n = int(np.prod(e.shape))
                cols = e.shape[-1] if e.ld else 0
                kind = spec[e.name]
                if kind[0] == "uniform":
                    st, inc = pcg64_state(param_key(self._module_key(key, e.path), e.name))
                    mask = (1 << 64) - 1
                    _lib.call("cb_init_uniform", st & mask, st >> 64, inc & mask, inc >> 64, n, float(kind[1]),
                              float(kind[2]), cols, e.ld, e.col0, e.offset, rec["master"].data_ptr(), m0, m1,
                              work.data_ptr() if work is not None else None, wdt, ops.stream_ptr())
                else:
                    _lib.call("cb_init_const", n, float(kind[1]), cols, e.ld, e.col0, e.offset,
                              rec["master"].data_ptr(), m0, m1, work.data_ptr() if work is not None else None, wdt,
                              ops.stream_ptr())
            if self.d.world > 1:
                self._refresh_work(bi)
        torch.cuda.synchronize(self.device)
        if fallback:
            self.init_params_host(key)

    @_on_device
    def init_params_host(self, key) -> None:
        """Reference-identical init (init_state semantics) generated on the host, tensor by tensor."""
        from .module import param_key  # noqa: F401

        cache: dict = {}

        def values(e: Entry):
            if e.path not in cache:
                mod = self.module.child(e.path) if e.path else self.module
                cache.clear()
                cache[e.path] = mod.behavior.init_params(mod.config, self._module_key(key, e.path))
            return cache[e.path][e.name]

        for b, rec in zip(self.buckets, self.bufs):
            self._host_bucket(b, rec, values)
        torch.cuda.synchronize(self.device)

    @staticmethod
    def _module_key(key, path: str):
        from .module import state_segments

        for seg in state_segments(path) if path else []:
            key = child_key(key, seg, 0)
        return key

    @_on_device
    def load_state(self, state: dict) -> None:
        """Loads a reference-layout numpy state tree (e.g. from the reference's init_state)."""
        for b, rec in zip(self.buckets, self.bufs):
            self._host_bucket(b, rec, lambda e: _tree_get(state, e.path, e.name))
        torch.cuda.synchronize(self.device)

    @_on_device
    def load_opt_state(self, opt_state: dict | None) -> None:
        """AdamW state in the reference's tree layout: {"m": tree, "v": tree, "step": int}
        (None resets to the zero state of step 0)."""
        if opt_state is None:
            for rec in self.bufs:
                rec["m"].zero_()
                rec["v"].zero_()
            self.step_count = 0
            return
        for which in ("m", "v"):
            tree = opt_state[which]
            for b, rec in zip(self.buckets, self.bufs):
                host = np.zeros(rec["total"], dtype=np.float32)
                for e in b.entries:
                    arr = np.asarray(_tree_get(tree, e.path, e.name), dtype=np.float64)
                    if e.ld:
                        rows, cols = _rc(e)
                        host[e.offset:e.offset + rows * e.ld].reshape(rows, e.ld)[:, e.col0:e.col0 + cols] = \
                            arr.reshape(rows, cols)
                    else:
                        host[e.offset:e.offset + arr.size] = arr.reshape(-1)
                r0 = 0 if b.replicated else self.d.rank * rec["shard"]
                rec[which].copy_(torch.from_numpy(host[r0:r0 + rec["shard"]]).to(self.device))
        self.step_count = int(opt_state.get("step", 0))
        torch.cuda.synchronize(self.device)

    def opt_state_numpy(self) -> dict:
        return {"m": self._export("m"), "v": self._export("v"), "step": self.step_count}

    def _gather_full(self, buf: torch.Tensor, rec) -> torch.Tensor:
        if self.d.world == 1 or buf.numel() == rec["total"]:
            return buf
        full = torch.empty(rec["total"], device=self.device, dtype=buf.dtype)
        self.d.dist.all_gather_into_tensor(full, buf, group=self.d.group)
        return full

    @_on_device
    def _export(self, which: str) -> dict:
        out: dict = {}
        for b, rec in zip(self.buckets, self.bufs):
            if which == "grad" and self.d.world > 1 and not b.replicated:
                src = self._gather_full(rec["grad_shard"], rec)  # the reduce-scattered global mean
            else:
                src = rec[which]
            if which in ("master", "m", "v"):
                src = self._gather_full(src, rec)
            host = src.float().cpu().numpy().astype(np.float64)
            for e in b.entries:
                if e.ld:
                    rows, cols = _rc(e)
                    arr = host[e.offset:e.offset + rows * e.ld].reshape(rows, e.ld)[:, e.col0:e.col0 + cols]
                    arr = arr.copy().reshape(e.shape)
                else:
                    arr = host[e.offset:e.offset + int(np.prod(e.shape))].reshape(e.shape).copy()
                _tree_set(out, e.path, e.name, arr)
        return out

    def state_numpy(self) -> dict:
        return self._export("master")

    def grads_numpy(self) -> dict:
        """Global-batch gradients of the last step (under FSDP: the gathered reduce-scattered
        shards; replicated buckets were all-reduced in the step)."""
        if self._grad_shards_stale:
            from .errors import ComposerError

            raise ComposerError("step() did not keep the gradients (FSDP: the reduce-scatter's sum is fused into "
                                "AdamW; one GPU: AdamW fused into the weight-gradient GEMMs, or the gradient ring "
                                "— set engine.keep_grad_shards = True, and CB_GRAD_RING=0 for the ring, before the "
                                "step to read them)")
        return self._export("grad")

    # -------------------------------------------------------------------- step
    def upload_tokens(self, tokens) -> torch.Tensor:
        if isinstance(tokens, torch.Tensor) and tokens.is_cuda:
            return tokens
        arr = np.asarray(tokens)
        if arr.ndim != 2 or arr.shape[1] < 2 or not np.issubdtype(arr.dtype, np.integer):
            raise ShapeError("trainer expects integer tokens of shape [batch, seq>=2]")
        vocab = self.cfg.get("model.vocab_size")
        if arr.size and (arr.min() < 0 or arr.max() >= vocab):
            raise ShapeError(f"token ids out of range [0, {vocab})")
        host = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).pin_memory()
        return host.to(self.device, non_blocking=True)

    def step_key(self, step: int):
        return child_key(root_key(self.seed), "step", step)

    @_on_device
    def loss(self, tokens, step: int | None = None, key=None, collection: bool = False):
        """Forward-only loss (the reference's invoke(module, state, key, batch) result); with
        collection=True also the OutputCollection (summaries)."""
        toks = self.upload_tokens(tokens)
        provider = FSDPProvider(self) if self.d.world > 1 else None
        if provider:
            provider.start_step()
        if key is None:
            key = self.step_key(self.step_count if step is None else step)
        out, col = invoke(self.module, self.state, key, {"tokens": toks}, keep_outputs=False, provider=provider,
                          options=self.options)
        if collection:
            if self.d.world > 1:
                t = torch.tensor([out], device=self.device, dtype=torch.float64)
                self.d.dist.all_reduce(t, op=self.d.dist.ReduceOp.AVG, group=self.d.group)
                out = float(t.item())
            return out, col
        if self.d.world > 1:
            t = torch.tensor([out], device=self.device, dtype=torch.float64)
            self.d.dist.all_reduce(t, op=self.d.dist.ReduceOp.AVG, group=self.d.group)
            return float(t.item())
        return out

    @_on_device
    def compute_grads(self, tokens, update: bool = False, key=None):
        """Forward + backward; gradients land in the (sharded) grad buffers.  Returns (loss, collection).

        update=True also applies AdamW (step counter advanced first): each layer bucket is
        updated as soon as its gradient is final — right after that layer's backward, inline on
        the compute stream (one GPU), or after its reduce-scatter on the comm stream (FSDP).
        """
        toks = self.upload_tokens(tokens)
        if key is None:
            key = self.step_key(self.step_count)
        self._grad_shards_stale = False
        # FSDP: were the shards last written by a step() whose AdamW finished before its loss
        # all-reduce?  Then every peer's shards are final once that all-reduce completed, and
        # this step's forward gathers (ordered after it on the compute stream) need no barrier
        synced = getattr(self, "_gather_synced", False) and self.d.world > 1
        self._gather_synced = False
        if update:
            self.step_count += 1
        if self.d.world > 1:
            provider = FSDPProvider(self, update=update, synced=synced)
        else:
            if self._grad_ring and not update:
                from .errors import ComposerError

                raise ComposerError("this engine keeps single-GPU gradients in a two-layer ring (the model's "
                                    "gradients exceed CB_GRAD_RING_MIN_GB): compute_grads(update=False) cannot keep "
                                    "every layer's gradient; set CB_GRAD_RING=0 before building the engine")
            provider = LocalUpdateProvider(self) if update else None
        if provider is not None and self.device.type == "cuda":
            # the gradient buffers are cleared on a side stream while the forward runs (nothing
            # touches them before the backward, whose first hook waits for this)
            cur = torch.cuda.current_stream(self.device)
            if not hasattr(self, "_zero_stream"):
                self._zero_stream = torch.cuda.Stream(self.device)
            ready = torch.cuda.Event()
            ready.record(cur)
            written = set(provider.fused) | set(provider.overwrite)  # gradients never accumulated
            with torch.cuda.stream(self._zero_stream):
                self._zero_stream.wait_event(ready)
                for i, rec in enumerate(self.bufs):
                    if not (self._grad_ring and rec.get("ringed")) and i not in written:
                        ops.zero_(rec["grad"])
                zeroed = torch.cuda.Event()
                zeroed.record(self._zero_stream)
            provider.grads_zeroed = zeroed
        else:
            for rec in self.bufs:
                if not (self._grad_ring and rec.get("ringed")):
                    ops.zero_(rec["grad"])
        if provider:
            provider.start_step()
        if self.device.type == "cuda":
            # bytes the forward leaves allocated for the backward (saved activations, logits,
            # gathered copies) — compared with aot_analyze's saved_activation_bytes in bench.py.
            # (a weak reference: a closure over self in self.options would make a reference
            # cycle that keeps a dropped engine's HBM alive until the next gc pass)
            import weakref

            base = torch.cuda.memory_allocated(self.device)
            ref = weakref.ref(self)
            dev = self.device

            def forward_done():
                eng = ref()
                if eng is not None:
                    eng.last_forward_bytes = torch.cuda.memory_allocated(dev) - base

            self.options["forward_done"] = forward_done
        try:
            loss, col, _ = value_and_grad(self.module, self.state, self.grads, key, {"tokens": toks},
                                          provider=provider, options=self.options)
        finally:
            # a backward that raised must not leave a gradient region marked for overwrite /
            # fused update (a later buffer at the same address would be treated as one)
            ops.set_overwrite(None)
            ops.set_fused_update(None)
        if provider:
            provider.finish_backward()
        if self._wgrad_stream is not None:
            self._join_wgrad(torch.cuda.current_stream(self.device))
            self._wgrad_pending.clear()  # operands released after the compute stream's wait
        if self.d.world > 1:
            self.d.dist.all_reduce(loss, op=self.d.dist.ReduceOp.AVG, group=self.d.group)
            # every rank's AdamW of this step ran on its comm stream before its compute stream's
            # wait in finish_backward, i.e. before it joined this all-reduce
            self._gather_synced = bool(update) and os.environ.get("CB_FSDP_FWD_BARRIER", "0") != "1"
        return loss, col

    def _join_wgrad(self, stream) -> None:
        """`stream` waits for every weight-gradient GEMM issued so far (layers._wgrad)."""
        if self._wgrad_stream is not None and stream is not None:
            ev = torch.cuda.Event()
            ev.record(self._wgrad_stream)
            stream.wait_event(ev)

    # layer-bucket parameters whose whole gradient is one accumulating weight-gradient GEMM per
    # step (ops.gemm), so their AdamW can run in that GEMM's epilogue
    _FUSABLE = {("Attention", "wq"), ("Attention", "wk"), ("Attention", "wv"), ("Attention", "wo"),
                ("GroupedQueryAttention", "wq"), ("GroupedQueryAttention", "wk"),
                ("GroupedQueryAttention", "wv"), ("GroupedQueryAttention", "wo"),
                ("FeedForward", "w1"), ("FeedForward", "w1_gate"), ("FeedForward", "w2")}

    def dense_layer_buckets(self) -> dict[int, int]:
        """{bucket index: parameter count} of the layer buckets (bf16 working copy) holding only
        attention / dense-FFN projection weights, each of whose elements gets exactly one
        accumulating weight-gradient GEMM (ops.gemm) per backward — a MoE expert with no routed
        rows gets none, the tied embedding two, so their buckets are excluded."""
        out = {}
        if self.device.type != "cuda":
            return out
        for i, b in enumerate(self.buckets):
            if b.name == "root" or b.replicated or self.bufs[i]["wshard"].dtype != torch.bfloat16:
                continue
            if all((e.module_kind, e.name) in self._FUSABLE and len(e.shape) == 2 for e in b.entries):
                out[i] = sum(int(np.prod(e.shape)) for e in b.entries)
        return out

    def overwrite_buckets(self) -> dict[int, int]:
        """The dense layer buckets whose weight-gradient GEMMs write their gradient instead of
        adding it to a cleared buffer (ops.Overwrite): no clearing pass over those gradients
        (the 7B step: 26 GB of memset per step).  CB_WGRAD_OVERWRITE=0 turns it off."""
        if os.environ.get("CB_WGRAD_OVERWRITE", "1") == "0":
            return {}
        return self.dense_layer_buckets()

    def fused_update_buckets(self) -> dict[int, int]:
        """{bucket index: parameter count} of the buckets whose AdamW the single-GPU step runs in
        the weight-gradient GEMMs' epilogues (cb_gemm_adamw): opt-in (CB_FUSED_ADAMW=1), one
        GPU, bf16 working copy, layer buckets holding only attention / dense-FFN projection
        weights (a MoE expert with no routed rows has no GEMM but still a momentum update),
        gradients not kept for reading (keep_grad_shards).

        Off by default: measured, the update does not hide in the epilogue.  The weight-gradient
        GEMMs are bound by L2->SM operand traffic, and the epilogue's 24 bytes of optimizer
        state per element queue behind it — each 7B wgrad GEMM grows by the separate AdamW
        kernel's whole duration (QKV 0.88 -> 1.12 ms vs 0.25 ms of AdamW), the 7B step is 1.5%
        slower and the 1B step 0.8% faster (profiles/r02_fused_adamw_ab.txt)."""
        if self.d.world > 1 or self.keep_grad_shards or os.environ.get("CB_FUSED_ADAMW", "0") != "1":
            return {}
        return self.dense_layer_buckets()

    def _adamw_bucket(self, i: int, parts: list | None = None, scale: float = 1.0) -> None:
        """AdamW on bucket i's shard; with `parts` the gradient is scale * their in-order sum
        (the copy-engine reduce-scatter's slices, cb_adamw_parts), stored to the gradient shard
        only when keep_grad_shards is set."""
        rec = self.bufs[i]
        wshard = rec["wshard"]
        bf = wshard if (wshard.dtype == torch.bfloat16) else None
        if parts is not None:
            ops.adamw_parts(parts, scale, rec["grad_shard"] if self.keep_grad_shards else None, rec["master"],
                            rec["m"], rec["v"], bf, self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                            self.step_count)
            if not self.keep_grad_shards:
                self._grad_shards_stale = True
        else:
            ops.adamw(rec["master"], rec["grad_shard"], rec["m"], rec["v"], bf, self.lr, self.beta1, self.beta2,
                      self.eps, self.weight_decay, self.step_count)
        if bf is None and wshard.data_ptr() != rec["master"].data_ptr():
            ops.copy2d(rec["master"].view(1, -1), wshard.view(1, -1))

    @_on_device
    def apply_update(self) -> None:
        self._gather_synced = False  # the shards change after this step's loss all-reduce
        self.step_count += 1
        for i in range(len(self.buckets)):
            self._adamw_bucket(i)

    @_on_device
    def step(self, tokens):
        """One training step: forward, backward and the AdamW update (overlapped with backward)."""
        return self.compute_grads(tokens, update=True)


class GatherPlan:
    """Host-side plan of the parameter all-gathers of one FSDP step (pure Python: which bucket
    is gathered where and when, with or without the ordering barrier); FSDPProvider executes
    it on the comm stream.  tests/test_fsdp.py checks its invariants on CPU.

    Under ZeRO-3 (reshard) layer position p lives in gather slot p % 2: gathered before its
    forward (prefetched while position p - 1 computes) and again before its backward unless it
    is still resident (the forward's last two positions), prefetched while position p + 1's
    backward runs.  Without resharding every bucket has its own full buffer and is gathered once
    per step.  A forward gather carries the barrier that orders it after the peers' AdamW of the
    bucket (previous step); a backward re-gather needs none (see FSDPProvider._ag)."""

    def __init__(self, layer_order: list, reshard: bool):
        self.order = list(layer_order)
        self.pos = {b: p for p, b in enumerate(self.order)}
        self.reshard = reshard
        self.holder: dict[int, int] = {}  # slot -> bucket it holds
        self.done: set[int] = set()       # keep mode: buckets gathered this step

    def slot(self, b: int):
        return self.pos[b] % 2 if (self.reshard and b in self.pos) else None

    def _need(self, b: int) -> bool:
        s = self.slot(b)
        return (b not in self.done) if s is None else (self.holder.get(s) != b)

    def _take(self, b: int, backward: bool, out: list) -> None:
        if not self._need(b):
            return
        s = self.slot(b)
        if s is None:
            self.done.add(b)
        else:
            self.holder[s] = b
        out.append((b, s, not backward))

    def start(self, root: int) -> list:
        """Gathers issued at the start of the step: the root bucket, then the first layer."""
        out: list = []
        self._take(root, False, out)
        if self.order:
            self._take(self.order[0], False, out)
        return out

    def forward(self, b: int) -> list:
        """Gathers issued just before bucket b's forward: b (if not prefetched) and the next layer."""
        out: list = []
        self._take(b, False, out)
        p = self.pos.get(b)
        if p is not None and p + 1 < len(self.order):
            self._take(self.order[p + 1], False, out)
        return out

    def backward(self, b: int) -> list:
        """Gathers issued just before bucket b's backward (ZeRO-3 only): b if no longer resident
        and the previous layer."""
        out: list = []
        p = self.pos.get(b)
        if not self.reshard or p is None:
            return out
        self._take(b, True, out)
        if p > 0:
            self._take(self.order[p - 1], True, out)
        return out

    def resident(self, b: int) -> bool:
        return not self._need(b)


class FSDPProvider(ParamProvider):
    """Per-layer parameter all-gather (prefetched one layer ahead) and gradient
    reduce-scatter on a side (comm) stream: copy-engine peer reads of symmetric memory, or
    NCCL.  Under ZeRO-3 (eng._reshard / eng._grad_ring) layer p's gathered working copy and
    its full gradient live in ring slot p % 2: a gather waits for the compute stream to be
    done with the slot's previous layer, and the comm stream clears a gradient slot right
    after its reduce-scatter has been read by every peer."""

    def __init__(self, eng: TrainEngine, update: bool = False, synced: bool = False):
        self.e = eng
        self.update = update  # run AdamW on each bucket right after its reduce-scatter (comm stream)
        # the peers' shards are final (written by the previous step() before its loss
        # all-reduce): forward gathers skip their barrier
        self.synced = synced
        self.dist = eng.d.dist
        self.group = eng.d.group
        self.compute = torch.cuda.current_stream(eng.device)
        if not hasattr(eng, "_comm_stream"):
            eng._comm_stream = torch.cuda.Stream(eng.device, priority=_side_priority())
        self.comm = eng._comm_stream
        self.index = {b.name: i for i, b in enumerate(eng.buckets)}
        self.layer_order = eng.layer_order
        self.gathered: dict[int, torch.cuda.Event] = {}  # bucket -> gather-done event (this step)
        self.plan = GatherPlan(self.layer_order, eng._reshard)
        self.gslot_free: dict[int, torch.cuda.Event] = {}  # grad ring slot -> cleared event
        self.fused = {}
        self.overwrite = eng.overwrite_buckets()
        self.ow_cur = None

    def _run(self, actions: list) -> None:
        for i, slot, barrier in actions:
            self._ag(i, slot, barrier)

    def _ag(self, i: int, slot, barrier: bool) -> None:
        """Gathers bucket i (into ring slot `slot`, or its own full buffer when None) on the comm
        stream; `barrier`: order the reads after every peer's AdamW of the bucket."""
        rec, b = self.e.bufs[i], self.e.buckets[i]
        if b.replicated:
            return
        ready = torch.cuda.Event()
        ready.record(self.compute)  # the compute stream is done with the slot's previous layer
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ready)
            r, s, N = self.e.d.rank, rec["shard"], self.e.d.world
            work, own = rec["work"], rec["wshard"]
            h = rec.get("symm")
            if h is None:
                self.dist.all_gather_into_tensor(work, own, group=self.group)
            else:
                if slot is not None:  # the own slice too (in keep mode it is already in place)
                    work[r * s:(r + 1) * s].copy_(own)
                # pull every peer's shard over NVLink with the copy engines (no SMs taken from
                # the compute kernels).  Ordering with the shards' writers, the AdamW updates:
                # * forward gather: one barrier — each peer's AdamW of this bucket (previous
                #   step, earlier on its comm stream) has written its shard — unless the previous
                #   step() already ordered every peer's AdamW before its loss all-reduce, which
                #   this gather follows on this rank's streams (self.synced; CB_FSDP_FWD_BARRIER=1
                #   keeps the barrier);
                # * backward (re-)gather: none — no AdamW of this bucket can run anywhere before
                #   every rank has passed this bucket's reduce-scatter barrier, i.e. finished
                #   its backward of it, which comes after this gather;
                # * no barrier after the reads: a rank's next AdamW of this bucket waits for the
                #   same reduce-scatter barrier, which every reader passes only after its reads.
                if barrier and not self.synced:
                    self.e._barrier(h)
                for k in range(1, N):
                    p = (r + k) % N
                    if slot is not None:
                        src = h.get_buffer(p, (s,), work.dtype)
                    else:
                        src = h.get_buffer(p, (rec["total"],), work.dtype)[p * s:(p + 1) * s]
                    work[p * s:(p + 1) * s].copy_(src)
            done = torch.cuda.Event()
            done.record(self.comm)
        self.gathered[i] = done

    def _wait(self, i: int) -> None:
        """The compute stream waits for bucket i's most recent gather."""
        ev = self.gathered.get(i)
        if ev is not None:
            self.compute.wait_event(ev)

    def _rs(self, i: int) -> None:
        rec, b = self.e.bufs[i], self.e.buckets[i]
        ready = torch.cuda.Event()
        ready.record(self.compute)
        ring = self.e._grad_ring and rec.get("ringed")
        gslot = self.e._pos[i] % 2 if ring else None
        fused = False
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ready)
            self.e._join_wgrad(self.comm)
            N, r, s = self.e.d.world, self.e.d.rank, rec["shard"]
            h = self.e._gring_symm[gslot] if (ring and self.e._ce_reduce) else rec.get("gsymm")
            if b.replicated:
                self.dist.all_reduce(rec["grad"], op=self.dist.ReduceOp.AVG, group=self.group)
            elif h is not None:
                # barrier 1: every peer's backward of this bucket is complete (its comm stream
                # joined its compute and weight-gradient streams first); barrier 2: every peer
                # has read this rank's slices before they are cleared for the next use
                grad, stage = rec["grad"], self.e._rs_stage
                hn = self.e._gring[0].numel() if ring else rec["total"]  # size of the mapped buffer
                self.e._barrier(h)
                parts, j = [], 0
                for q in range(N):
                    if q == r:
                        parts.append(grad[r * s:(r + 1) * s])
                    else:
                        slot = stage[j * s:(j + 1) * s]
                        slot.copy_(h.get_buffer(q, (hn,), torch.float32)[r * s:(r + 1) * s])
                        parts.append(slot)
                        j += 1
                self.e._barrier(h)
                if self.update:  # the in-order sum fused into AdamW (no summed-gradient round trip)
                    self.e._adamw_bucket(i, parts=parts, scale=1.0 / N)
                    fused = True
                else:
                    ops.sum_parts(parts, rec["grad_shard"], 1.0 / N)
            else:
                self.dist.reduce_scatter_tensor(rec["grad_shard"], rec["grad"], op=self.dist.ReduceOp.AVG,
                                                group=self.group)
            if ring:  # the slot is free for the layer two positions further in the backward
                if i not in self.overwrite:  # (cleared unless that layer's GEMMs overwrite it)
                    ops.zero_(rec["grad"])
                ev = torch.cuda.Event()
                ev.record(self.comm)
                self.gslot_free[gslot] = ev
            if self.update and not fused:
                self.e._adamw_bucket(i)

    def start_step(self) -> None:
        self._run(self.plan.start(0))
        self._wait(0)

    def before_forward(self, path: str) -> None:
        i = self.index.get(path)
        if i is None:
            return
        self._run(self.plan.forward(i))
        self._wait(i)

    def before_backward(self, path: str) -> None:
        _wait_grads_zeroed(self)
        i = self.index.get(path)
        if i is None:
            return
        pos = self.e._pos.get(i)
        if pos is None:
            return
        if self.e._reshard:
            self._run(self.plan.backward(i))
            self._wait(i)
        if self.e._grad_ring:
            ev = self.gslot_free.pop(pos % 2, None)
            if ev is not None:
                self.compute.wait_event(ev)
        _begin_overwrite(self, i)

    def after_backward(self, path: str) -> None:
        i = self.index.get(path)
        if i is not None:
            _end_overwrite(self, i)
            self._rs(i)

    def finish_backward(self) -> None:
        _wait_grads_zeroed(self)
        for i, b in enumerate(self.e.buckets):
            if b.name == "root" or b.replicated:
                self._rs(i)
        done = torch.cuda.Event()
        done.record(self.comm)
        self.compute.wait_event(done)


class LocalUpdateProvider(ParamProvider):
    """Single-GPU step: AdamW of each layer bucket right after that layer's backward, on the
    compute stream (the root and replicated buckets, whose gradients complete last, at the
    end)."""

    def __init__(self, eng: TrainEngine):
        self.e = eng
        self.compute = torch.cuda.current_stream(eng.device)
        if not hasattr(eng, "_opt_stream"):
            eng._opt_stream = torch.cuda.Stream(eng.device, priority=_side_priority())
        # each layer's AdamW on the compute stream, between the layers' backward kernels: run
        # beside them (CB_ADAMW_INLINE=0, the comm stream) its HBM/L2 traffic slowed the backward
        # GEMMs by more than its own duration — inline is +1.0% (7B), +1.8% (1B), +1.2% (MoE)
        # per step (profiles/r02_adamw_inline_ab.txt)
        self.side = self.compute if os.environ.get("CB_ADAMW_INLINE", "1") == "1" else eng._opt_stream
        self.index = {b.name: i for i, b in enumerate(eng.buckets)}
        self.done: set[int] = set()
        self.gslot_free: dict[int, torch.cuda.Event] = {}  # gradient ring slot -> cleared event
        self.fused = eng.fused_update_buckets()
        self.overwrite = {i: n for i, n in eng.overwrite_buckets().items() if i not in self.fused}
        self.cur = None
        self.ow_cur = None

    def _update(self, i: int) -> None:
        ready = torch.cuda.Event()
        ready.record(self.compute)
        rec = self.e.bufs[i]
        with torch.cuda.stream(self.side):
            self.side.wait_event(ready)
            self.e._join_wgrad(self.side)
            if i in self.fused:
                # master / m / v were updated by the weight-gradient GEMMs' epilogues (the
                # gradient never reached HBM); the bf16 working copy is refreshed here, after
                # every data-gradient GEMM of the layer has read the old one
                ops.copy2d(rec["master"].view(1, -1), rec["wshard"].view(1, -1))
                self.e._grad_shards_stale = True
                self.done.add(i)
                return
            self.e._adamw_bucket(i)
            if self.e._grad_ring and rec.get("ringed"):
                # the gradient slot is consumed: clear it for the layer two positions further on
                # (unless that layer's GEMMs overwrite it)
                if i not in self.overwrite:
                    ops.zero_(rec["grad"])
                ev = torch.cuda.Event()
                ev.record(self.side)
                self.gslot_free[self.e._pos[i] % 2] = ev
                self.e._grad_shards_stale = True  # the layer gradients are gone after the step
        self.done.add(i)

    def before_backward(self, path: str) -> None:
        _wait_grads_zeroed(self)
        i = self.index.get(path)
        if self.e._grad_ring and i is not None and i in self.e._pos:
            ev = self.gslot_free.pop(self.e._pos[i] % 2, None)
            if ev is not None:
                self.compute.wait_event(ev)
        if i in self.fused:
            rec, e = self.e.bufs[i], self.e
            self.cur = (i, ops.FusedUpdate(rec["grad"], rec["master"], rec["m"], rec["v"], None, e.lr, e.beta1,
                                           e.beta2, e.eps, e.weight_decay, e.step_count))
            ops.set_fused_update(self.cur[1])
        _begin_overwrite(self, i)

    def after_backward(self, path: str) -> None:
        i = self.index.get(path)
        if i is not None:
            if self.cur is not None and self.cur[0] == i:
                ops.set_fused_update(None)
                fu, self.cur = self.cur[1], None
                if fu.covered != self.fused[i]:
                    from .errors import KernelError

                    raise KernelError(f"fused AdamW: the weight-gradient GEMMs of {self.e.buckets[i].name} covered "
                                      f"{fu.covered} of its {self.fused[i]} parameters")
            _end_overwrite(self, i)
            self._update(i)

    def finish_backward(self) -> None:
        _wait_grads_zeroed(self)
        for i in range(len(self.e.buckets)):
            if i not in self.done:
                self._update(i)
        fin = torch.cuda.Event()
        fin.record(self.side)
        self.compute.wait_event(fin)


class _MemopBarrier:
    """Barrier of all ranks from stream memory operations: the engine's int32 signal slots in
    symmetric memory (slot q on rank p = the last epoch rank q posted to p); every call posts
    the next epoch to its slot on each peer and waits for each peer's post on its own slots.
    All ranks issue barriers in the same program order on their comm streams, so epochs match."""

    def __init__(self, eng, group):
        import ctypes

        N, r = eng.d.world, eng.d.rank
        self.buf = _symm_mem().empty(N, dtype=torch.int32, device=eng.device).zero_()
        self.h = _symm_mem().rendezvous(self.buf, group)
        peers = [p for p in range(N) if p != r]
        self.views = [self.h.get_buffer(p, (N,), torch.int32) for p in peers]
        self.remote = (ctypes.c_void_p * len(peers))(*[v[r:r + 1].data_ptr() for v in self.views])
        self.local = (ctypes.c_void_p * len(peers))(*[self.buf[p:p + 1].data_ptr() for p in peers])
        self.n = len(peers)
        self.epoch = 0
        torch.cuda.synchronize(eng.device)
        eng.d.dist.barrier(group=group)  # every rank's slots are zero before the first post

    def __call__(self) -> None:
        import ctypes

        self.epoch += 1
        _lib.call("cb_stream_signal", ctypes.addressof(self.remote), self.n, self.epoch, ops.stream_ptr())
        _lib.call("cb_stream_wait", ctypes.addressof(self.local), self.n, self.epoch, ops.stream_ptr())


# symmetric-memory barriers time out (the kernel traps) instead of spinning forever when a
# peer has died; generous, because a peer may legitimately be a whole layer behind
_BARRIER_TIMEOUT_MS = int(os.environ.get("CB_SYMM_BARRIER_TIMEOUT_MS", "120000"))


def _symm_mem():
    import torch.distributed._symmetric_memory as symm_mem

    return symm_mem


def _begin_overwrite(provider, i) -> None:
    """Layer bucket i's backward starts: its weight-gradient GEMMs write its gradient buffer."""
    if i in provider.overwrite:
        provider.ow_cur = (i, ops.Overwrite(provider.e.bufs[i]["grad"]))
        ops.set_overwrite(provider.ow_cur[1])


def _end_overwrite(provider, i) -> None:
    """Layer bucket i's backward is done: every one of its parameters must have been written
    (a gradient element no GEMM wrote would hold another layer's value — fail loudly)."""
    cur = getattr(provider, "ow_cur", None)
    if cur is None or cur[0] != i:
        return
    ops.set_overwrite(None)
    provider.ow_cur = None
    if cur[1].covered != provider.overwrite[i]:
        from .errors import KernelError

        raise KernelError(f"weight-gradient overwrite: the GEMMs of {provider.e.buckets[i].name} wrote "
                          f"{cur[1].covered} of its {provider.overwrite[i]} gradient elements")


def _wait_grads_zeroed(provider) -> None:
    """The compute stream waits (once per step) for the side-stream clearing of the gradient
    buffers before the first backward kernel can write them."""
    ev = getattr(provider, "grads_zeroed", None)
    if ev is not None:
        provider.compute.wait_event(ev)
        provider.grads_zeroed = None


def _side_priority() -> int:
    """Priority of the optimizer / collective side streams: high (-1), so a layer's AdamW and
    its collectives get SMs ahead of queued compute blocks (MoE step +0.5%, 1B neutral,
    `profiles/r01s2_side_priority_ab.txt`); CB_SIDE_STREAM_PRIORITY=0 for torch's default."""
    return int(os.environ.get("CB_SIDE_STREAM_PRIORITY", "-1"))
