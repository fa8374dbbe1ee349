"""Functional step entry points on the reference's own data layout (SURVEY §8(b) "Step entry").

The reference's step is ``invoke(module, state, key, batch) -> (loss, OutputCollection)``
(reference module.py:351-365): pure, fp64 numpy state tree in, nothing mutated.  These two
functions keep that contract for callers that hold reference-layout state, and add the
training step the reference does not have:

* ``forward_loss(module, state, key, batch)``       -> (loss, OutputCollection)
* ``train_step(module, state, opt_state, key, batch)`` -> (loss, summaries, new_state,
  new_opt_state[, grads])

Both run on the GPU through ``TrainEngine`` (the same kernels as the benchmark path); the
state trees are uploaded to / downloaded from the device around the call, so they are the
drop-in form, not the fast path (``TrainEngine.step`` keeps everything resident).  Inputs
are never mutated.  ``opt_state`` is ``None`` (fresh AdamW) or ``{"m": tree, "v": tree,
"step": int}`` with ``m`` / ``v`` in the state's tree layout.
"""

from __future__ import annotations

from typing import Any

import numpy as np

from .errors import ShapeError

_CACHE: dict[Any, Any] = {}


def _engine(module, device, precision):
    """One TrainEngine per (config, device, precision), reused across calls."""
    import torch

    from .engine import TrainEngine

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (id(module.config), str(dev), precision)
    hit = _CACHE.get(key)
    if hit is None or hit[0] is not module.config:  # the cached config object pins its id
        _CACHE.clear()
        hit = (module.config, TrainEngine(module.config, device=dev, precision=precision, init=False))
        _CACHE[key] = hit
    return hit[1]


def _tokens(batch) -> np.ndarray:
    if not isinstance(batch, dict) or "tokens" not in batch:
        raise ShapeError("batch must be a dict with 'tokens' [batch, seq] int64")
    return np.asarray(batch["tokens"])


def forward_loss(module, state: dict, key, batch: dict, *, device=None, precision: str | None = None):
    """The reference's ``invoke`` result (loss, OutputCollection) computed on the GPU."""
    eng = _engine(module, device, precision)
    eng.load_state(state)
    return eng.loss(_tokens(batch), key=key, collection=True)


def train_step(module, state: dict, opt_state: dict | None, key, batch: dict, *, device=None,
               precision: str | None = None, return_grads: bool = False):
    """One forward + backward + AdamW step (the Trainer's ``learner`` hyperparameters).

    Returns ``(loss, summaries, new_state, new_opt_state)`` — plus ``grads`` (the full
    gradient tree) when ``return_grads`` — with the reference's tree layout; ``summaries`` is
    the flat ``{path/name: [values]}`` view of the step's OutputCollection.
    """
    eng = _engine(module, device, precision)
    eng.load_state(state)
    eng.load_opt_state(opt_state)
    loss, col = eng.compute_grads(_tokens(batch), key=key)
    grads = eng.grads_numpy() if return_grads else None
    eng.apply_update()
    out = (float(loss.item()), col.flat_summaries(), eng.state_numpy(), eng.opt_state_numpy())
    return out + (grads,) if return_grads else out
