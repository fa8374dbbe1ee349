"""Remat policy resolution (reference mesh.py:204-252), executed by TransformerLayer.

A policy maps remat-tag patterns to a decision: "save", "recompute" or "offload". An
exact tag key beats glob keys; among globs the longest pattern wins; unmatched tags are
saved.  Named aliases are the reference's.  On the GPU a layer block (norm + attention,
or norm + feed-forward) is rematerialised when any of its tags resolves to "recompute":
its forward runs without saving activations and its backward re-runs it first.
"offload" is executed as "save" (no host offload on this path).
"""

from __future__ import annotations

import fnmatch
from typing import Mapping

from .errors import TypeMismatchError

SAVE, RECOMPUTE, OFFLOAD = "save", "recompute", "offload"
DECISIONS = (SAVE, RECOMPUTE, OFFLOAD)

POLICY_ALIASES: dict[str, dict[str, str]] = {
    "save_all": {},
    "recompute_all": {"*": RECOMPUTE},
    "offload_dots": {"*": OFFLOAD},
    "save_qkvo_flash": {"q_proj": SAVE, "k_proj": SAVE, "v_proj": SAVE, "o_proj": SAVE, "context": SAVE,
                        "*": RECOMPUTE},
}


def resolve_policy(policy) -> dict[str, str]:
    if isinstance(policy, str):
        if policy not in POLICY_ALIASES:
            raise TypeMismatchError(f"unknown remat policy alias {policy!r}")
        return dict(POLICY_ALIASES[policy])
    out = {}
    for tag, decision in dict(policy).items():
        if decision not in DECISIONS:
            raise TypeMismatchError(f"unknown remat decision {decision!r} for tag {tag!r}")
        out[tag] = decision
    return out


def decide_tag(tag: str, policy: Mapping[str, str]) -> str:
    if tag in policy:
        return policy[tag]
    globs = [p for p in policy if ("*" in p or "?" in p) and fnmatch.fnmatchcase(tag, p)]
    if globs:
        globs.sort(key=lambda p: (-len(p), p))
        return policy[globs[0]]
    return SAVE
