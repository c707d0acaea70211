"""Attention policies: PolicyConfig / ForcedAdmission (engine.hpp:17-40) and
Session::effective_gate (engine.cpp:126-151), mirrored from the C++ face
(include/wgkv_b200.hpp).  A policy other than the learned gate reaches the
device as the ``forced_gates`` argument of ``Session.prefill_layer`` /
``decode_layer`` / ``gate_forward_batch``; ``policy_gates`` builds it.
"""
from dataclasses import dataclass, field

import numpy as np

KINDS = ("full", "wgkv", "local_sink", "static_heads", "wgkv_plus_topk")  # PolicyKind order (engine.hpp:17)
MODES = ("none", "stride", "recent_fraction")                               # ForcedAdmission::Mode


@dataclass
class ForcedAdmission:
    mode: str = "none"
    keep_every: int = 4      # stride: admit positions with pos % keep_every == phase
    phase: int = 0
    fraction: float = 0.25   # recent_fraction: newest fraction of the pre-window prompt


@dataclass
class Policy:
    kind: str = "wgkv"
    window: int = 256
    sink: int = 128
    retrieval_bitmap: list = field(default_factory=list)  # static_heads: layers * kv_heads entries
    topk_budget: int = 0
    forced: ForcedAdmission = field(default_factory=ForcedAdmission)

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown policy: {self.kind}")
        if self.forced.mode not in MODES:
            raise ValueError(f"unknown forced admission mode: {self.forced.mode}")


def uses_mlp_gates(p: Policy) -> bool:
    """engine.cpp:203: the gate MLP decides (pass forced_gates=None)."""
    return p.kind in ("wgkv", "wgkv_plus_topk") and p.forced.mode == "none"


def effective_gates(p: Policy, layer: int, head: int, kv_heads: int, positions, prompt_len: int) -> np.ndarray:
    """Vectorised Session::effective_gate for one (layer, global kv head)."""
    pos = np.asarray(positions, dtype=np.int64)
    if p.kind == "full":
        return np.ones(pos.shape)
    if p.kind == "local_sink":
        return (pos < p.sink).astype(np.float64)
    if p.kind == "static_heads":
        return np.full(pos.shape, 1.0 if p.retrieval_bitmap[layer * kv_heads + head] else 0.0)
    if p.forced.mode == "stride":
        return (pos % p.forced.keep_every == p.forced.phase).astype(np.float64)
    if p.forced.mode == "recent_fraction":
        pre_window = max(0, prompt_len - p.window)
        x = p.forced.fraction * pre_window  # std::llround: half away from zero
        cutoff = pre_window - int(np.floor(x + 0.5) if x >= 0 else np.ceil(x - 0.5))
        return (pos >= cutoff).astype(np.float64)
    raise RuntimeError("effective_gate: the gate MLP decides under this policy")


def policy_gates(p: Policy, layer: int, kv_head_offset: int, kv_heads_local: int, kv_heads_total: int,
                 nseq: int, pos0: int, T: int, prompt_len: int):
    """forced_gates [nseq][kv_heads_local][T] (float32) or None when the MLP decides."""
    if uses_mlp_gates(p):
        return None
    pos = np.arange(pos0, pos0 + T)
    one = np.stack([effective_gates(p, layer, kv_head_offset + h, kv_heads_total, pos, prompt_len)
                    for h in range(kv_heads_local)])
    return np.broadcast_to(one, (nseq, kv_heads_local, T)).astype(np.float32)
