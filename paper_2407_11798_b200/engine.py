"""Pipeline orchestration (placeholder while the engine is being ported)."""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from .errors import EngineError


def plan_layer_split(n_layers: int, n_nodes: int,
                     node_speed_weights: Optional[Sequence[float]] = None
                     ) -> List[Tuple[int, int]]:
    """Contiguous per-stage layer ranges proportional to speed weights
    (engine.py:186-224): floor of the exact share, remainder to the earliest
    stages, every stage at least one layer."""
    if n_nodes < 1:
        raise EngineError("need at least one node")
    if n_layers < n_nodes:
        raise EngineError(f"{n_layers} layers cannot cover {n_nodes} nodes")
    if node_speed_weights is None:
        w = [1.0] * n_nodes
    else:
        w = [float(x) for x in node_speed_weights]
        if len(w) != n_nodes:
            raise EngineError("need one speed weight per node")
        if any(x <= 0 for x in w):
            raise EngineError("speed weights must be positive")
    tot = sum(w)
    sizes = [int(n_layers * x / tot) for x in w]
    i = 0
    while sum(sizes) < n_layers and i < n_nodes:
        sizes[i] += 1
        i += 1
    if sum(sizes) != n_layers:
        raise EngineError("layer split does not cover the model")
    if min(sizes) < 1:
        raise EngineError("weights leave some node without a layer")
    out, lo = [], 0
    for s in sizes:
        out.append((lo, lo + s))
        lo += s
    return out


def token_checksum(tokens: Sequence) -> str:
    return hashlib.sha256(",".join(str(t) for t in tokens).encode()).hexdigest()


@dataclass
class RunRecord:
    run_id: int
    kind: str
    tokens: tuple
    min_pos: int
    max_pos: int
    seq_id: int
    logit_slots: Dict[int, int]
    basis: tuple = ()
    status: str = "in-flight"
    launch_time: float = 0.0
    judged: int = 0

    def chain(self):
        for pos, tok in self.basis:
            yield pos, tok
        for i, tok in enumerate(self.tokens):
            yield self.min_pos + i, tok


@dataclass
class ExperimentConfig:
    pass


@dataclass
class RunMetrics:
    pass


@dataclass
class SimResult:
    pass


def simulate(cfg, **kw):
    raise NotImplementedError


def generate(*a, **kw):
    raise NotImplementedError
