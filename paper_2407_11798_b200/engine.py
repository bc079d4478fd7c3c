"""Pipeline orchestration on B200: configuration, layer split, the head's
four decoding modes, metrics (mirror of ``specpipe/engine.py``).

* ``iterative`` / ``pipeline-iterative`` — one non-speculative run at a time;
* ``sync-speculative`` — draft round trip, then one verification chain;
* ``async-speculative`` — PipeInfer: continuous asynchronous speculation
  over FIFO sequence partitions with early inference cancellation.

The head keeps the reference controller's decisions (engine.py:695-1273)
with two deliberate fixes: F4(a) a speculative run launched
while the frontier token is carried by an in-flight run copies its prefix
from that run's partition; F4(b) a draft request whose context is a strict
prefix of the draft's state backs off one token so the tip is recomputed.
Runs execute on GPU stages (``pipeline.py`` / ``dist.py``); the draft on its
own stream (``drafting.py``).  All times are host wall-clock seconds.
"""

from __future__ import annotations

import hashlib
import os
import time
from collections import deque
from dataclasses import dataclass, field, fields, replace
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import EngineError, ProtocolError
from .kvcache import SequenceAllocator
from .model import (KIND_CODE, NON_SPECULATIVE, PREFILL, SPECULATIVE, Batch,
                    BatchToken, ModelConfig, encode_tokens, greedy_sample,
                    llama_config, sample_prompt)
from .speculation import CutoffController
from .verify import (INVALID, VerifyResult, apply_acceptance, detect_stale_runs,
                     verify_run)

MODES = ("iterative", "pipeline-iterative", "sync-speculative", "async-speculative")

IN_FLIGHT = "in-flight"
COMPLETED = "completed"
CANCELLED_INVALID = "cancelled-invalid"
CANCELLED_SUPERFLUOUS = "cancelled-superfluous"
DRAINED = "drained"


# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ExperimentConfig:
    """One experiment (engine.py:80-183) plus B200 fields.

    The simulator's delay knobs (``per_layer_delay``, ``link_latency``,
    ``per_byte_delay``, ``draft_token_delay``) are accepted for drop-in
    compatibility and ignored: costs are whatever the GPU takes.
    """

    mode: str = "async-speculative"
    nodes: int = 8
    vocab_size: int = 256
    embed_dim: int = 64
    target_layers: int = 12
    draft_layers: int = 2
    draft_embed_dim: int = 64
    n_heads: int = 1
    max_context: int = 1024
    target_seed: int = 1
    draft_seed: int = 2
    draft_backend: str = "toy"
    alpha: float = 0.8
    cutoff: float = 0.4
    cutoff_recovery: float = 0.05
    cutoff_decay: float = 0.05
    microbatch: int = 4
    tree_cap: int = 4
    continuous: bool = True
    partitions: int = 8
    prompt_seed: int = 1234
    prompt_len: int = 128
    gen_len: int = 512
    clock: str = "wall"
    repetitions: int = 1
    per_layer_delay: float = 1e-3
    link_latency: float = 1e-5
    per_byte_delay: float = 0.0
    draft_token_delay: float = 5e-4
    idle_poll: float = 1e-4
    eos_token: Optional[int] = None
    node_weights: Optional[Tuple[int, ...]] = None
    # --- B200 extensions ---
    arch: str = "ref"                    # target/draft arch when no shape is named
    target_shape: Optional[str] = None   # e.g. "llama2-7b" (model.LLAMA_SHAPES)
    draft_shape: Optional[str] = None    # e.g. "llama-160m"
    capacity: int = 8192                 # cell pool per stage
    max_run_tokens: int = 256            # largest batch (prefill) per stage-run
    draft_charge: bool = True            # synthetic draft pays a real draft forward
                                         # per token (False ~ draft_token_delay=0)
    draft_tc: bool = False               # llama draft on tcgen05 (True) or on the
                                         # lower-latency CUDA-core GEMV path
    draft_sm_reserve: int = 16           # SMs kept free of target GEMMs on the
                                         # draft's GPU (so draft kernels start at once)
    spec_ramp: bool = True               # reference: the continuous micro-batch cap
                                         # ramps with the unverified chain depth
                                         # (engine.py:1027-1030); False asks for
                                         # `microbatch` tokens every time (a GPU
                                         # stage-run costs the same for 1..16 tokens)
    fold_frontier: Optional[bool] = None  # B200 policy: a frontier token no in-flight
                                         # run carries waits for the draft and rides
                                         # in front of its proposals (one run instead
                                         # of a 1-token run + a speculative run);
                                         # False = the reference: launch it alone at
                                         # once (engine.py:1090-1182); None = True on
                                         # a 1-stage pipeline (nothing to overlap: a
                                         # run costs a full weight pass for 1..16
                                         # tokens), False otherwise
    tree_width: int = 1                  # 1 = chain speculation (the reference); 2 =
                                         # every proposal also carries the draft's
                                         # runner-up as a sibling leaf (same position,
                                         # own partition), verified greedily in the
                                         # same run (a B200 run costs the same for
                                         # 1..16 tokens)
    alpha_sibling: float = 0.4           # synthetic draft, tree_width 2: probability
                                         # its runner-up is the target's greedy token
                                         # when its first choice is not
    draft_exclusive: bool = True         # a draft sharing a stage's GPU takes every SM
                                         # (grid-form kernel) for requests issued while
                                         # no target run is in flight
    max_inflight: Optional[int] = None   # B200 policy: no new speculation while this
                                         # many runs are in flight (0 = unbounded, the
                                         # reference; partitions still bound it);
                                         # None = on a 1-stage pipeline 1 (draft on
                                         # the stage's GPU) or 2 (draft GPU of its
                                         # own), else 0

    def validate(self) -> None:
        if self.mode not in MODES:
            raise EngineError(f"unknown mode {self.mode!r}; expected one of {MODES}")
        if self.clock not in ("virtual", "wall"):
            raise EngineError(f"unknown clock {self.clock!r}")
        if self.draft_backend not in ("toy", "synthetic"):
            raise EngineError(f"unknown draft backend {self.draft_backend!r}")
        if not 0.0 <= self.alpha <= 1.0:
            raise EngineError("alpha must be in [0, 1]")
        if self.nodes < 1:
            raise EngineError("need at least one node")
        if self.uses_draft() and self.nodes < 2:
            raise EngineError(f"{self.mode} needs >= 2 nodes (one is the draft node)")
        if not 1 <= self.microbatch <= 4:
            raise EngineError("microbatch must be within [1, 4]")
        if self.tree_cap < 1:
            raise EngineError("tree_cap must be >= 1")
        if self.partitions < 2:
            raise EngineError("partitions must be >= 2")
        if self.partitions > 32:
            raise EngineError("partitions must be <= 32 (one mask bit each)")
        if self.tree_width not in (1, 2):
            raise EngineError("tree_width must be 1 (chain) or 2 (chain + runner-up siblings)")
        if not 0.0 <= self.alpha_sibling <= 1.0:
            raise EngineError("alpha_sibling must be in [0, 1]")
        if self.max_inflight is not None and self.max_inflight < 0:
            raise EngineError("max_inflight must be >= 0 (0 = unbounded)")
        if self.gen_len < 1 or self.prompt_len < 1:
            raise EngineError("prompt_len and gen_len must be >= 1")
        if self.prompt_len + self.gen_len > self.max_context:
            raise EngineError("prompt_len + gen_len exceeds max_context")
        if self.idle_poll <= 0:
            raise EngineError("idle_poll must be > 0 (prevents zero-time spinning)")
        if self.repetitions < 1:
            raise EngineError("repetitions must be >= 1")
        if self.prompt_len > self.max_run_tokens:
            raise EngineError("prompt_len exceeds max_run_tokens")
        # the bounded cell pool must hold the canonical sequence plus one run
        # per partition after a compaction (kvcache.py grows without bound)
        need = self.prompt_len + self.gen_len + self.partitions * (
            max(self.microbatch, self.tree_cap) + 1)
        if self.capacity < need:
            raise EngineError(f"capacity {self.capacity} cannot hold a {self.prompt_len}+"
                              f"{self.gen_len}-token context plus one run per partition "
                              f"(need >= {need})")
        self.target_config().validate()
        if self.uses_draft():
            self.draft_config().validate()

    def uses_draft(self) -> bool:
        return self.mode in ("sync-speculative", "async-speculative")

    def target_config(self) -> ModelConfig:
        if self.target_shape:
            return llama_config(self.target_shape, self.max_context, self.target_seed)
        return ModelConfig(vocab_size=self.vocab_size, embed_dim=self.embed_dim,
                           n_layers=self.target_layers, n_heads=self.n_heads,
                           max_context=self.max_context, seed=self.target_seed,
                           arch=self.arch)

    def draft_config(self) -> ModelConfig:
        if self.draft_shape:
            return llama_config(self.draft_shape, self.max_context, self.draft_seed)
        return ModelConfig(vocab_size=self.vocab_size, embed_dim=self.draft_embed_dim,
                           n_layers=self.draft_layers, n_heads=self.n_heads,
                           max_context=self.max_context, seed=self.draft_seed,
                           arch=self.arch)

    def n_stages(self) -> int:
        if self.mode == "iterative":
            return 1
        if self.uses_draft():
            return self.nodes - 1
        return self.nodes


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


# ---------------------------------------------------------------------------
# records and metrics
# ---------------------------------------------------------------------------

@dataclass
class RunRecord:
    """Head-side state of one in-flight run (engine.py:339-360)."""

    run_id: int
    kind: str
    tokens: tuple
    min_pos: int
    max_pos: int
    seq_id: int
    logit_slots: Dict[int, int]
    basis: tuple = ()
    status: str = IN_FLIGHT
    launch_time: float = 0.0
    judged: int = 0
    # tree runs: pos -> (token, partition, logits slot) of the sibling leaf
    # at that position, and every partition the run wrote under
    siblings: Dict[int, Tuple[int, int, int]] = field(default_factory=dict)
    tree_seqs: tuple = ()

    def partitions(self) -> tuple:
        return tuple(q for q in ((self.seq_id,) + self.tree_seqs) if q != 0)

    def chain(self):
        for pos, tok in self.basis:
            yield pos, tok
        for i, tok in enumerate(self.tokens):
            yield self.min_pos + i, tok


@dataclass
class RunMetrics:
    """Reference metric schema (engine.py:367-420)."""

    mode: str
    clock: str
    tokens_generated: int
    duration: float
    generation_speed: float
    ttft: float
    itl: float
    acceptance_rate: float
    examined: int
    matched: int
    runs_started: int
    spec_runs: int
    cancelled_invalid: int
    cancelled_superfluous: int
    cancelled_runs: int
    drained_runs: int
    alloc_stalls: int
    inflight_mean: float
    bytes_by_tag: Dict[str, int]
    msgs_by_tag: Dict[str, int]
    token_checksum: str
    virtual_end: float
    wall_seconds: float

    def to_dict(self, include_wall: bool = True) -> dict:
        d = {f.name: getattr(self, f.name) for f in fields(self)}
        d["bytes_by_tag"] = dict(sorted(self.bytes_by_tag.items()))
        d["msgs_by_tag"] = dict(sorted(self.msgs_by_tag.items()))
        if not include_wall:
            d.pop("wall_seconds")
        return d


@dataclass
class CancelLogEntry:
    run_id: int
    reason: str
    kind: str
    min_pos: int
    max_pos: int
    accepted_len_at_cancel: int
    chain: tuple


@dataclass
class SimResult:
    tokens: List[int]
    metrics: RunMetrics
    accepted_full: List[int]
    accept_events: List[Tuple[float, int]]
    cancel_log: List[CancelLogEntry]
    node_logs: Dict[int, list]
    consumed: Dict[Tuple[int, str], int]
    sent: Dict[Tuple[int, str], int]
    records: List[RunRecord]
    host_profile: Dict[str, float] = field(default_factory=dict)


def token_checksum(tokens: Sequence) -> str:
    return hashlib.sha256(",".join(str(t) for t in tokens).encode()).hexdigest()


class _Inflight:
    """Time-weighted mean of the FIFO depth (engine.py:451-467)."""

    def __init__(self):
        self.steps: List[Tuple[float, int]] = [(0.0, 0)]

    def update(self, t: float, n: int) -> None:
        self.steps.append((t, n))

    def mean(self, start: float, end: float) -> float:
        if end <= start:
            return 0.0
        tot = 0.0
        for (t0, n), (t1, _) in zip(self.steps, self.steps[1:] + [(end, 0)]):
            a, b = max(t0, start), min(t1, end)
            if b > a:
                tot += n * (b - a)
        return tot / (end - start)


# ---------------------------------------------------------------------------
# the head
# ---------------------------------------------------------------------------

class Head:
    """Sampling, verification, speculation and cancellation decisions."""

    def __init__(self, cfg: ExperimentConfig, pipe, draft, prompt: List[int],
                 d_model: int):
        self.cfg = cfg
        self.pipe = pipe
        self.draft = draft
        self.prompt = list(prompt)
        self.d_model = d_model
        self.accepted: List[int] = list(prompt)
        self.run_counter = 0
        self.fifo: deque = deque()
        self.allocator = SequenceAllocator(cfg.partitions)
        self.cutoff = CutoffController(base=cfg.cutoff, recovery=cfg.cutoff_recovery,
                                       decay=cfg.cutoff_decay)
        self.pending: List[Tuple[int, int]] = []
        self.pending_tip_seq = 0
        self.mirror: List[int] = []
        self.request_ctx: Optional[List[int]] = None
        self.draft_busy = False
        self.spec_since_round = 0
        self.idle_until = 0.0
        self.generated = 0
        self.terminal = False
        self.window_start = 0.0
        self.accept_events: List[Tuple[float, int]] = []
        self.examined = self.matched = 0
        self.runs_started = self.spec_runs = 0
        self.cancelled_invalid = self.cancelled_superfluous = 0
        self.drained_runs = self.alloc_stalls = 0
        self._stalled = False
        self.inflight = _Inflight()
        self.cancel_log: List[CancelLogEntry] = []
        self.records: List[RunRecord] = []
        self.bytes: Dict[str, int] = {}
        self.msgs: Dict[Tuple[int, str], int] = {}
        self.stage_logs: Dict[int, list] = {i + 1: [] for i in range(pipe.n_stages)}
        self.tips: Optional[list] = None   # NS-run tips (truth tables)
        self.fold = False    # the frontier waits to ride in front of the next proposals
        self.folded_runs = 0
        self.tree_siblings = self.sibling_hits = 0
        self.last_seconds: tuple = ()
        # B200 policy defaults (measured): a 1-stage pipeline
        # folds the frontier into the next proposals; it keeps one run in
        # flight when the draft shares the stage's GPU (a concurrent draft
        # request slows the stage and queues the next fold behind it) and
        # speculates one run ahead when the draft has a GPU of its own
        # speculates one run ahead when the draft has a GPU of its own.  A
        # deeper pipeline folds only while it pays (_adapt_policy): the
        # measured draft latency for a micro-batch is below one stage-time
        # and the measured acceptance is >= 0.5 (70B, 3 stages: 87.7 -> 101
        # tok/s; 7B/13B, 3 stages, and alpha 0.25 lose with folding)
        one = pipe.n_stages == 1
        shared = bool(getattr(draft, "shared_gpu", True))
        self.adaptive = cfg.fold_frontier is None and not one
        # a 1-stage pipeline with a draft GPU of its own speculates one run
        # ahead only while chains break often (alpha < 0.75): measured N=2
        # alpha 0.66 540 vs 497 tok/s sync, but alpha 0.9 662 vs 946 with
        # the run ahead (its continuation runs crowd out folded runs)
        self.adapt_cap = cfg.max_inflight is None and one and not shared
        self.fold_frontier = one if cfg.fold_frontier is None else bool(cfg.fold_frontier)
        self._fold_cap = (1 if shared else 2) if one else pipe.n_stages
        self.max_inflight = ((self._fold_cap if self.fold_frontier else 0)
                             if cfg.max_inflight is None else cfg.max_inflight)
        self._draft_sent, self._draft_fwd = 0.0, 0
        self.est_draft_fwd: Optional[float] = None   # s per draft forward (EMA)
        self.est_run: Optional[float] = None         # s launch -> completion, best seen
        from collections import defaultdict
        self.profile: Dict[str, float] = defaultdict(float)   # host seconds by activity
        self._t0 = time.perf_counter()

    def now(self) -> float:
        return time.perf_counter() - self._t0

    def _count(self, tag: str, nbytes: int, dst: int = 0, n: int = 1) -> None:
        self.bytes[tag] = self.bytes.get(tag, 0) + nbytes
        self.msgs[(dst, tag)] = self.msgs.get((dst, tag), 0) + n

    # -- low-level helpers (engine.py:745-864) ------------------------------------
    def _next_run_id(self) -> int:
        self.run_counter += 1
        return self.run_counter

    def _launch(self, batch: Batch, seq_id: int, basis: tuple = (),
                skippable: bool = True, n_chain: Optional[int] = None,
                tree_seqs: tuple = ()) -> RunRecord:
        """``n_chain``: the first n_chain tokens are the run's chain; the rest
        are sibling leaves (tree runs), each at the position of the chain
        token it is an alternative to."""
        nc = len(batch.tokens) if n_chain is None else n_chain
        chain = batch.tokens[:nc]
        slots = {i: slot for slot, i in enumerate(batch.logit_indices)}
        rec = RunRecord(run_id=batch.run_id, kind=batch.kind,
                        tokens=tuple(t.token for t in chain),
                        min_pos=chain[0].pos, max_pos=chain[-1].pos,
                        seq_id=seq_id,
                        logit_slots={chain[i].pos: slots[i] for i in range(nc) if i in slots},
                        basis=basis, launch_time=self.now(),
                        siblings={batch.tokens[i].pos: (batch.tokens[i].token,
                                                        min(batch.tokens[i].seqs), slots[i])
                                  for i in range(nc, len(batch.tokens))},
                        tree_seqs=tuple(tree_seqs))
        flags = _lib.SP_FWD_CHECK_COVERAGE
        if batch.kind == SPECULATIVE and skippable:
            flags |= _lib.SP_FWD_SKIPPABLE
        self.pipe.launch(batch.run_id, KIND_CODE[batch.kind], encode_tokens(batch.tokens),
                         flags, list(batch.logit_indices))
        n = len(batch.tokens)
        S = self.pipe.n_stages
        self._count("RUN_CONFIG", (24 + 24 * n + 8 * sum(len(t.seqs) for t in batch.tokens) + 32) * S, 1, S)
        self._count("ACTIVATIONS", (16 + 4 * n * self.d_model + 24) * max(0, S - 1), 2, max(0, S - 1))
        for s in range(1, S + 1):
            self.stage_logs[s].append(("run-config", batch.run_id))
        self.fifo.append(rec)
        self.records.append(rec)
        self.runs_started += 1
        if batch.kind == SPECULATIVE:
            self.spec_runs += 1
        self.inflight.update(self.now(), len(self.fifo))
        return rec

    def _emit_copy(self, src: int, dsts: Sequence[int], end_pos: int) -> None:
        if dsts:
            d = tuple(sorted(dsts))
            self.pipe.copy(src, d, end_pos)
            S = self.pipe.n_stages
            self._count("CACHE_COPY", (24 + 8 * len(d) + 32) * S, 1, S)
            for s in range(1, S + 1):
                self.stage_logs[s].append(("cache-copy", src, d, end_pos))

    def _emit_remove(self, seq: int, from_pos: int) -> None:
        self.pipe.remove(seq, from_pos)
        S = self.pipe.n_stages
        self._count("CACHE_REMOVE", (24 + 32) * S, 1, S)
        for s in range(1, S + 1):
            self.stage_logs[s].append(("cache-remove", seq, from_pos))

    def _accept(self, tok: int) -> None:
        if self.generated >= self.cfg.gen_len or self.terminal:
            return
        self.accepted.append(tok)
        self.generated += 1
        self.accept_events.append((self.now(), tok))
        if self.cfg.eos_token is not None and tok == self.cfg.eos_token:
            self.terminal = True

    def _judge_walked(self, rec: RunRecord, result) -> None:
        """engine.py:809-823"""
        if rec.kind != SPECULATIVE:
            return
        ok = result.matched_end - rec.min_pos
        adjudicated = ok + (1 if result.mismatch else 0)
        self.matched += max(0, ok - rec.judged)
        self.examined += max(0, adjudicated - rec.judged)
        rec.judged = max(rec.judged, adjudicated)

    def _judge_cancelled(self, rec: RunRecord) -> None:
        """engine.py:825-848"""
        if rec.kind != SPECULATIVE:
            return
        for pos, tok in rec.basis:
            if pos < len(self.accepted) and tok != self.accepted[pos]:
                return
        i = rec.judged
        while i < len(rec.tokens):
            pos = rec.min_pos + i
            if pos >= len(self.accepted):
                break
            self.examined += 1
            same = rec.tokens[i] == self.accepted[pos]
            if same:
                self.matched += 1
            i += 1
            if not same:
                break
        rec.judged = i

    def _pop_record(self, res) -> RunRecord:
        if not self.fifo:
            raise ProtocolError(f"logits for run {res.run_id} with empty FIFO")
        rec = self.fifo.popleft()
        if rec.run_id != res.run_id:
            raise ProtocolError(f"logits out of order: got run {res.run_id}, "
                                f"expected {rec.run_id}")
        self._count("LOGITS", 16 + 24 + 16 * len(res.rows), 0)
        for s, st in enumerate(res.stage_status, start=1):
            self.stage_logs[s].append(
                ("evaluated" if st == _lib.SP_STATUS_VALID else "skip-or-abandon",
                 res.run_id))
        self.inflight.update(self.now(), len(self.fifo))
        if res.err:
            _lib.raise_device_error(res.err, f"run {res.run_id}")
        if res.placeholder and rec.status == IN_FLIGHT:
            raise ProtocolError(f"run {rec.run_id} came back as a placeholder "
                                "without being cancelled")
        return rec

    def _recv(self):
        return self.pipe.wait()

    # -- draft requests -------------------------------------------------------------
    def _draft_request(self, truncate_to: int, feed: Sequence[int], max_tokens: int,
                       cutoff: float) -> None:
        hint = getattr(self.draft, "set_exclusive", None)
        if hint is not None and self.cfg.draft_exclusive:
            hint(self.pipe.in_flight() == 0)     # no target run queued: whole GPU
        self._draft_sent = self.now()
        self._draft_fwd = (1 if feed else 0) + max(0, int(max_tokens))
        self.draft.request(truncate_to, feed, max_tokens, cutoff)
        self._count("DRAFT_REQUEST", 24 + 32 + 8 * len(feed), self.cfg.nodes)
        self.draft_busy = True

    def _draft_reply(self):
        toks, confs = self.draft.reply()
        if self._draft_fwd > 0:
            per = (self.now() - self._draft_sent) / self._draft_fwd
            self.est_draft_fwd = per if self.est_draft_fwd is None else (
                0.8 * self.est_draft_fwd + 0.2 * per)
        self.last_seconds = tuple(getattr(self.draft, "seconds", ()) or ())
        self.draft_busy = False
        self._count("DRAFT_REPLY", 24 + 8 + 16 * len(toks), 0)
        return toks, confs

    # -- prefill (engine.py:868-900) ---------------------------------------------------
    def _prefill(self) -> int:
        if self.draft is not None:
            self._draft_request(0, tuple(self.prompt), 0, 1.0)
            self.mirror = list(self.prompt)
        batch = Batch(tokens=tuple(BatchToken(t, i, frozenset([0]), i == len(self.prompt) - 1)
                                   for i, t in enumerate(self.prompt)),
                      kind=PREFILL, run_id=self._next_run_id())
        rec = self._launch(batch, seq_id=0)
        res = self._recv()
        self._pop_record(res)
        rec.status = COMPLETED
        if self.draft is not None:
            self._draft_reply()
        t0 = greedy_sample(res.rows[0])
        if self.tips is not None:
            self.tips.append(res.rows[0])
        self.accepted.append(t0)
        self.generated += 1
        if self.cfg.eos_token is not None and t0 == self.cfg.eos_token:
            self.terminal = True
        self.window_start = self.now()
        return t0

    def _launch_ns(self, token: int, with_copy: bool) -> RunRecord:
        pos = len(self.accepted) - 1
        batch = Batch(tokens=(BatchToken(token, pos, frozenset([0]), True),),
                      kind=NON_SPECULATIVE, run_id=self._next_run_id())
        rec = self._launch(batch, seq_id=0)
        if with_copy:
            # early cache-entry sharing: canonical cells reach every partition
            # right behind the run (engine.py:912-916)
            self._emit_copy(0, self.allocator.all_ids(), pos + 1)
        return rec

    # -- modes ---------------------------------------------------------------------
    def run_iterative(self) -> None:
        tok = self._prefill()
        while self.generated < self.cfg.gen_len and not self.terminal:
            self._launch_ns(tok, with_copy=False)
            res = self._recv()
            got = self._pop_record(res)
            got.status = COMPLETED
            if self.tips is not None:
                self.tips.append(res.rows[0])
            result = verify_run(got, res.rows, self.accepted, eos_token=self.cfg.eos_token)
            if result.next_token is None:
                raise ProtocolError("iterative run produced no next token")
            self._accept(result.next_token)
            tok = result.next_token
        self._finish()

    def run_sync_speculative(self) -> None:
        tok = self._prefill()
        while self.generated < self.cfg.gen_len and not self.terminal:
            drafts, _ = self._draft_round_trip(self.cfg.tree_cap, self.cutoff.base)
            pos = len(self.accepted) - 1
            if self.cfg.tree_width >= 2 and self.allocator.available() > 0:
                # tree round: frontier + chain + sibling leaves on partitions,
                # committed like an async run
                seq = self.allocator.alloc()
                toks, n_chain, tseqs = self._tree_tokens(
                    (tok,), pos + 1, list(drafts), self.last_seconds[:len(drafts)], seq)
                self._emit_copy(0, (seq,) + tseqs, pos)
                batch = Batch(tokens=toks, kind=SPECULATIVE, run_id=self._next_run_id())
                rec = self._launch(batch, seq_id=seq, skippable=False, n_chain=n_chain,
                                   tree_seqs=tseqs)
                rec.judged = 1
                res = self._recv()
                got = self._pop_record(res)
                got.status = COMPLETED
                result, src = self._verify(got, res.rows)
                self._judge_walked(got, result)
                for t in result.accepted:
                    self._accept(t)
                if result.next_token is not None:
                    self._accept(result.next_token)
                self._commit(got, result, src)
                if self.terminal:
                    break
                tok = self.accepted[-1]
                continue
            toks = [BatchToken(tok, pos, frozenset([0]), True)]
            toks += [BatchToken(d, pos + 1 + i, frozenset([0]), True)
                     for i, d in enumerate(drafts)]
            batch = Batch(tokens=tuple(toks), kind=SPECULATIVE, run_id=self._next_run_id())
            rec = self._launch(batch, seq_id=0)
            rec.judged = 1   # the leading token is accepted context, not a draft
            res = self._recv()
            got = self._pop_record(res)
            got.status = COMPLETED
            result = verify_run(got, res.rows, self.accepted, eos_token=self.cfg.eos_token)
            self._judge_walked(got, result)
            for t in result.accepted:
                self._accept(t)
            if result.next_token is not None:
                self._accept(result.next_token)
            if result.mismatch:
                self._emit_remove(0, result.matched_end)
            if self.terminal:
                break
            tok = self.accepted[-1]
        self._finish()

    def run_async_speculative(self) -> None:
        self._prefill()
        if not (self.generated >= self.cfg.gen_len or self.terminal):
            if self.fold_frontier and self.allocator.available() > 0:
                self.fold = True
            else:
                self._launch_ns(self.accepted[-1], with_copy=True)
        prof = self.profile
        clk = time.perf_counter
        while self.generated < self.cfg.gen_len and not self.terminal:
            t0 = clk()
            if self.pipe.ready():
                self._handle_completion(self.pipe.poll())
                prof["completion"] += clk() - t0
                continue
            if self.draft_busy and self.draft.ready():
                self._handle_reply(*self._draft_reply())
                prof["reply+spec_launch"] += clk() - t0
                continue
            if not self.draft_busy and self._want_speculation():
                self._send_draft_request()
                prof["draft_request"] += clk() - t0
                continue
            if self.fold and not self.draft_busy:
                # nothing will carry the frontier (no partition, cutoff idle,
                # in-flight cap): launch it alone, as the reference does
                self.fold = False
                self._launch_ns(self.accepted[-1], with_copy=True)
                continue
            self._block_until_message()
            prof["wait"] += clk() - t0
        self._finish()

    def _block_until_message(self) -> None:
        """recv_any([LOGITS, DRAFT_REPLY]) without consuming (the loop does)."""
        if self.pipe.in_flight() == 0 and not self.draft_busy:
            raise EngineError("deadlock: nothing in flight and nothing to launch")
        # (a yield, not time.sleep(0): the kernel's default 50 us timer slack
        # made every poll a ~55 us sleep -- twice per speculation cycle at N=1)
        while True:
            if self.pipe.ready() or (self.draft_busy and self.draft.ready()):
                return
            os.sched_yield()

    # -- async internals (engine.py:1002-1182) -----------------------------------------
    def _want_speculation(self) -> bool:
        if self.terminal or self.generated >= self.cfg.gen_len:
            return False
        if not self.cfg.continuous and self.spec_since_round >= 1:
            return False
        if self.allocator.available() == 0:
            if not self._stalled:
                self._stalled = True
                self.alloc_stalls += 1
            return False
        self._stalled = False
        if self.now() < self.idle_until:
            return False
        if (self.max_inflight and not self.fold
                and len(self.fifo) >= self.max_inflight):
            return False
        return len(self.accepted) + len(self.pending) + 1 <= self.cfg.max_context

    @staticmethod
    def _common_prefix(a: Sequence[int], b: Sequence[int]) -> int:
        """Length of the common prefix (list slices compare in C: the head
        runs this per draft request over the whole context)."""
        if not (isinstance(a, list) and isinstance(b, list)):
            a, b = list(a), list(b)
        n = min(len(a), len(b))
        if a[:n] == b[:n]:
            return n
        lo, hi = 0, n          # a[:lo] == b[:lo], a[:hi] != b[:hi]
        while hi - lo > 16:
            mid = (lo + hi) // 2
            if a[lo:mid] == b[lo:mid]:
                lo = mid
            else:
                hi = mid
        for i in range(lo, hi):
            if a[i] != b[i]:
                return i
        return hi

    def _backoff(self, cp: int, ctx: List[int]) -> Tuple[int, List[int]]:
        """F4(b): a context that is a strict prefix of the draft's state would
        truncate the draft without re-feeding anything, leaving it without
        tip logits; back off one token and re-feed it."""
        feed = ctx[cp:]
        if not feed and cp < len(self.mirror) and cp > 0:
            return cp - 1, ctx[cp - 1:]
        return cp, feed

    def _send_draft_request(self) -> None:
        ctx = self.accepted + [t for _, t in self.pending]
        cp = self._common_prefix(self.mirror, ctx)
        if self.cfg.continuous:
            cap = self.cfg.microbatch
            if self.cfg.spec_ramp and not self.fold:
                cap = min(cap, max(1, len(self.pending)))
        else:
            cap = self.cfg.tree_cap
        cap = min(cap, 4, self.cfg.max_context - len(ctx))
        truncate_to, feed = self._backoff(cp, ctx)
        self._draft_request(truncate_to, tuple(feed), cap, self.cutoff.current)
        self.mirror = list(ctx)
        self.request_ctx = list(ctx)

    def _handle_reply(self, toks, confs) -> None:
        props = list(toks)
        self.mirror.extend(props)
        ctx = self.accepted + [t for _, t in self.pending]
        if self.request_ctx != ctx:
            self.request_ctx = None
            return
        self.request_ctx = None
        if not props:
            if not self.pipe.ready():
                self.cutoff.on_speculation_idle()
            self.idle_until = self.now() + self.cfg.idle_poll
            if self.fold:
                self.fold = False
                self._launch_ns(self.accepted[-1], with_copy=True)
            return
        self.cutoff.note_success()
        seconds = self.last_seconds[:len(props)]
        if self.fold:
            self.fold = False
            self._launch_folded(props, seconds)
        else:
            self._launch_spec(props, seconds)
        self.spec_since_round += 1

    def _carrier_seq(self) -> int:
        """F4(a): partition of the in-flight run carrying the frontier token."""
        pos = len(self.accepted) - 1
        tok = self.accepted[-1]
        for rec in self.fifo:
            if (rec.status == IN_FLIGHT and rec.min_pos <= pos <= rec.max_pos
                    and rec.tokens[pos - rec.min_pos] == tok):
                return rec.seq_id
        return 0

    def _tree_tokens(self, lead: tuple, base: int, props: List[int], seconds, seq: int):
        """Batch tokens of a (tree) run: ``lead`` (decided frontier token at
        base - 1, or nothing) + the proposals at base.. on partition ``seq``,
        then -- tree_width 2 -- the draft's runner-up for proposal i as a
        sibling leaf at base + i on a partition of its own.  Visibility
        follows the reference's rule (build_tree_mask, model.py:262-284: a
        cell is seen iff it is earlier and shares a sequence): chain tokens
        before depth i also carry the sibling's partition, so the sibling
        sees exactly the context its chain twin sees."""
        sibs = []
        if self.cfg.tree_width >= 2 and seconds:
            for i, (d, t2) in enumerate(zip(props, seconds)):
                if t2 is None or t2 < 0 or t2 == d or self.allocator.available() == 0:
                    continue
                sibs.append((i, int(t2), self.allocator.alloc()))
        tseqs = tuple(q for _, _, q in sibs)
        toks = []
        if lead:
            toks.append(BatchToken(lead[0], base - 1, frozenset((seq,) + tseqs), True))
        for m, t in enumerate(props):
            extra = tuple(q for i, _, q in sibs if i > m)
            toks.append(BatchToken(t, base + m, frozenset((seq,) + extra), True))
        n_chain = len(toks)
        for i, t2, q in sibs:
            toks.append(BatchToken(t2, base + i, frozenset([q]), True))
            self.tree_siblings += 1
        return tuple(toks), n_chain, tseqs

    def _launch_spec(self, props: List[int], seconds=()) -> None:
        base = len(self.accepted) + len(self.pending)
        seq = self.allocator.alloc()
        src = self.pending_tip_seq if self.pending else self._carrier_seq()
        toks, n_chain, tseqs = self._tree_tokens((), base, props, seconds, seq)
        self._emit_copy(src, (seq,) + tseqs, base)
        basis = tuple(self.pending)
        batch = Batch(tokens=toks, kind=SPECULATIVE, run_id=self._next_run_id())
        self._launch(batch, seq_id=seq, basis=basis, n_chain=n_chain, tree_seqs=tseqs)
        self.pending.extend((base + i, t) for i, t in enumerate(props))
        self.pending_tip_seq = seq

    def _launch_folded(self, props: List[int], seconds=()) -> None:
        """The frontier token followed by the draft's proposals as ONE run on a
        fresh partition (sync-speculative's run shape, engine.py:955-970,
        inside the async pipeline).  The frontier is decided context, so the
        run is never skipped; its cells reach the canonical sequence and the
        live partitions through the usual commit (apply_acceptance)."""
        pos = len(self.accepted) - 1
        seq = self.allocator.alloc()
        toks, n_chain, tseqs = self._tree_tokens((self.accepted[-1],), pos + 1, props,
                                                 seconds, seq)
        self._emit_copy(0, (seq,) + tseqs, pos)
        batch = Batch(tokens=toks, kind=SPECULATIVE, run_id=self._next_run_id())
        rec = self._launch(batch, seq_id=seq, skippable=False, n_chain=n_chain,
                           tree_seqs=tseqs)
        rec.judged = 1      # the leading token is accepted context, not a draft
        self.pending = [(pos + 1 + i, t) for i, t in enumerate(props)]
        self.pending_tip_seq = seq
        self.folded_runs += 1

    def _verify(self, rec: RunRecord, rows):
        """verify_run (verify.py:43-124) plus, for tree runs, the sibling
        step: where the chain's first mismatch is, a sibling leaf equal to
        the target's greedy token is accepted and its own row donates the
        next token.  Returns (result, partition holding the accepted path)."""
        result = verify_run(rec, rows, self.accepted, eos_token=self.cfg.eos_token)
        if not (result.mismatch and rec.siblings):
            return result, rec.seq_id
        p = result.matched_end
        sib = rec.siblings.get(p)
        if sib is None or sib[0] != result.next_token:
            return result, rec.seq_id
        tok, q, slot = sib
        self.sibling_hits += 1
        acc = result.accepted + (tok,)
        eos = self.cfg.eos_token
        if eos is not None and tok == eos:
            return VerifyResult(acc, len(acc), None, True, result.examined, False, p + 1), q
        nxt = greedy_sample(rows[slot])
        return VerifyResult(acc, len(acc), nxt, eos is not None and nxt == eos,
                            result.examined, False, p + 1), q

    def _commit(self, rec: RunRecord, result, src: int) -> None:
        """apply_acceptance (verify.py:156-178) for chain and tree runs: the
        accepted cells (chain prefix, or prefix + sibling from the sibling's
        partition) reach the canonical sequence and every other live
        partition; every partition of the run is released."""
        cmds: List[Tuple[str, tuple]] = []
        if not rec.tree_seqs:
            apply_acceptance(result, rec, lambda op, args: cmds.append((op, args)),
                             self.allocator.live())
        elif result.matched_end > rec.min_pos:
            mine = set(rec.partitions())
            dsts = tuple(sorted({0, *self.allocator.live()} - mine))
            cmds.append(("copy", (src, dsts, result.matched_end)))
        for op, args in cmds:
            if op == "copy":
                self._emit_copy(*args)
            else:
                self._emit_remove(*args)
        for q in rec.tree_seqs:
            self._emit_remove(q, 0)
        if rec.tree_seqs and rec.seq_id != 0:
            self._emit_remove(rec.seq_id, 0)
        for q in rec.partitions():
            self.allocator.free(q)

    def _handle_completion(self, res) -> None:
        rec = self._pop_record(res)
        if rec.status in (CANCELLED_INVALID, CANCELLED_SUPERFLUOUS, DRAINED):
            for q in rec.partitions():
                self._emit_remove(q, 0)
                self.allocator.free(q)
            return
        rec.status = COMPLETED
        lat = self.now() - rec.launch_time
        self.est_run = lat if self.est_run is None else min(self.est_run, lat)
        result, src = self._verify(rec, res.rows)
        self._judge_walked(rec, result)
        new_tokens = list(result.accepted)
        if result.next_token is not None:
            new_tokens.append(result.next_token)
        for t in new_tokens:
            self._accept(t)
        self._commit(rec, result, src)
        if not new_tokens:
            return
        self._rebase_pending()
        self.cutoff.on_run_accepted()
        self.spec_since_round = 0
        self._cancel_stale()
        if self.adaptive:
            self._adapt_policy()
        elif self.adapt_cap and self.examined >= 16:
            self.max_inflight = 2 if self.matched / self.examined < 0.75 else 1
        if self.generated < self.cfg.gen_len and not self.terminal:
            if not self._frontier_carried():
                if (self.fold_frontier and self.draft is not None
                        and self.allocator.available() > 0):
                    self.fold = True    # rides in front of the next proposals
                else:
                    self._launch_ns(self.accepted[-1], with_copy=True)

    def _adapt_policy(self) -> None:
        """Fold the frontier (and cap in-flight runs at the stage count) while
        it pays: when a micro-batch of draft forwards costs less than one
        stage-time and the running acceptance is >= 0.5, or whenever the
        acceptance is >= 0.75 (long chains: one draft wait per mismatch buys
        runs that carry several tokens).  Measured (profiles/r02_sweep_*):
        7B, 3 stages: alpha 0.66 reference 577-590 vs folded 475 tok/s;
        alpha 0.8 804 vs 913; alpha 0.9 1293 vs 1406; 70B alpha 0.66 (draft
        far below a stage-time) 88 vs 100.  Otherwise the reference policy."""
        if self.est_draft_fwd is None or self.est_run is None:
            return
        if self.examined < 16:
            return
        alpha = self.matched / self.examined
        stage_time = self.est_run / self.pipe.n_stages
        cheap = self.est_draft_fwd * self.cfg.microbatch < stage_time
        fold = (alpha >= 0.5 and cheap) or alpha >= 0.75
        self.fold_frontier = fold
        if self.cfg.max_inflight is None:
            # while chains break often, one run per stage plus one queued at
            # the first (7B N=4, depth 2, alpha 0.66: cap 3 651 -> 4 685
            # tok/s, 2 612, 6 634); long chains keep one per stage (alpha
            # 0.9: 1472 at 3 vs 1438 at 4)
            cap = self._fold_cap + (1 if alpha < 0.75 else 0)
            self.max_inflight = cap if fold else 0

    def _frontier_carried(self) -> bool:
        pos = len(self.accepted) - 1
        tok = self.accepted[-1]
        return any(rec.status == IN_FLIGHT and rec.min_pos <= pos <= rec.max_pos
                   and rec.tokens[pos - rec.min_pos] == tok for rec in self.fifo)

    def _rebase_pending(self) -> None:
        kept: List[Tuple[int, int]] = []
        broken = False
        for pos, tok in self.pending:
            if pos < len(self.accepted):
                if tok != self.accepted[pos]:
                    broken = True
                    break
                continue
            kept.append((pos, tok))
        self.pending = [] if broken else kept
        if not self.pending:
            self.pending_tip_seq = 0

    def _cancel_stale(self) -> None:
        stale = detect_stale_runs(self.fifo, self.accepted)
        for rec, reason in stale:
            rec.status = CANCELLED_INVALID if reason == INVALID else CANCELLED_SUPERFLUOUS
            self._judge_cancelled(rec)
            if reason == INVALID:
                self.cancelled_invalid += 1
            else:
                self.cancelled_superfluous += 1
            self.cancel_log.append(CancelLogEntry(
                rec.run_id, reason, rec.kind, rec.min_pos, rec.max_pos,
                len(self.accepted), tuple(rec.chain())))
            self._count("CANCEL", (24 + 16) * self.pipe.n_stages, 1, self.pipe.n_stages)
        # Publish newest first: the device reads these words while it runs,
        # so a stage that sees an older run cancelled must also see every
        # later one (a descendant built on a skipped partition is doomed too;
        # the reference delivers them together, engine.py:1180-1182).
        for rec, _ in reversed(stale):
            self.pipe.cancel_run(rec.run_id)

    # -- shutdown ------------------------------------------------------------------
    def _finish(self) -> None:
        for rec in reversed(self.fifo):
            if rec.status == IN_FLIGHT:
                rec.status = DRAINED
                self.drained_runs += 1
                self.pipe.cancel_run(rec.run_id)
        while self.fifo:
            res = self._recv()
            rec = self._pop_record(res)
            for q in rec.partitions():
                if q in self.allocator.live():
                    self.allocator.free(q)
        if self.draft_busy:
            self._draft_reply()

    def _draft_round_trip(self, max_tokens: int, cutoff: float):
        ctx = list(self.accepted)
        cp = self._common_prefix(self.mirror, ctx)
        room = self.cfg.max_context - len(ctx)
        truncate_to, feed = self._backoff(cp, ctx)
        self._draft_request(truncate_to, tuple(feed), max(0, min(max_tokens, room)), cutoff)
        self.mirror = ctx
        toks, confs = self._draft_reply()
        self.mirror.extend(toks)
        return toks, confs

    # -- metrics (engine.py:1234-1273) ---------------------------------------------
    def build_metrics(self, wall_seconds: float) -> RunMetrics:
        times = [t for t, _ in self.accept_events]
        k = len(times)
        if k:
            duration = times[-1] - self.window_start
            ttft = times[0] - self.window_start
            gaps = [b - a for a, b in zip(times, times[1:])]
            itl = sum(gaps) / len(gaps) if gaps else 0.0
            speed = k / duration if duration > 0 else float("inf")
        else:
            duration = ttft = itl = speed = 0.0
        out = self.accepted[len(self.prompt):]
        msgs: Dict[str, int] = {}
        for (_, tag), n in self.msgs.items():
            msgs[tag] = msgs.get(tag, 0) + n
        return RunMetrics(
            mode=self.cfg.mode, clock="wall", tokens_generated=len(out),
            duration=duration, generation_speed=speed, ttft=ttft, itl=itl,
            acceptance_rate=(self.matched / self.examined) if self.examined else 0.0,
            examined=self.examined, matched=self.matched,
            runs_started=self.runs_started, spec_runs=self.spec_runs,
            cancelled_invalid=self.cancelled_invalid,
            cancelled_superfluous=self.cancelled_superfluous,
            cancelled_runs=self.cancelled_invalid + self.cancelled_superfluous,
            drained_runs=self.drained_runs, alloc_stalls=self.alloc_stalls,
            inflight_mean=self.inflight.mean(self.window_start,
                                             times[-1] if k else self.window_start),
            bytes_by_tag=dict(self.bytes), msgs_by_tag=msgs,
            token_checksum=token_checksum(out), virtual_end=self.now(),
            wall_seconds=wall_seconds)


# ---------------------------------------------------------------------------
# engine: models + pipeline + draft kept resident across runs
# ---------------------------------------------------------------------------

def truth_table(target_model, prompt: List[int], n: int):
    """Target greedy stream and runner-ups along it (for the synthetic draft).

    ``truth[p]``/``runner[p]`` are the greedy token and runner-up predicted
    for absolute position p given the true context [0, p)."""
    from .model import SerialDecoder
    cfg = target_model.config
    n = min(n, cfg.max_context - len(prompt))
    dec = SerialDecoder(target_model, capacity=cfg.max_context + 64)
    tip = dec.feed(prompt)
    truth, runner = list(prompt), [0] * len(prompt)
    for _ in range(n):
        truth.append(tip.argmax)
        runner.append(tip.second)
        if len(dec) + 1 >= cfg.max_context:
            break
        tip = dec.feed([tip.argmax])
    del dec
    return truth, runner


class Engine:
    """Keeps the GPU-resident models, stages and draft server for a config."""

    def __init__(self, cfg: ExperimentConfig, target_model=None, draft_model=None,
                 pipeline=None, device=None):
        import torch
        from .model import build_model
        from .pipeline import LocalPipeline
        cfg.validate()
        self.cfg = cfg
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.target = target_model or build_model(cfg.target_config(), self.device)
        self.draft_model = None
        if cfg.uses_draft():
            dc = cfg.draft_config()
            self.draft_model = draft_model or build_model(
                dc, self.device, tiled=(cfg.draft_tc if dc.arch == "llama" else None))
        ranges = plan_layer_split(self.target.config.n_layers, cfg.n_stages(), cfg.node_weights)
        self.pipe = pipeline or LocalPipeline(self.target, ranges, partitions=cfg.partitions,
                                              capacity=cfg.capacity,
                                              max_tokens=cfg.max_run_tokens)
        self.draft = None
        self._draft_stream = None
        if cfg.uses_draft():
            # the draft's tiny kernels must not queue behind the target's
            # GEMMs on a shared GPU: highest stream priority + reserved SMs
            hi = torch.cuda.Stream.priority_range()[1] if hasattr(
                torch.cuda.Stream, "priority_range") else -1
            self._draft_stream = torch.cuda.Stream(self.device, priority=hi)
            if cfg.draft_sm_reserve > 0:
                ctas = 2 * max(16, 148 - cfg.draft_sm_reserve)
                for st in getattr(self.pipe, "stages", []):
                    if st.device == self.device and st.cfg.arch == "llama":
                        st.set_cta_budget(ctas)
        self._tables: Dict[tuple, tuple] = {}
        self.last_head_policy: Dict[str, object] = {}

    def _make_draft(self, prompt: List[int], prompt_seed: int):
        from .drafting import ModelDraftServer, TableDraftServer
        cfg = self.cfg
        if not cfg.uses_draft():
            return None
        if cfg.draft_backend == "synthetic":
            key = tuple(prompt)
            need = len(prompt) + min(cfg.gen_len + 16, cfg.max_context - len(prompt) - 1)
            if key not in self._tables or len(self._tables[key][0]) < need:
                if len(self._tables) > 64:
                    self._tables.clear()
                self._tables[key] = self.truth(prompt, cfg.gen_len + 16)
            truth, runner = self._tables[key]
            seed = cfg.draft_seed * 1000003 + prompt_seed
            prev = getattr(self, "_table_draft", None)
            srv = TableDraftServer(self.draft_model, truth, runner, cfg.alpha, seed,
                                   stream=self._draft_stream,
                                   capacity=min(cfg.capacity, 16 * cfg.max_context),
                                   stage=None if prev is None else prev.stage,
                                   charge=cfg.draft_charge,
                                   alpha_sibling=(cfg.alpha_sibling if cfg.tree_width >= 2
                                                  else 0.0))
            if prev is not None:
                srv.forwards = 0
            srv.shared_gpu = self._shares_gpu()
            self._table_draft = srv
            return srv
        if self.draft is None:
            self.draft = ModelDraftServer(self.draft_model, stream=self._draft_stream,
                                          capacity=min(cfg.capacity, 16 * cfg.max_context))
            self.draft.shared_gpu = self._shares_gpu()
        else:
            self.draft.reset()
        return self.draft

    def _shares_gpu(self) -> bool:
        """A target stage of this process runs on the draft's GPU."""
        dev = self.draft_model.device if self.draft_model is not None else None
        return any(getattr(st, "device", None) == dev for st in getattr(self.pipe, "stages", []))

    def run(self, prompt_seed: Optional[int] = None, prompt: Optional[List[int]] = None,
            mode: Optional[str] = None) -> SimResult:
        cfg = self.cfg if mode is None else replace(self.cfg, mode=mode)
        seed = cfg.prompt_seed if prompt_seed is None else prompt_seed
        if prompt is None:
            prompt = sample_prompt(seed, cfg.prompt_len, self.target.config.vocab_size)
        self.pipe.reset()
        draft = self._make_draft(prompt, seed)
        wall0 = time.perf_counter()
        head = Head(cfg, self.pipe, draft, prompt, self.target.config.embed_dim)
        # only an async head that can launch skippable runs needs the
        # conditional (skip) graph bodies; they cost every full run ~0.1 ms
        cancellable = cfg.mode == "async-speculative" and not (
            head.fold_frontier and head.max_inflight == 1 and not head.adaptive)
        if hasattr(self.pipe, "set_skip_graphs"):
            self.pipe.set_skip_graphs(cancellable)
        runner = {"iterative": head.run_iterative,
                  "pipeline-iterative": head.run_iterative,
                  "sync-speculative": head.run_sync_speculative,
                  "async-speculative": head.run_async_speculative}[cfg.mode]
        comp0 = getattr(self.pipe, "compactions", 0)
        runner()
        wall = time.perf_counter() - wall0
        self.last_head_policy = {"fold_frontier": head.fold_frontier,
                                 "max_inflight": head.max_inflight,
                                 "adaptive": head.adaptive, "folded_runs": head.folded_runs,
                                 "sibling_hits": head.sibling_hits,
                                 # cell-pool compactions in this run (each drains
                                 # the stages' streams once: dist.py R_COMPACT)
                                 "compactions": getattr(self.pipe, "compactions", 0) - comp0}
        metrics = head.build_metrics(wall)
        sent = dict(head.msgs)
        node_logs = dict(head.stage_logs)
        if draft is not None:
            node_logs[cfg.nodes] = [("served", draft.forwards)]
        return SimResult(tokens=head.accepted[len(prompt):], metrics=metrics,
                         accepted_full=list(head.accepted),
                         accept_events=list(head.accept_events),
                         cancel_log=list(head.cancel_log), node_logs=node_logs,
                         consumed=dict(sent), sent=sent, records=list(head.records),
                         host_profile=dict(head.profile))

    def truth(self, prompt: List[int], n: int):
        """Greedy stream and runner-ups of the target along the true path,
        computed by an iterative pass through this engine's own pipeline:
        ``truth[p]``/``runner[p]`` are the greedy token / runner-up predicted
        for absolute position p (synthetic-draft table)."""
        n = min(n, self.cfg.max_context - len(prompt) - 1)
        cfg = replace(self.cfg, mode="iterative", gen_len=n, eos_token=None,
                      prompt_len=len(prompt))
        self.pipe.reset()
        head = Head(cfg, self.pipe, None, prompt, self.target.config.embed_dim)
        head.tips = []
        head.run_iterative()
        self.pipe.reset()
        truth = list(prompt) + [r.argmax for r in head.tips]
        runner = [0] * len(prompt) + [r.second for r in head.tips]
        return truth, runner

    def launch_count(self) -> int:
        """Kernels this process has launched through the C ABI so far."""
        n = sum(st.launches for st in getattr(self.pipe, "stages", []))
        for d in (self.draft, getattr(self, "_table_draft", None)):
            if d is not None:
                n += d.stage.launches
        return n

    def generate(self, prompt: Sequence[int], gen_len: Optional[int] = None) -> List[int]:
        """The north star's generate(): accepted tokens after ``prompt``."""
        if gen_len is not None and gen_len != self.cfg.gen_len:
            self.cfg = replace(self.cfg, gen_len=gen_len)
        return self.run(prompt=list(prompt)).tokens


_ENGINES: Dict[tuple, Engine] = {}


def _engine_key(cfg: ExperimentConfig, target_model=None, draft_model=None) -> tuple:
    """Everything that shapes an Engine's resident state: the models, the
    stage split, the cell pools and run buffers, the draft's kernel path."""
    return (cfg.target_config(), cfg.draft_config() if cfg.uses_draft() else None,
            cfg.n_stages(), cfg.node_weights, cfg.partitions, cfg.capacity,
            cfg.max_run_tokens, cfg.uses_draft(), cfg.draft_tc, cfg.draft_sm_reserve,
            id(target_model), id(draft_model))


def _engine_for(cfg: ExperimentConfig, target_model=None, draft_model=None) -> "Engine":
    key = _engine_key(cfg, target_model, draft_model)
    eng = _ENGINES.get(key)
    if eng is None:
        if len(_ENGINES) > 4:
            _ENGINES.clear()
        eng = Engine(cfg, target_model, draft_model)
        _ENGINES[key] = eng
    eng.cfg = cfg
    return eng


def simulate(cfg: ExperimentConfig, target_model=None, draft_model=None) -> SimResult:
    """Run one experiment to completion on the GPU (engine.py:1293-1356).

    Engines (models + stages) are cached per model-shaping config so
    repeated calls with different seeds/modes reuse resident weights.
    """
    cfg.validate()
    return _engine_for(cfg, target_model, draft_model).run()


def generate(prompt: Sequence[int], cfg: Optional[ExperimentConfig] = None,
             **overrides) -> List[int]:
    """Greedy generation of ``cfg.gen_len`` tokens after ``prompt``."""
    cfg = replace(cfg or ExperimentConfig(), prompt_len=len(prompt), **overrides)
    cfg.validate()
    return _engine_for(cfg).run(prompt=list(prompt)).tokens
