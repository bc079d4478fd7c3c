"""Asynchronous draft servers: the GPU stand-in for the reference's dedicated
draft node (``_DraftNode``, engine.py:640-688).

A request (DraftRequestPayload, engine.py:313-322) truncates the draft
context, feeds new tokens, then speculates up to ``max_tokens`` while the
confidence stays >= the request's cutoff (speculate_microbatch with
microbatch 1 and no recovery/decay, engine.py:669-680).  Everything runs on
the draft's own CUDA stream; the head polls ``ready()`` and collects
``reply()`` without blocking the target pipeline.

* ``ModelDraftServer`` — a real draft model (ToyDraft semantics).  The
  confidence test runs on the device: each step's LM head folds
  ``conf >= cutoff`` into a gate that the next step reads, and the next
  step's token is the previous argmax.  For llama bf16 drafts with
  row-major weights the whole request (feed + chain) is ONE persistent
  kernel (``sp_stage_decode_chain``, K15); otherwise one graph-replayed
  ``sp_stage_step`` per forward.  Either way: one readback per request.
* ``TableDraftServer`` — alpha-controlled synthetic proposals
  (SyntheticDraft, speculation.py:98-139): the target's greedy token with
  PCG64 probability alpha, else its runner-up, from a table of the target's
  own greedy stream.  The cost of a real draft-shape
  forward is still paid on the GPU for every fed and proposed token.
"""

from __future__ import annotations

import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import SpeculationError
from .model import PREFILL, KIND_CODE, BatchToken, encode_tokens
from .runtime import RES_DTYPE, Stage


def _check_rc(rc: int) -> None:
    if rc:
        from . import _lib
        _lib.check(rc, "sp_copy_async")


class _DraftBase:
    def __init__(self, draft_model, stream=None, capacity: Optional[int] = None,
                 max_tokens: int = 256, stage: Optional[Stage] = None):
        import torch
        self.model = draft_model
        cfg = draft_model.config
        self.max_context = cfg.max_context
        if stage is not None:          # reuse a resident stage (cleared)
            self.stream = stage.stream
            self.stage = stage
            stage.reset()
        else:
            self.stream = stream if stream is not None else torch.cuda.Stream(draft_model.device)
            cap = capacity or max(1024, 8 * cfg.max_context)
            self.stage = Stage(draft_model, 0, cfg.n_layers, capacity=cap,
                               max_tokens=max_tokens, n_seq_ids=1, stream=self.stream)
        # result blocks: [status, err, -, -] + one row result (sp_stage_step);
        # block 0 row = the chain's starting tip, 1..4 the chain steps, 7 feeds
        self.res = torch.zeros((8, 2, 4), dtype=torch.int32, device=draft_model.device)
        self.res_host = torch.zeros((8, 2, 4), dtype=torch.int32).pin_memory()
        self._blocks: List[int] = []
        cfgm = draft_model.config
        self.fused_ok = bool(self.stage.lib.sp_stage_decode_chain_ok(self.stage.h))
        # one persistent launch per request (K15): the cluster form (16 SMs)
        # by default, the grid form (every SM) on a dedicated draft GPU;
        # SP_DRAFT_FUSED=0 falls back to one graph-replayed step per forward
        self.fused = self.fused_ok and os.environ.get("SP_DRAFT_FUSED", "1") != "0"
        # set by the Engine when a target stage runs on the draft's GPU: each
        # request then takes the grid form while no target run is queued (the
        # GPU is otherwise idle) and the 16-SM cluster form beside one
        self.shared_gpu = False
        self._kind = None
        if self.fused:     # a reused stage may carry another server's choice
            self.stage.lib.sp_stage_set_draft_kernel(self.stage.h, 0)
        # fused path: rows 0..64 of (argmax, second, conf, max_logit) + err word
        self.rows = torch.zeros((66, 4), dtype=torch.int32, device=draft_model.device)
        self.rows_host = torch.zeros((66, 4), dtype=torch.int32).pin_memory()
        self.event = torch.cuda.Event()
        self.tokens: List[int] = []
        # tokens [0, cached) have K/V cells; the persistent kernels do not
        # forward a request's LAST proposal (only the next request needs its
        # cells, and feeds it then in the same forward as its own tokens:
        # one draft forward per request saved)
        self.cached = 0
        self.seconds: tuple = ()   # the draft's runner-up per proposal (tree speculation)
        self._pending = None
        self.forwards = 0          # draft-model forwards issued (cost accounting)
        # diagnostics (SP_RUN_TIMING=1): timing events around each request
        self.timing = os.environ.get("SP_RUN_TIMING") == "1"
        self.timeline: list = []
        self._t0 = None
        torch.cuda.synchronize(draft_model.device)

    def __len__(self) -> int:
        return len(self.tokens)

    def reset(self) -> None:
        if self._pending is not None:
            self.reply()
        self.stage.reset()
        self.tokens = []
        self.cached = 0
        self.stream.synchronize()

    # -- shared GPU steps -------------------------------------------------------
    def _truncate(self, n: int) -> None:
        """Rows == positions: drop tokens >= n and every cell past the kept
        tokens (dead chain steps and a not-yet-forwarded proposal included)."""
        if n < len(self.tokens):
            self.stage.invalidate_tip()
            del self.tokens[n:]
        if self.cached > len(self.tokens):
            self.cached = len(self.tokens)
        elif self.cached < len(self.tokens):
            self.stage.invalidate_tip()      # the tip predates the uncached token
        self.stage.truncate(self.cached)

    def _launch_chain(self, feed: Sequence[int], pos0: int, steps: int, cutoff: float,
                      step_tokens: Optional[Sequence[int]] = None) -> None:
        """Fused request: feed + ``steps`` steps in one persistent launch;
        results -> rows[0..steps], err -> rows[65, 0].  Feeds longer than the
        kernel's 4-token tile (prefill) go through the batched path first."""
        import torch
        feed = list(feed)
        if len(feed) > 4:
            self._forward(feed, pos0)
            pos0 += len(feed)
            feed = []
        self.stage.decode_chain(feed, pos0, steps, cutoff, self.rows.data_ptr(),
                                self.rows[65].data_ptr(), step_tokens)
        self.forwards += (1 if feed else 0) + steps
        # result rows to pinned host memory, stream-ordered (a direct async
        # copy: no torch stream context on the request's critical path)
        lib, st = self.stage.lib, self._raw_stream()
        _check_rc(lib.sp_copy_async(self.rows_host.data_ptr(), self.rows.data_ptr(),
                                    self.rows.numel() * 4, st))
        if self._blocks:      # (only a batched feed forward left a result block)
            _check_rc(lib.sp_copy_async(self.res_host.data_ptr(), self.res.data_ptr(),
                                        self.res.numel() * 4, st))
        self.event.record(self.stream)

    def _chain(self, feed: Sequence[int], steps: int, cutoff: float) -> None:
        self._launch_chain(feed, len(self.tokens), steps, cutoff)
        self.tokens.extend(feed)

    def _check_fused_err(self) -> None:
        self._check_err()
        err = int(self.rows_host[65, 0])
        if err:
            from . import _lib
            _lib.raise_device_error(err, "draft")

    def _forward(self, toks: Sequence[int], base: int, chain: bool = False,
                 cutoff: float = 0.0, block: int = 7) -> None:
        """One draft forward + LM head over its last token as one replayed
        graph; result block -> ``res[block]``.  ``chain``: token 0 is the
        previous argmax, gated on the device (conf >= cutoff)."""
        from . import _lib
        batch = [BatchToken(t, base + i, frozenset([0]), i == len(toks) - 1)
                 for i, t in enumerate(toks)]
        self.stage.step(encode_tokens(batch), run_id=0, kind=KIND_CODE[PREFILL], flags=0,
                        rows=[len(toks) - 1],
                        head=_lib.SP_STEP_CHAIN if chain else _lib.SP_STEP_TIP,
                        cutoff=cutoff, res_copy=self.res[block].data_ptr())
        self.forwards += 1
        self._blocks.append(block)

    def _finish_enqueue(self, nrows: int) -> None:
        _check_rc(self.stage.lib.sp_copy_async(self.res_host.data_ptr(), self.res.data_ptr(),
                                               self.res.numel() * 4, self._raw_stream()))
        self.event.record(self.stream)

    def _raw_stream(self):
        import ctypes
        h = getattr(self, "_stream_handle", None)
        if h is None:
            h = self._stream_handle = ctypes.c_void_p(self.stream.cuda_stream)
        return h

    def _check_err(self) -> None:
        blocks, self._blocks = self._blocks, []
        for b in blocks:
            err = int(self.res_host[b, 0, 1])
            if err:
                from . import _lib
                _lib.raise_device_error(err, "draft")

    def set_exclusive(self, idle: bool) -> None:
        """Kernel choice for the next request on a shared GPU (see shared_gpu)."""
        if not (self.fused and self.shared_gpu):
            return
        from . import _lib
        kind = _lib.SP_DRAFT_KIND_GRID if idle else _lib.SP_DRAFT_KIND_CLUSTER
        if kind != self._kind:
            _lib.check(self.stage.lib.sp_stage_set_draft_kernel(self.stage.h, kind),
                       "sp_stage_set_draft_kernel")
            self._kind = kind

    def _mark_start(self) -> None:
        if self.timing:
            import torch
            self._t0 = torch.cuda.Event(enable_timing=True)
            self._t0.record(self.stream)

    def _mark_end(self, n_feed: int, n_props: int) -> None:
        if self.timing and self._t0 is not None:
            import torch
            e = torch.cuda.Event(enable_timing=True)
            e.record(self.stream)
            self.timeline.append((n_feed, n_props, self._t0, e))
            self._t0 = None

    def ready(self) -> bool:
        return self._pending is not None and self.event.query()

    def busy(self) -> bool:
        return self._pending is not None


class ModelDraftServer(_DraftBase):
    """ToyDraft semantics (speculation.py:65-95) with a device-side loop."""

    def request(self, truncate_to: int, feed: Sequence[int], max_tokens: int,
                cutoff: float) -> None:
        if self._pending is not None:
            raise SpeculationError("draft request while one is in flight")
        self._mark_start()
        self._truncate(truncate_to)
        feed = list(feed)
        room = self.max_context - len(self.tokens) - len(feed)
        budget = max(0, min(int(max_tokens), room, 4))
        c32 = float(np.float32(cutoff))
        if self.fused:
            # uncached kept tokens ride in front of this request's feed; the
            # chain runs budget - 1 steps (the last proposal is not forwarded)
            full = self.tokens[self.cached:] + feed
            if full or budget > 0:
                self._launch_chain(full, self.cached, max(0, budget - 1), c32)
            else:
                self.event.record(self.stream)
            self.tokens.extend(feed)
            self.cached = len(self.tokens)
            self._pending = (budget, np.float32(cutoff), True)
            self._mark_end(len(full), budget)
            return
        if self.cached < len(self.tokens):        # (a kernel-path leftover)
            feed = self.tokens[self.cached:] + feed
            del self.tokens[self.cached:]
        if feed:
            self._forward(feed, len(self.tokens))
            self.tokens.extend(feed)
            self.cached = len(self.tokens)
        if budget > 0:
            self.stage.chain_begin(c32, self.res[0, 1].data_ptr())
            base = len(self.tokens)
            for j in range(budget):
                self._forward([0], base + j, chain=True, cutoff=c32, block=1 + j)
        self._finish_enqueue(budget + 1)
        self._pending = (budget, np.float32(cutoff), False)
        self._mark_end(len(feed), budget)

    def reply(self) -> Tuple[tuple, tuple]:
        budget, c32, fused = self._pending
        self.event.synchronize()
        self._pending = None
        if fused:
            self._check_fused_err()
        else:
            self._check_err()
        self.seconds = ()
        if budget == 0:
            return (), ()
        if fused:
            r = self.rows_host[:budget + 1].numpy().view(RES_DTYPE).reshape(-1)
        else:
            r = self.res_host[:budget + 1, 1].numpy().view(RES_DTYPE).reshape(-1)
        toks, confs, secs = [], [], []
        for j in range(budget):
            conf = np.float32(r[j]["c"])
            if j == 0 and (conf < 0 or r[0]["a"] < 0):
                raise SpeculationError("draft has no context yet")
            if conf < c32:
                break
            toks.append(int(r[j]["a"]))
            confs.append(float(conf))
            secs.append(int(r[j]["b"]))
        # fused: proposals 1 .. budget-1 were forwarded (a proposal is fed
        # only while the gate is open, i.e. when it was returned)
        fed = min(len(toks), budget - 1) if fused else len(toks)
        self.cached = len(self.tokens) + fed
        self.tokens.extend(toks)
        self.seconds = tuple(secs)
        return tuple(toks), tuple(confs)


class TableDraftServer(_DraftBase):
    """SyntheticDraft semantics over a table of the target's greedy stream.

    ``truth[p]`` / ``runner[p]``: the target's greedy token and runner-up at
    absolute position ``p`` along the true path.  Off the true path (after a
    proposal that is not the truth) any proposal is equivalent: such tokens
    only ever feed runs that are invalidated, never verified or judged.
    """

    def __init__(self, draft_model, truth: Sequence[int], runner: Sequence[int],
                 alpha: float, seed: int, stream=None, capacity=None,
                 charge: bool = True, max_tokens: int = 256, stage=None,
                 alpha_sibling: float = 0.0):
        super().__init__(draft_model, stream, capacity, max_tokens, stage)
        if not 0.0 <= alpha <= 1.0:
            raise SpeculationError(f"alpha must be in [0,1], got {alpha}")
        self.alpha = float(alpha)
        self.rng = np.random.Generator(np.random.PCG64(seed))
        # tree speculation: the runner-up choice per proposal.  A separate
        # stream, so chain emissions stay the reference's draw sequence
        self.alpha_sibling = float(alpha_sibling)
        self.rng2 = np.random.Generator(np.random.PCG64(seed + 0x5EED))
        self.vocab = draft_model.config.vocab_size
        self.truth = list(truth)
        self.runner = list(runner)
        self.charge = charge
        self.on_path = 0   # length of the prefix of self.tokens equal to truth

    def _retrack(self, start: int) -> None:
        p = min(self.on_path, start)
        while p < len(self.tokens) and p < len(self.truth) and self.tokens[p] == self.truth[p]:
            p += 1
        self.on_path = p

    def request(self, truncate_to: int, feed: Sequence[int], max_tokens: int,
                cutoff: float) -> None:
        if self._pending is not None:
            raise SpeculationError("draft request while one is in flight")
        self._mark_start()
        if truncate_to < len(self.tokens):
            if self.charge:
                self._truncate(truncate_to)
            else:
                del self.tokens[truncate_to:]
            self.on_path = min(self.on_path, truncate_to)
        elif self.charge:
            self._truncate(len(self.tokens))
        feed = list(feed)
        feed_pos = len(self.tokens)
        pend = self.tokens[self.cached:] if self.charge else []   # kept, not yet forwarded
        if feed:
            if self.charge and not self.fused:
                self._forward(pend + feed, self.cached)
                pend = []
                self.cached = feed_pos + len(feed)
            self.tokens.extend(feed)
            self._retrack(feed_pos)
        room = self.max_context - len(self.tokens)
        budget = max(0, min(int(max_tokens), room, 4))
        props = []
        if budget > 0 and len(self.tokens) == 0:
            raise SpeculationError("draft has no context yet")
        secs = []
        if budget > 0 and not self.alpha < cutoff:
            for _ in range(budget):
                p = len(self.tokens)
                best = self.truth[p] if p < len(self.truth) else 0
                second = self.runner[p] if p < len(self.runner) else 1
                tok = best if self.rng.random() < self.alpha else second
                if self.alpha_sibling > 0.0:
                    # the runner-up: the other of (greedy, runner-up) when the
                    # first choice is the greedy token; when it is not, the
                    # greedy token with probability alpha_sibling, else a
                    # third token (off the greedy path either way)
                    hit = self.rng2.random() < self.alpha_sibling
                    if tok == best:
                        alt = second
                    elif hit:
                        alt = best
                    else:
                        alt = (best + 1) % self.vocab
                        if alt == tok:
                            alt = (best + 2) % self.vocab
                    secs.append(alt)
                if self.charge and not self.fused:
                    self._forward(pend + [tok], self.cached)
                    pend = []
                    self.cached = p + 1
                self.tokens.append(tok)
                self._retrack(p)
                props.append(tok)
        self.seconds = tuple(secs)
        if self.charge and self.fused and (feed or props):
            # the forwards a real draft would run, as one persistent launch:
            # kept-but-unforwarded tokens and the feed in one forward, then
            # every proposal but the last (the next request forwards it)
            full = pend + feed
            steps = max(0, len(props) - 1)
            if full or steps:
                self._launch_chain(full, self.cached, steps, 0.0, step_tokens=props[:steps])
                self.cached = feed_pos + len(feed) + steps
                self._pending = (tuple(props), True)
            else:
                self._finish_enqueue(1)
                self._pending = (tuple(props), False)
            self._mark_end(len(full), len(props))
            return
        self._finish_enqueue(1)
        self._pending = (tuple(props), False)
        self._mark_end(len(feed), len(props))

    def reply(self) -> Tuple[tuple, tuple]:
        props, fused = self._pending
        self.event.synchronize()
        self._pending = None
        if fused:
            self._check_fused_err()
        else:
            self._check_err()
        return props, tuple(self.alpha for _ in props)
