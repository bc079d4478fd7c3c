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
  ``conf >= cutoff`` into a gate word that the next step's kernels read, and
  the next step's token is the previous argmax, so a whole micro-batch is
  one stream of launches with a single readback.
* ``TableDraftServer`` — alpha-controlled synthetic proposals
  (SyntheticDraft, speculation.py:98-139): the target's greedy token with
  PCG64 probability alpha, else its runner-up, from a table of the target's
  own greedy stream.  The cost of a real draft-shape
  forward is still paid on the GPU for every fed and proposed token.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import SpeculationError
from .model import PREFILL, KIND_CODE, BatchToken, encode_tokens
from .runtime import RES_DTYPE, Stage


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
        self.res = torch.zeros((8, 4), dtype=torch.int32, device=draft_model.device)
        self.res_host = torch.zeros((8, 4), dtype=torch.int32).pin_memory()
        self.event = torch.cuda.Event()
        self.tokens: List[int] = []
        self._pending = None
        self.forwards = 0          # draft-model forwards issued (cost accounting)
        torch.cuda.synchronize(draft_model.device)

    def __len__(self) -> int:
        return len(self.tokens)

    def reset(self) -> None:
        if self._pending is not None:
            self.reply()
        self.stage.reset()
        self.tokens = []
        self.stream.synchronize()

    # -- shared GPU steps -------------------------------------------------------
    def _truncate(self, n: int) -> None:
        if n < len(self.tokens):
            self.stage.cache_remove(0, n)
            self.stage.invalidate_tip()
            del self.tokens[n:]

    def _forward(self, toks: Sequence[int], base: int, chain: bool = False,
                 update_tip: bool = True, gate: bool = False, cutoff: float = 0.0,
                 out_row: Optional[int] = None) -> None:
        batch = [BatchToken(t, base + i, frozenset([0]), i == len(toks) - 1)
                 for i, t in enumerate(toks)]
        self.stage.forward(encode_tokens(batch), run_id=0, kind=KIND_CODE[PREFILL],
                           flags=0, chain=chain)
        out = self.res[out_row].data_ptr() if out_row is not None else self.res[7].data_ptr()
        self.stage.lmhead([len(toks) - 1], out=out, err_out=self.res[6, 1:].data_ptr(),
                          update_tip=update_tip, chain_gate=gate, cutoff=cutoff)
        self.forwards += 1

    def _finish_enqueue(self, nrows: int) -> None:
        import torch
        with torch.cuda.stream(self.stream):
            self.res_host.copy_(self.res, non_blocking=True)
        self.event.record(self.stream)

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
        self._truncate(truncate_to)
        feed = list(feed)
        if feed:
            self._forward(feed, len(self.tokens))
            self.tokens.extend(feed)
        room = self.max_context - len(self.tokens)
        budget = max(0, min(int(max_tokens), room, 4))
        c32 = float(np.float32(cutoff))
        if budget > 0:
            self.stage.chain_begin(c32, self.res[0].data_ptr())
            base = len(self.tokens)
            for j in range(budget):
                self._forward([0], base + j, chain=True, gate=True, cutoff=c32,
                              out_row=1 + j)
        self._finish_enqueue(budget + 1)
        self._pending = (budget, np.float32(cutoff))

    def reply(self) -> Tuple[tuple, tuple]:
        budget, c32 = self._pending
        self.event.synchronize()
        self._pending = None
        err = int(self.res_host[6, 1])
        if err:
            from . import _lib
            _lib.raise_device_error(err, "draft")
        if budget == 0:
            return (), ()
        r = self.res_host[:budget + 1].numpy().view(RES_DTYPE).reshape(-1)
        toks, confs = [], []
        for j in range(budget):
            conf = np.float32(r[j]["c"])
            if j == 0 and (conf < 0 or r[0]["a"] < 0):
                raise SpeculationError("draft has no context yet")
            if conf < c32:
                break
            toks.append(int(r[j]["a"]))
            confs.append(float(conf))
        self.tokens.extend(toks)
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
                 charge: bool = True, max_tokens: int = 256, stage=None):
        super().__init__(draft_model, stream, capacity, max_tokens, stage)
        if not 0.0 <= alpha <= 1.0:
            raise SpeculationError(f"alpha must be in [0,1], got {alpha}")
        self.alpha = float(alpha)
        self.rng = np.random.Generator(np.random.PCG64(seed))
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
        if truncate_to < len(self.tokens):
            if self.charge:
                self._truncate(truncate_to)
            else:
                del self.tokens[truncate_to:]
            self.on_path = min(self.on_path, truncate_to)
        feed = list(feed)
        if feed:
            if self.charge:
                self._forward(feed, len(self.tokens))
            start = len(self.tokens)
            self.tokens.extend(feed)
            self._retrack(start)
        room = self.max_context - len(self.tokens)
        budget = max(0, min(int(max_tokens), room, 4))
        props = []
        if budget > 0 and len(self.tokens) == 0:
            raise SpeculationError("draft has no context yet")
        if budget > 0 and not self.alpha < cutoff:
            for _ in range(budget):
                p = len(self.tokens)
                best = self.truth[p] if p < len(self.truth) else 0
                second = self.runner[p] if p < len(self.runner) else 1
                tok = best if self.rng.random() < self.alpha else second
                if self.charge:
                    self._forward([tok], p)
                self.tokens.append(tok)
                self._retrack(p)
                props.append(tok)
        self._finish_enqueue(1)
        self._pending = tuple(props)

    def reply(self) -> Tuple[tuple, tuple]:
        props = self._pending
        self.event.synchronize()
        self._pending = None
        return props, tuple(self.alpha for _ in props)
