"""Target pipelines: where a launched run's stage evaluations execute.

The head (``engine.Head``) talks to a pipeline through five calls that stand
in for the reference's transactions (transport.py:234-271, engine.py:749-796):

* ``launch(run_id, kind, toks, flags, rows)`` — RUN_CONFIG + ACTIVATIONS:
  every stage's evaluation of the run is enqueued at once, in stream order;
* ``copy(src, dsts, end)`` / ``remove(seq, from)`` — CACHE_COPY / CACHE_REMOVE,
  enqueued on every stage behind the runs launched before them;
* ``cancel(run_id)`` — CANCEL: a device-visible word that overtakes queued
  work because kernels read it when they execute;
* ``poll()`` / ``wait()`` — LOGITS, strictly FIFO (``cudaEventQuery``
  replaces ``Network.probe``).

``LocalPipeline`` hosts all stages in this process on one GPU (stages run
back to back on one stream; used for 1-GPU runs and to exercise multi-stage
semantics).  ``dist.DistPipeline`` spreads the stages over torchrun ranks.
"""

from __future__ import annotations

import os
from collections import deque
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _lib
from .model import RowResult
from .runtime import RES_DTYPE, Stage

RESULT_RING = 64


@dataclass
class RunResult:
    run_id: int
    placeholder: bool
    rows: List[RowResult]
    err: int
    stage_status: List[int]


class LocalPipeline:
    def __init__(self, model, ranges, partitions: int = 8, capacity: int = 8192,
                 max_tokens: int = 256, cancel_size: int = 1024, stream=None,
                 device=None):
        import torch

        self.device = model.device if device is None else device
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self.cancel = torch.zeros(cancel_size, dtype=torch.int32).pin_memory()
        self.cancel_np = self.cancel.numpy()
        self.cancel_size = cancel_size
        self.stages = [Stage(model, lo, hi, capacity=capacity, max_tokens=max_tokens,
                             n_seq_ids=partitions, stream=self.stream,
                             cancel_table=self.cancel.data_ptr(),
                             cancel_size=cancel_size)
                       for lo, hi in ranges]
        # result block per in-flight run: [status, err, -, -] + rows
        self.res_host = torch.zeros((RESULT_RING, 1 + max_tokens, 4),
                                    dtype=torch.int32).pin_memory()
        self.res_np = self.res_host.numpy()
        self.events = [torch.cuda.Event() for _ in range(RESULT_RING)]
        torch.cuda.synchronize(self.device)
        self.fifo: deque = deque()
        self.max_tokens = max_tokens
        self.d = model.config.embed_dim
        self.io = [st.io() for st in self.stages]
        self.capacity = capacity
        self.compactions = 0
        self._compact_at = 0.75 * capacity
        # diagnostics (SP_RUN_TIMING=1, tools/async_timeline.py): per launched
        # run, timing events on the stage stream around its stage steps
        self.timing = os.environ.get("SP_RUN_TIMING") == "1"
        self.timeline: list = []

    @property
    def n_stages(self) -> int:
        return len(self.stages)

    def reset(self) -> None:
        if self.fifo:
            raise RuntimeError("reset with runs in flight")
        for st in self.stages:
            st.reset()
        self._compact_at = 0.75 * self.capacity
        self.cancel_np[:] = 0
        self.stream.synchronize()

    # -- transactions -----------------------------------------------------------
    def launch(self, run_id: int, kind: int, toks: np.ndarray, flags: int,
               rows: List[int]) -> None:
        """Every stage's evaluation as one graph-replayed ``sp_stage_step``;
        stage i reads stage i-1's fixed output buffer (activations + status
        word), the last stage's result block lands in pinned host memory."""
        if len(self.fifo) >= RESULT_RING:
            raise RuntimeError("too many runs in flight")
        if not rows:
            raise ValueError("a run must request at least one logits row")
        slot = run_id % RESULT_RING
        n = len(toks)
        if self.stages[0].n_cells() + n > self._compact_at:
            # bounded cell pool: let the queued runs finish, then reclaim the
            # dead cells (their results stay in the result ring for the head)
            self.stream.synchronize()
            live = 0
            for st in self.stages:
                live = st.compact()
            self.compactions += 1
            # a pool that stays mostly live compacts again only when half of
            # the remaining room is used (never on every launch)
            self._compact_at = max(0.75 * self.capacity, (live + self.capacity) / 2)
        if self.timing:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(self.stream)
        x_in = stat = None
        last = len(self.stages) - 1
        for i, st in enumerate(self.stages):
            st.step(toks, run_id, kind, flags, rows=rows if i == last else (),
                    x_in=x_in, in_status=stat,
                    res_copy=self.res_host[slot].data_ptr() if i == last else None)
            x_in = self.io[i][0]
            stat = x_in + 4 * n * self.d
        self.events[slot].record(self.stream)
        if self.timing:
            ev[1].record(self.stream)
            self.timeline.append((run_id, kind, n, ev[0], ev[1]))
        self.fifo.append((run_id, slot, len(rows)))

    def set_skip_graphs(self, on: bool) -> None:
        """Conditional graph bodies only where runs can be cancelled."""
        if getattr(self, "_skip_graphs", None) is not on:
            self.stream.synchronize()
            for st in self.stages:
                st.set_skip_graphs(on)
            self._skip_graphs = on

    def copy(self, src: int, dsts, end_pos: int) -> None:
        for st in self.stages:
            st.cache_copy(src, dsts, end_pos)

    def remove(self, seq: int, from_pos: int) -> None:
        for st in self.stages:
            st.cache_remove(seq, from_pos)

    def cancel_run(self, run_id: int) -> None:
        # host store into mapped pinned memory: visible to kernels at once
        self.cancel_np[run_id % self.cancel_size] = run_id

    # -- completions ------------------------------------------------------------
    def ready(self) -> bool:
        return bool(self.fifo) and self.events[self.fifo[0][1]].query()

    def _collect(self) -> RunResult:
        run_id, slot, nrow = self.fifo.popleft()
        blk = self.res_np[slot]
        status = int(blk[0, 0])
        placeholder = status == _lib.SP_STATUS_PLACEHOLDER
        err = int(blk[0, 1])
        rows = []
        if not placeholder and nrow:
            rr = blk[1:1 + nrow].view(RES_DTYPE).reshape(-1)
            rows = [RowResult(r["a"], r["b"], r["c"], r["d"]) for r in rr]
        # per-stage status is not read back: a placeholder anywhere reaches
        # the last stage, which is what the head acts on
        return RunResult(run_id, placeholder, rows, err, [status] * self.n_stages)

    def poll(self) -> Optional[RunResult]:
        return self._collect() if self.ready() else None

    def wait(self) -> RunResult:
        if not self.fifo:
            raise RuntimeError("wait with an empty FIFO")
        self.events[self.fifo[0][1]].synchronize()
        return self._collect()

    def in_flight(self) -> int:
        return len(self.fifo)

    def shutdown(self) -> None:
        self.stream.synchronize()
