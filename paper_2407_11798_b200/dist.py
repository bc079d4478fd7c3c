"""Multi-GPU pipeline: one process per B200 under torchrun.

Rank r hosts pipeline stage r (a contiguous layer range from
``plan_layer_split``); rank 0 also hosts the head and the draft (its own
stream).  The reference's transactions (transport.py:234-271) map onto:

* RUN_CONFIG / CACHE_COPY / CACHE_REMOVE / SHUTDOWN — records in a
  single-writer ring in POSIX shared memory.  Every worker reads every record
  in order and enqueues the matching work on its compute stream, so stream
  order *is* the reference's per-stage transaction order.  The host never
  waits for the GPU.
* ACTIVATIONS — NCCL point-to-point ``isend``/``irecv`` between consecutive
  ranks (NVLink), issued on the compute stream; the message carries the
  M x d activations plus a status word (placeholder, engine.py:545-554).
* CANCEL — words in the same shared region, page-locked and mapped into
  every GPU's address space: the head's store overtakes all queued work
  because kernels read the word when they execute (early cancellation).
* LOGITS — the last rank copies its fused-head result block into the shared
  region and raises a ready flag from the stream (``sp_signal``); the head
  polls the flag (FIFO).
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import time
import uuid
from collections import deque
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import check
from .model import RowResult, TOKEN_DTYPE
from .pipeline import RunResult
from .runtime import RES_DTYPE, Stage

# record types
R_RUN, R_COPY, R_REMOVE, R_RESET, R_SHUTDOWN, R_MARK, R_COMPACT = 1, 2, 3, 4, 5, 6, 7

RING = 2048            # control records
SLOT = 4096            # bytes per record (header + <= 254 tokens)
CANCEL = 4096          # cancel words (run_id % CANCEL)
RESULTS = 64           # result slots (>= runs in flight)
ACT_RING = 16          # activation buffers per rank (>= runs in flight)
PAGE = 4096


def _align(n: int, a: int = PAGE) -> int:
    return (n + a - 1) // a * a


class ControlPlane:
    """Shared-memory ring + cancel words + result blocks (one per job)."""

    def __init__(self, name: str, create: bool, n_ranks: int, max_tokens: int,
                 n_stat: int):
        from multiprocessing import shared_memory
        import platform
        # Records are published by a plain store of the ring index after the
        # record bytes, and results are read after their flag: correct under
        # x86-TSO only (no acquire/release from numpy).  A weakly ordered host
        # (aarch64 Grace) needs real fences here -- refuse rather than race.
        if platform.machine() not in ("x86_64", "AMD64"):
            raise RuntimeError("dist.ControlPlane relies on x86-TSO store ordering; "
                               f"host is {platform.machine()}")
        self.n_ranks = n_ranks
        self.res_rows = 1 + max_tokens   # [status, err, -, -] + rows
        self.res_bytes = _align(self.res_rows * 16, 256)
        self.off_ring = PAGE
        self.off_cancel = self.off_ring + RING * SLOT
        self.off_res = self.off_cancel + _align(CANCEL * 4)
        self.off_flags = self.off_res + RESULTS * self.res_bytes
        self.size = _align(self.off_flags + RESULTS * 4)
        if create:
            self.shm = shared_memory.SharedMemory(name=name, create=True, size=self.size)
            self.shm.buf[:self.size] = b"\0" * self.size
        else:
            self.shm = shared_memory.SharedMemory(name=name, create=False)
            try:  # only the creator owns (and unlinks) the segment
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        buf = self.shm.buf
        self.hdr = np.ndarray((64,), dtype=np.int64, buffer=buf, offset=0)
        self.ring = np.ndarray((RING, SLOT), dtype=np.uint8, buffer=buf, offset=self.off_ring)
        self.cancel = np.ndarray((CANCEL,), dtype=np.int32, buffer=buf, offset=self.off_cancel)
        self.res = np.ndarray((RESULTS, self.res_bytes // 4), dtype=np.int32, buffer=buf,
                              offset=self.off_res)
        self.flags = np.ndarray((RESULTS,), dtype=np.int32, buffer=buf, offset=self.off_flags)
        self.base = self.hdr.ctypes.data   # offset 0 of the mapping
        self.dev_base = None
        self.creator = create
        self.cursor = 0

    # device mapping of [cancel .. flags] (page-aligned)
    def register(self) -> None:
        lib = _lib.load()
        dev = C.c_void_p()
        n = self.size - self.off_cancel
        check(lib.sp_host_register(self.base + self.off_cancel, n, C.byref(dev)),
              "sp_host_register")
        self.dev_base = dev.value - self.off_cancel

    def dev(self, off: int) -> int:
        return self.dev_base + off

    def cancel_dev(self) -> int:
        return self.dev(self.off_cancel)

    def res_dev(self, slot: int) -> int:
        return self.dev(self.off_res + slot * self.res_bytes)

    def flag_dev(self, slot: int) -> int:
        return self.dev(self.off_flags + 4 * slot)

    # -- writer (rank 0) ---------------------------------------------------------
    def write(self, rtype: int, payload: bytes) -> None:
        idx = int(self.hdr[1])
        while True:
            lag = min(int(self.hdr[8 + r]) for r in range(1, self.n_ranks))
            if idx - lag < RING:
                break
            os.sched_yield()
        if len(payload) + 8 > SLOT:
            raise ValueError("control record too large")
        rec = self.ring[idx % RING]
        rec[:8] = np.frombuffer(struct.pack("<ii", rtype, len(payload)), dtype=np.uint8)
        rec[8:8 + len(payload)] = np.frombuffer(payload, dtype=np.uint8)
        self.hdr[1] = idx + 1          # publish (x86-TSO: record stores land first)

    # -- readers (ranks >= 1) ------------------------------------------------------
    def read(self, rank: int):
        idx = self.cursor
        while int(self.hdr[1]) <= idx:
            os.sched_yield()
        rec = self.ring[idx % RING]
        rtype, n = struct.unpack("<ii", rec[:8].tobytes())
        payload = rec[8:8 + n].tobytes()
        self.cursor = idx + 1
        self.hdr[8 + rank] = self.cursor
        return rtype, payload

    def close(self, unlink: bool = False) -> None:
        try:
            if self.dev_base is not None:
                _lib.load().sp_host_unregister(C.c_void_p(self.base + self.off_cancel))
                self.dev_base = None
        except Exception:
            pass
        del self.hdr, self.ring, self.cancel, self.res, self.flags
        try:
            self.shm.close()
        except BufferError:   # a caller still holds a view; the OS unmaps at exit
            pass
        if unlink:
            self.shm.unlink()


def _pack_run(run_id, kind, flags, toks: np.ndarray, rows) -> bytes:
    r = np.asarray(rows, dtype=np.int32)
    return (struct.pack("<iiiii", run_id, kind, flags, len(toks), len(r))
            + r.tobytes() + np.ascontiguousarray(toks, dtype=TOKEN_DTYPE).tobytes())


def _unpack_run(p: bytes):
    run_id, kind, flags, n, nr = struct.unpack("<iiiii", p[:20])
    rows = np.frombuffer(p[20:20 + 4 * nr], dtype=np.int32)
    toks = np.frombuffer(p[20 + 4 * nr:20 + 4 * nr + 16 * n], dtype=TOKEN_DTYPE).copy()
    return run_id, kind, flags, toks, rows


class _StageRank:
    """Per-rank stage state shared by the head side and the worker loop."""

    def __init__(self, model, lo, hi, rank, world, plane: ControlPlane, cfg_part,
                 capacity, max_tokens, first: int = 0):
        import torch
        self.rank, self.world = rank, world
        self.first = first          # rank of the first pipeline stage
        self.plane = plane
        self.stream = torch.cuda.Stream(model.device)
        self.stage = Stage(model, lo, hi, capacity=capacity, max_tokens=max_tokens,
                           n_seq_ids=cfg_part, stream=self.stream,
                           cancel_table=plane.cancel_dev(), cancel_size=CANCEL)
        d = model.config.embed_dim
        self.d = d
        self.words = max_tokens * d + 4
        self.inbuf = torch.zeros(self.words, dtype=torch.float32, device=model.device)
        self.outbuf = torch.zeros((ACT_RING, self.words), dtype=torch.float32, device=model.device)
        self.gx_out = self.stage.io()[0]
        self.works = deque()
        torch.cuda.synchronize(model.device)

    def _reap(self) -> None:
        while self.works and self.works[0].is_completed():
            self.works.popleft()

    def run(self, run_id, kind, flags, toks, rows) -> None:
        """One stage-run as a graph-replayed ``sp_stage_step``.  The receive
        buffer is fixed (NCCL's stream waits on this stream before writing
        it, so the previous run has consumed it); the send goes from a ring
        slot so a slow peer never holds up the next run's output."""
        import torch
        import torch.distributed as dist
        n = len(toks)
        nw = n * self.d + 4
        last = self.rank == self.world - 1
        recv = self.rank > self.first
        with torch.cuda.stream(self.stream):
            if recv:
                dist.irecv(self.inbuf[:nw], src=self.rank - 1,
                           group=_pair(self.rank - 1)).wait()
            x_in = self.inbuf.data_ptr() if recv else None
            stat = x_in + 4 * n * self.d if recv else None
            slot = run_id % RESULTS
            self.stage.step(toks, run_id, kind, flags, rows=rows if last else (),
                            x_in=x_in, in_status=stat,
                            res_copy=self.plane.res_dev(slot) if last and len(rows) else None)
            s = self.stream.cuda_stream
            if not last:
                while len(self.works) >= ACT_RING - 1:   # slot reuse: its send is done
                    self.works.popleft().wait()
                xout = self.outbuf[run_id % ACT_RING]
                check(self.stage.lib.sp_copy_async(xout.data_ptr(), self.gx_out, 4 * nw, s))
                self.works.append(dist.isend(xout[:nw], dst=self.rank + 1,
                                             group=_pair(self.rank)))
            else:
                if not len(rows):  # status word only
                    check(self.stage.lib.sp_copy_async(self.plane.res_dev(slot),
                                                       self.gx_out + 4 * n * self.d, 4, s))
                check(self.stage.lib.sp_signal(self.plane.flag_dev(slot), run_id, s))
        self._reap()

    def finish(self) -> None:
        import torch
        self.stream.synchronize()
        while self.works:
            self.works.popleft().wait()
        torch.cuda.synchronize()

    def copy(self, src, dst_mask, end) -> None:
        dsts = [i for i in range(32) if (dst_mask >> i) & 1]
        self.stage.cache_copy(src, dsts, end)

    def remove(self, seq, frm) -> None:
        self.stage.cache_remove(seq, frm)


def worker_loop(model, lo, hi, rank, world, plane: ControlPlane, partitions,
                capacity, max_tokens, on_mark=None, first: int = 0,
                stage_rank=None) -> None:
    """Ranks >= 1: serve control records until SHUTDOWN (never blocks on the GPU).
    ``stage_rank`` replaces the GPU stage (``_StageRank``) -- CPU control-plane
    tests only."""
    sr = (stage_rank or _StageRank)(model, lo, hi, rank, world, plane, partitions, capacity,
                                    max_tokens, first)
    while True:
        rtype, p = plane.read(rank)
        if rtype == R_RUN:
            sr.run(*_unpack_run(p))
        elif rtype == R_COPY:
            sr.copy(*struct.unpack("<iIi", p[:12]))
        elif rtype == R_REMOVE:
            sr.remove(*struct.unpack("<ii", p[:8]))
        elif rtype == R_RESET:
            sr.stage.reset()
            sr.stream.synchronize()
        elif rtype == R_COMPACT:      # after every run queued before it
            sr.stream.synchronize()
            sr.stage.compact()
        elif rtype == R_MARK:
            sr.stream.synchronize()
            if on_mark is not None:
                on_mark(struct.unpack("<i", p[:4])[0], sr.stage.launches)
        elif rtype == R_SHUTDOWN:
            sr.finish()
            return


class DistPipeline:
    """Head-side pipeline over torchrun ranks (rank 0 = head + stage 0)."""

    def __init__(self, model, ranges, plane: ControlPlane, world: int, partitions=8,
                 capacity=8192, max_tokens=256, local_stage: bool = True, stage_rank=None):
        """``local_stage``: rank 0 hosts stage 0 (and the draft shares its
        GPU); False: rank 0 is the head + dedicated draft node and the
        stages live on ranks 1.. (the reference's n_stages = nodes - 1 with a
        draft node, engine.py:171-176)."""
        self.plane = plane
        self.world = world
        self.n_stage_ranks = len(ranges)
        self.capacity = capacity
        self.cells_since = 0       # cells appended on every stage since the last compaction
        self.compactions = 0
        self.sr = None
        self.stages = []
        if local_stage:
            lo, hi = ranges[0]
            self.sr = (stage_rank or _StageRank)(model, lo, hi, 0, world, plane, partitions,
                                                 capacity, max_tokens)
            self.stages = [self.sr.stage]
        self.fifo: deque = deque()
        self.n_stat = (world + 3) // 4

    @property
    def n_stages(self) -> int:
        return self.n_stage_ranks

    def reset(self) -> None:
        if self.fifo:
            raise RuntimeError("reset with runs in flight")
        self.plane.write(R_RESET, b"")
        self.cells_since = 0
        if self.sr is not None:
            self.sr.stage.reset()
            self.sr.stream.synchronize()
        self.plane.cancel[:] = 0
        self.plane.flags[:] = 0

    def mark(self, tag: int) -> None:
        self.plane.write(R_MARK, struct.pack("<i", tag))

    def launch(self, run_id, kind, toks, flags, rows) -> None:
        if len(self.fifo) >= RESULTS:
            raise RuntimeError("too many runs in flight")
        if self.cells_since + len(toks) > self.capacity // 2:
            # every stage reclaims its dead cells at this point of its record
            # stream (live cells <= context + in-flight speculation)
            self.plane.write(R_COMPACT, b"")
            if self.sr is not None:
                self.sr.stream.synchronize()
                self.sr.stage.compact()
            self.cells_since = 0
            self.compactions += 1
        self.cells_since += len(toks)
        self.plane.write(R_RUN, _pack_run(run_id, kind, flags, toks, rows))
        if self.sr is not None:
            self.sr.run(run_id, kind, flags, toks, rows)
        self.fifo.append((run_id, len(rows)))

    def copy(self, src, dsts, end_pos) -> None:
        m = 0
        for d in dsts:
            m |= 1 << int(d)
        self.plane.write(R_COPY, struct.pack("<iIi", src, m, end_pos))
        if self.sr is not None:
            self.sr.copy(src, m, end_pos)

    def remove(self, seq, from_pos) -> None:
        self.plane.write(R_REMOVE, struct.pack("<ii", seq, from_pos))
        if self.sr is not None:
            self.sr.remove(seq, from_pos)

    def cancel_run(self, run_id: int) -> None:
        self.plane.cancel[run_id % CANCEL] = run_id

    def ready(self) -> bool:
        if not self.fifo:
            return False
        run_id = self.fifo[0][0]
        return int(self.plane.flags[run_id % RESULTS]) == run_id

    def _collect(self) -> RunResult:
        run_id, nrow = self.fifo.popleft()
        blk = self.plane.res[run_id % RESULTS]
        status = int(blk[0])
        err = int(blk[1])
        rows = []
        if status == _lib.SP_STATUS_VALID and nrow:
            rr = blk[4:4 + 4 * nrow].view(RES_DTYPE).reshape(-1)
            rows = [RowResult(r["a"], r["b"], r["c"], r["d"]) for r in rr]
        return RunResult(run_id, status == _lib.SP_STATUS_PLACEHOLDER, rows, err,
                         [status] * self.n_stage_ranks)

    def poll(self) -> Optional[RunResult]:
        return self._collect() if self.ready() else None

    def wait(self) -> RunResult:
        if not self.fifo:
            raise RuntimeError("wait with an empty FIFO")
        while not self.ready():
            os.sched_yield()
        return self._collect()

    def in_flight(self) -> int:
        return len(self.fifo)

    def shutdown(self) -> None:
        self.plane.write(R_SHUTDOWN, b"")
        if self.sr is not None:
            self.sr.stream.synchronize()


# ---------------------------------------------------------------------------
# process-level setup
# ---------------------------------------------------------------------------

def init(max_tokens: int = 256):
    """torchrun bootstrap: NCCL for activations, gloo for host control."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # SP_DIST_GPUS=G (tests only): more ranks than GPUs, rank r on GPU r % G.
    # The world group is then gloo (NCCL refuses two ranks of one GPU in a
    # communicator); the activation pairs (r, r + 1) sit on different GPUs
    # and stay NCCL.  Timings of such a run mean nothing.
    oversub = int(os.environ.get("SP_DIST_GPUS", "0"))
    if oversub:
        local = local % oversub
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gloo = dist.new_group(backend="gloo")
    # one NCCL communicator per adjacent pair: a rank's receive (from i-1)
    # and send (to i+1) then run on different streams instead of being
    # serialised as ops of one communicator
    global _PAIRS
    _PAIRS = [dist.new_group([i, i + 1], backend="nccl") for i in range(world - 1)]
    name = [f"sp_{os.getpid()}_{uuid.uuid4().hex[:8]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0, group=gloo)
    n_stat = (world + 3) // 4
    # rank 0 creates the segment; the others attach only after the barrier
    plane = ControlPlane(name[0], True, world, max_tokens, n_stat) if rank == 0 else None
    dist.barrier(group=gloo)
    if rank != 0:
        plane = ControlPlane(name[0], False, world, max_tokens, n_stat)
    plane.register()
    dist.barrier(group=gloo)
    return rank, world, local, plane, gloo


_PAIRS: list = []


def _pair(i: int):
    return _PAIRS[i] if 0 <= i < len(_PAIRS) else None


def build_slice(cfg, rank: int, world: int, node_weights=None, first: int = 0):
    """This rank's layer range and weights (plan_layer_split, engine.py:186-224).
    Stages live on ranks first..world-1; a rank below ``first`` (the head +
    dedicated draft node) gets a one-layer shell of the target (its config and
    the roofline probe's weights)."""
    import torch
    from .engine import plan_layer_split
    from .model import build_model
    tc = cfg.target_config()
    ranges = plan_layer_split(tc.n_layers, world - first, node_weights)
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank < first:
        model = build_model(tc, dev, layer_range=(0, 1), embedding=False, head=False)
    else:
        model = build_model(tc, dev, layer_range=ranges[rank - first])
    return model, ranges


def bench_main(args):
    """bench.py under torchrun (N > 1): rank 0 runs the head, the others serve."""
    import torch
    import torch.distributed as dist
    rank, world, local, plane, gloo = init()
    import bench as B
    from .engine import Engine, ExperimentConfig
    from .model import build_model, sample_prompt
    # dedicated draft node: rank 0 = head + draft (the persistent draft kernel
    # gets the whole GPU), stages on ranks 1.. -- the reference's layout
    # (n_stages = nodes - 1); otherwise every rank hosts a stage and the draft
    # shares rank 0's GPU
    mode = getattr(args, "draft_gpu", "off")
    # measured (profiles/r02_sweep_n2_n4.txt): the dedicated layout wins at
    # N=2 (531-540 vs 416 tok/s) and N=4 (590 vs 439)
    dedicated = world >= 2 and mode in ("on", "auto")
    first = 1 if dedicated else 0
    if dedicated and rank == 0:
        os.environ.setdefault("SP_DRAFT_FUSED", "1")
        os.environ.setdefault("SP_DRAFT_KERNEL", "grid")
    cfg = ExperimentConfig(mode="async-speculative", nodes=world if dedicated else world + 1,
                           target_shape=args.target, draft_shape=args.draft,
                           draft_backend="synthetic", alpha=args.alpha,
                           prompt_len=B.PROMPT_LEN, gen_len=args.gen_len,
                           max_context=B.MAX_CTX, target_seed=1, draft_seed=2,
                           capacity=8192, node_weights=getattr(args, "node_weights", None),
                           **B.bench_knobs(args))
    model, ranges = build_slice(cfg, rank, world, cfg.node_weights, first)
    marks = []
    if rank != 0:
        lo, hi = ranges[rank - first]
        worker_loop(model, lo, hi, rank, world, plane, cfg.partitions, cfg.capacity,
                    cfg.max_run_tokens, on_mark=lambda t, nl: marks.append((t, time.perf_counter(), nl)),
                    first=first)
        out = [None]
        t = {m: v for m, v, _ in marks}
        nl = {m: c for m, _, c in marks}
        launched = (nl[2] - nl[1]) if (1 in nl and 2 in nl) else None
        dist.gather_object((t.get(1), t.get(2), launched), None, dst=0, group=gloo)
        dist.barrier(group=gloo)
        plane.close()
        dist.destroy_process_group()
        return None
    dev = torch.device("cuda", local)
    draft = build_model(cfg.draft_config(), dev, tiled=cfg.draft_tc)
    pipe = DistPipeline(model, ranges, plane, world, cfg.partitions, cfg.capacity,
                        cfg.max_run_tokens, local_stage=not dedicated)
    eng = Engine(cfg, target_model=model, draft_model=draft, pipeline=pipe)
    line = B.measure(eng, args, n_gpus=world, pipe=pipe)
    pipe.shutdown()
    times = [None] * world
    dist.gather_object((None, None, None), times, dst=0, group=gloo)
    spans = [t1 - t0 for (t0, t1, _) in times[1:] if t0 is not None and t1 is not None]
    line["rank_spans_s"] = [round(x, 4) for x in spans]
    # every rank's kernel launches in the timed region (rank 0's are in the line)
    per = [line.get("gpu_launches")] + [c for (_, _, c) in times[1:]]
    line["gpu_launches_per_rank"] = per
    line["gpu_launches"] = sum(c for c in per if c)
    dist.barrier(group=gloo)
    plane.close(unlink=True)
    dist.destroy_process_group()
    return line
