"""Python handle over one ``sp_stage`` (C ABI: include/specpipe_b200.h).

A ``Stage`` owns a contiguous layer range of a ``DeviceModel`` on one GPU:
its cell table and K/V rows, its activation buffer and a result block.  All
work is enqueued on ``self.stream``; only the explicit ``*_sync`` helpers
and the API-mirror conveniences (``eval_batch``, ``decode_step``) wait.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check
from .errors import CacheError, ModelError
from .model import KIND_CODE, PREFILL, RowResult, encode_tokens

RES_DTYPE = np.dtype([("a", "<i4"), ("b", "<i4"), ("c", "<f4"), ("d", "<f4")])


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_contiguous():
        raise ModelError("device weights must be contiguous (row-major [d_out, d_in])")
    return t.data_ptr()


class Stage:
    def __init__(self, model, lo: int, hi: int, capacity: int = 4096,
                 max_tokens: int = 256, n_seq_ids: int = 8, stream=None,
                 cancel_table=None, cancel_size: int = 0):
        import torch

        self.lib = _lib.load()
        self.model = model
        cfg = model.config
        self.cfg = cfg
        self.lo, self.hi = lo, hi
        self.capacity, self.max_tokens, self.n_seq = capacity, max_tokens, n_seq_ids
        self.device = model.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._dims = cfg.dims(tiled=getattr(model, "tiled", None), swz=getattr(model, "swz", False))
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.sp_stage_create(C.byref(self._dims), lo, hi, capacity,
                                           max_tokens, n_seq_ids, C.byref(h)),
                  "sp_stage_create")
        self.h = h
        if lo == 0:
            if model.embedding is None:
                raise ModelError("stage 0 needs the embedding")
            check(self.lib.sp_stage_set_embedding(h, _ptr(model.embedding),
                                                  _ptr(model.pos_table)))
        for l in range(lo, hi):
            L = model.layers.get(l)
            if L is None:
                raise ModelError(f"layer {l} not materialised in this model slice")
            check(self.lib.sp_stage_set_layer(h, l, _ptr(L["qkv"]), _ptr(L["o"]),
                                              _ptr(L["up"]), _ptr(L["down"]),
                                              _ptr(L["attn_norm"]),
                                              _ptr(L["mlp_norm"])))
        if hi == cfg.n_layers and model.w_out is not None:
            check(self.lib.sp_stage_set_head(h, _ptr(model.w_out), _ptr(model.final_norm)))
            if getattr(model, "w_out_tc", None) is not None and \
                    os.environ.get("SP_LMHEAD_CUDA_CORES") != "1":
                check(self.lib.sp_stage_set_head_tiled(h, _ptr(model.w_out_tc)),
                      "sp_stage_set_head_tiled")
        if cancel_table is not None:
            self.set_cancel_table(cancel_table, cancel_size)
        d = cfg.embed_dim
        self.x = torch.zeros((max_tokens, d), dtype=torch.float32, device=self.device)
        self.xin = torch.zeros((max_tokens, d), dtype=torch.float32, device=self.device)
        # result block: row 0 = [status, err, n_rows, run_id], rows 1.. = sp_row_result
        self.res = torch.zeros((max_tokens + 1, 4), dtype=torch.int32, device=self.device)
        self.res_host = torch.zeros((max_tokens + 1, 4), dtype=torch.int32).pin_memory()
        self.logits_dev = None
        self._last_batch = None
        self._last_hi = None
        self.launches = 0
        # buffers were zero-filled on the creating stream: order them before
        # any kernel on self.stream can touch them
        torch.cuda.synchronize(self.device)

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                self.lib.sp_stage_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    # -- plumbing -------------------------------------------------------------
    @property
    def s(self) -> int:
        return self.stream.cuda_stream

    def set_cancel_table(self, table, size: int) -> None:
        self._cancel_table = table  # keep alive
        ptr = table if isinstance(table, int) else table.data_ptr()
        check(self.lib.sp_stage_set_cancel_table(self.h, ptr, size))

    def set_cta_budget(self, ctas: int) -> None:
        """Cap the CTAs of this stage's tensor-core GEMMs (leaves SMs free
        for a stream co-scheduled on the same GPU, e.g. the draft)."""
        check(self.lib.sp_stage_set_cta_budget(self.h, int(ctas)))

    def n_cells(self) -> int:
        return self.lib.sp_stage_n_cells(self.h)

    # -- enqueue-only primitives -------------------------------------------------
    def forward(self, toks: np.ndarray, run_id: int, kind: int, flags: int,
                x_in: Optional[int] = None, in_status: Optional[int] = None,
                x_out: Optional[int] = None, out_status: Optional[int] = None,
                chain: bool = False, layer_a: int = -1, layer_b: int = -1) -> None:
        n = len(toks)
        rc = self.lib.sp_stage_forward_range(
            self.h, toks.ctypes.data, n, run_id, kind, flags, x_in, in_status,
            x_out if x_out is not None else self.x.data_ptr(), out_status,
            1 if chain else 0, layer_a, layer_b, self.s)
        check(rc, "sp_stage_forward")
        nl = (self.hi - self.lo) if layer_a < 0 else (layer_b - layer_a)
        self.launches += 5 * nl + (2 if flags & _lib.SP_FWD_CONTINUE else 4)

    def step(self, toks: np.ndarray, run_id: int, kind: int, flags: int,
             rows: Sequence[int] = (), head: int = 0, cutoff: float = 0.0,
             x_in: Optional[int] = None, in_status: Optional[int] = None,
             res_copy: Optional[int] = None) -> None:
        """One whole stage-run (+ fused LM head over ``rows``) through the
        graph-cached ``sp_stage_step``: outputs land in the stage's fixed
        buffers (``io()``); the result block [status, err, -, -] + rows is
        copied to ``res_copy`` (device or pinned host) when given."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        rc = self.lib.sp_stage_step(self.h, toks.ctypes.data, len(toks), run_id, kind, flags,
                                    r.ctypes.data if len(r) else None, len(r), int(head),
                                    float(cutoff), x_in, in_status, res_copy, self.s)
        check(rc, "sp_stage_step")
        self.launches += 5 * (self.hi - self.lo) + 4 + (2 if len(r) else 0)

    def decode_chain(self, feed: Sequence[int], pos0: int, steps: int, cutoff: float,
                     out: int, err_out: int, step_tokens: Optional[Sequence[int]] = None) -> None:
        """A whole draft request in one persistent launch (K15): forward the
        fed tokens, then ``steps`` chained (or given) single-token steps;
        row results -> ``out[0..steps]``."""
        f = np.ascontiguousarray(feed, dtype=np.int32)
        st = None if step_tokens is None else np.ascontiguousarray(step_tokens, dtype=np.int32)
        rc = self.lib.sp_stage_decode_chain(
            self.h, f.ctypes.data if len(f) else None, len(f), int(pos0),
            None if st is None else st.ctypes.data, int(steps), float(cutoff), out, err_out,
            self.s)
        check(rc, "sp_stage_decode_chain")
        self.launches += 1

    def compact(self) -> int:
        """Reclaim dead cells (stable; synchronises the stream); new count."""
        rc = self.lib.sp_stage_compact(self.h, self.s)
        if rc < 0:
            check(-rc, "sp_stage_compact")
        return rc

    def set_skip_graphs(self, on: bool) -> None:
        """Conditional (IF) graph bodies for cancellable stage-runs (see
        sp_stage_set_skip_graphs)."""
        check(self.lib.sp_stage_set_skip_graphs(self.h, 1 if on else 0), "sp_stage_set_skip_graphs")

    def truncate(self, n_cells: int) -> None:
        check(self.lib.sp_stage_truncate(self.h, int(n_cells)), "sp_stage_truncate")

    def io(self):
        """(x_out, result block) device pointers written by ``step``."""
        x, r = C.c_void_p(), C.c_void_p()
        check(self.lib.sp_stage_io(self.h, C.byref(x), C.byref(r)), "sp_stage_io")
        return x.value, r.value

    def lmhead(self, rows: Sequence[int], x: Optional[int] = None,
               out: Optional[int] = None, logits: Optional[int] = None,
               err_out: Optional[int] = None, update_tip: bool = False,
               chain_gate: bool = False, cutoff: float = 0.0) -> None:
        r = np.ascontiguousarray(rows, dtype=np.int32)
        rc = self.lib.sp_stage_lmhead(
            self.h, x if x is not None else self.x.data_ptr(), r.ctypes.data, len(r),
            out if out is not None else self.res[1:].data_ptr(), logits,
            err_out if err_out is not None else self.res[0, 1:].data_ptr(),
            1 if update_tip else 0, 1 if chain_gate else 0, float(cutoff), self.s)
        check(rc, "sp_stage_lmhead")
        self.launches += 2

    def cache_copy(self, src: int, dsts, end_pos: int) -> None:
        mask = 0
        for dd in dsts:
            if not 0 <= dd < self.n_seq:
                raise CacheError(f"sequence id {dd} outside [0, {self.n_seq})")
            mask |= 1 << int(dd)
        check(self.lib.sp_stage_cache_copy(self.h, int(src), mask, int(end_pos), self.s),
              "cache_copy")
        self.launches += 1

    def cache_remove(self, seq: int, from_pos: int) -> None:
        check(self.lib.sp_stage_cache_remove(self.h, int(seq), int(from_pos), self.s),
              "cache_remove")
        self.launches += 1

    def cache_keep(self, seq: int) -> None:
        check(self.lib.sp_stage_cache_keep(self.h, int(seq), self.s), "cache_keep")

    def insert_meta(self, toks: np.ndarray) -> None:
        check(self.lib.sp_stage_cache_insert_meta(self.h, toks.ctypes.data, len(toks), self.s),
              "insert_meta")

    def reset(self) -> None:
        check(self.lib.sp_stage_reset(self.h, self.s))
        self._last_batch = None

    def chain_begin(self, cutoff: float, out: int) -> None:
        check(self.lib.sp_stage_chain_begin(self.h, float(cutoff), out, self.s))

    def invalidate_tip(self) -> None:
        check(self.lib.sp_stage_invalidate_tip(self.h, self.s))

    # -- blocking queries ----------------------------------------------------
    def meta_sync(self):
        n = self.n_cells()
        pos = np.zeros(max(n, 1), dtype=np.int32)
        mask = np.zeros(max(n, 1), dtype=np.uint32)
        check(self.lib.sp_stage_meta_sync(self.h, pos.ctypes.data, mask.ctypes.data,
                                          len(pos), self.s))
        return pos[:n].astype(np.int64), mask[:n]

    def error_sync(self, clear: bool = True) -> int:
        v = self.lib.sp_stage_error_sync(self.h, 1 if clear else 0, self.s)
        if v < 0:
            raise RuntimeError("sp_stage_error_sync failed (CUDA error)")
        return v

    def plan_sync(self, n: int):
        ld = self.lib.sp_stage_ld_vis(self.h)
        vis = np.zeros((n, ld), dtype=np.int32)
        ln = np.zeros(n, dtype=np.int32)
        check(self.lib.sp_stage_plan_sync(self.h, vis.ctypes.data, ln.ctypes.data, n, self.s))
        return [vis[i, :ln[i]].tolist() for i in range(n)]

    def plan_only_sync(self, toks: np.ndarray, check_coverage: bool = False):
        check(self.lib.sp_stage_plan_only(self.h, toks.ctypes.data, len(toks),
                                          1 if check_coverage else 0, self.s))
        return self.plan_sync(len(toks))

    def read_kv_sync(self, layer: int, row: int):
        k = np.zeros(self.cfg.kv_dim, dtype=np.float32)
        v = np.zeros(self.cfg.kv_dim, dtype=np.float32)
        check(self.lib.sp_stage_read_kv_sync(self.h, layer, row, k.ctypes.data,
                                             v.ctypes.data, self.s))
        return k, v

    def synchronize(self) -> None:
        self.stream.synchronize()

    def raise_errors(self, where: str) -> None:
        bits = self.error_sync(clear=True)
        _lib.raise_device_error(bits, where)

    # -- API-mirror conveniences (synchronous) ------------------------------------
    def continues(self, batch, lo: int) -> bool:
        """Is (batch, lo) the next sub-range of the previous eval_batch?"""
        return batch is self._last_batch and lo == self._last_hi

    def ld_vis(self) -> int:
        return self.lib.sp_stage_ld_vis(self.h)

    def eval_batch(self, batch, lo: int, hi: int, x_in, plan=None) -> np.ndarray:
        """eval_layers on this stage's cache; continuation of a split range.
        ``plan``: (vis, len) rows from a caller's TreeAttentionMask."""
        toks = encode_tokens(batch.tokens)
        n = len(toks)
        if n > self.max_tokens:
            raise CacheError(f"batch of {n} exceeds max_tokens {self.max_tokens}")
        flags = _lib.SP_FWD_CONTINUE if self.continues(batch, lo) else 0
        if plan is not None and not flags:
            vis, ln = plan
            vis = np.ascontiguousarray(vis, dtype=np.int32)
            ln = np.ascontiguousarray(ln, dtype=np.int32)
            check(self.lib.sp_stage_set_plan(self.h, vis.ctypes.data, ln.ctypes.data, n, self.s),
                  "sp_stage_set_plan")
        if x_in is not None:
            self.xin[:n].copy_(x_in)
        with_stream = self.stream
        import torch
        with torch.cuda.stream(with_stream):
            self.forward(toks, run_id=0, kind=KIND_CODE.get(batch.kind, 0), flags=flags,
                         x_in=self.xin.data_ptr() if lo > 0 else None,
                         layer_a=lo, layer_b=hi)
            out = self.x[:n].float().cpu().numpy()
        self.raise_errors("eval_layers")
        self._last_batch, self._last_hi = batch, hi
        return out

    def decode_step(self, batch, full_logits: bool = False):
        """Forward the whole stage + fused head on the flagged rows; returns the
        last flagged row (RowResult, or float64 logits if ``full_logits``)."""
        import torch
        toks = encode_tokens(batch.tokens)
        idx = [i for i, t in enumerate(batch.tokens) if t.want_logits]
        self.forward(toks, run_id=0, kind=KIND_CODE.get(batch.kind, 0), flags=0)
        logits_ptr = None
        if full_logits:
            if self.logits_dev is None:
                self.logits_dev = torch.zeros((self.max_tokens, self.cfg.vocab_size),
                                              dtype=torch.float32, device=self.device)
            logits_ptr = self.logits_dev.data_ptr()
        self.lmhead(idx, logits=logits_ptr)
        nb = len(idx) + 1
        self.res_host[:nb].copy_(self.res[:nb], non_blocking=True)
        self.stream.synchronize()
        hdr = self.res_host[0].numpy()
        _lib.raise_device_error(int(hdr[1]), "decode")
        if full_logits:
            return self.logits_dev[len(idx) - 1].double().cpu().numpy()
        r = self.res_host[len(idx)].numpy().view(RES_DTYPE)[0]
        return RowResult(r["a"], r["b"], r["c"], r["d"])


def head_logits(model, acts: np.ndarray, idx) -> np.ndarray:
    """Full-logit rows for the flagged activations (parity/debug path)."""
    import torch
    st = getattr(model, "_head_stage", None)
    n = len(acts)
    if st is None or st.max_tokens < n:
        L = model.config.n_layers
        st = Stage(model, L - 1, L, capacity=16, max_tokens=max(16, n), n_seq_ids=1)
        model._head_stage = st
    if st.logits_dev is None or st.logits_dev.shape[0] < st.max_tokens:
        st.logits_dev = torch.zeros((st.max_tokens, model.config.vocab_size),
                                    dtype=torch.float32, device=model.device)
    st.x[:n].copy_(torch.from_numpy(np.ascontiguousarray(acts, dtype=np.float32)))
    st.lmhead(idx, logits=st.logits_dev.data_ptr())
    out = st.logits_dev[:len(idx)].double().cpu().numpy()
    st.stream.synchronize()
    st.raise_errors("logits")
    return out
