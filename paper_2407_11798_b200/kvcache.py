"""Sequence-partitioned KV cache (mirror of ``specpipe/kvcache.py``) on the GPU.

Cells carry a position and a sequence bitmask; copy/remove/free/keep edit
membership only (kvcache.py:1-14).  One metadata table serves every layer of
a stage (the reference keeps identical per-layer tables, kvcache.py:96-100);
K/V rows live in HBM next to it and are written once by the QKV epilogue.
Sequence id 0 is canonical; 1..P-1 are FIFO partitions.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Iterable, List

import numpy as np

from .errors import AllocationExhausted, CacheError
from .model import BatchToken, ModelConfig, encode_tokens


class SequenceAllocator:
    """FIFO pool of speculative sequence ids 1..P-1 (kvcache.py:33-66)."""

    def __init__(self, partitions: int = 8):
        if partitions < 2:
            raise CacheError("need at least 2 partitions (canonical + 1)")
        if partitions > 32:
            raise CacheError("at most 32 partitions (one bit each in the cell mask)")
        self.partitions = partitions
        self._free = deque(range(1, partitions))
        self._live = set()

    def alloc(self) -> int:
        if not self._free:
            raise AllocationExhausted(f"all {self.partitions - 1} partitions in use")
        seq = self._free.popleft()
        self._live.add(seq)
        return seq

    def free(self, seq: int) -> None:
        if seq == 0:
            raise CacheError("cannot free the canonical sequence")
        if seq not in self._live:
            raise CacheError(f"sequence {seq} is not allocated (double free?)")
        self._live.discard(seq)
        self._free.append(seq)

    def available(self) -> int:
        return len(self._free)

    def live(self) -> List[int]:
        return sorted(self._live)

    def all_ids(self) -> List[int]:
        return list(range(1, self.partitions))


@dataclass(frozen=True)
class KVCell:
    """Read-only view of one cell (kvcache.py:69-77)."""

    layer: int
    position: int
    sequences: frozenset
    key: np.ndarray
    value: np.ndarray


class CacheView(list):
    """Ordered (position, sequence_set) pairs of live cells plus raw rows."""

    def __init__(self, cells, rows):
        super().__init__(cells)
        self.rows = rows


def _mask_to_set(m: int) -> frozenset:
    return frozenset(i for i in range(32) if (int(m) >> i) & 1)


class KVCache:
    """Per-stage cell table + K/V rows on the GPU (kvcache.py:94-283).

    ``KVCache(embed_dim, layers, max_context, n_seq_ids)`` matches the
    reference constructor.  The device storage is created when the cache is
    first bound to a model by ``eval_layers`` (K/V widths depend on the
    model); a cache used before that (metadata-only, e.g. trace replay) gets
    a minimal table.  ``capacity`` bounds the cell pool (the reference grows
    without bound).
    """

    def __init__(self, embed_dim: int, layers: Iterable[int], max_context: int,
                 n_seq_ids: int = 8, capacity: int = 4096, max_tokens: int = 256,
                 model=None):
        self.embed_dim = embed_dim
        self.layers = tuple(layers)
        if not self.layers:
            raise CacheError("cache must cover at least one layer")
        if list(self.layers) != list(range(self.layers[0], self.layers[-1] + 1)):
            raise CacheError("a stage cache covers a contiguous layer range")
        if not 1 <= n_seq_ids <= 32:
            raise CacheError("n_seq_ids must be within [1, 32]")
        self.max_context = max_context
        self.n_seq_ids = n_seq_ids
        self.capacity = capacity
        self.max_tokens = max_tokens
        self._stage = None
        self._model = None
        if model is not None:
            self._bind(model)

    # -- binding --------------------------------------------------------------
    def _bind(self, model):
        if self._model is model and self._stage is not None:
            return self._stage
        from .runtime import Stage
        if self._stage is not None and self._stage.n_cells() > 0 and self._model is not None:
            raise CacheError("cache already bound to another model")
        if model.config.max_context != self.max_context:
            raise CacheError("cache/model max_context mismatch")
        if self._stage is not None and self._stage.n_cells() > 0:
            raise CacheError("cannot bind a model to a cache that already holds "
                             "metadata-only cells")
        lo, hi = self.layers[0], self.layers[-1] + 1
        self._stage = Stage(model, lo, hi, capacity=self.capacity,
                            max_tokens=self.max_tokens, n_seq_ids=self.n_seq_ids)
        self._model = model
        return self._stage

    @property
    def stage(self):
        if self._stage is None:
            self._meta_only()
        return self._stage

    def _meta_only(self):
        import torch
        from .model import DeviceModel
        from .runtime import Stage
        n_layers = self.layers[-1] + 1
        cfg = ModelConfig(vocab_size=2, embed_dim=16, n_layers=n_layers, n_heads=1,
                          max_context=self.max_context, seed=0)
        m = DeviceModel(cfg, torch.device("cuda"), (self.layers[0], n_layers))
        z = torch.zeros(16 * 16 * 4, dtype=torch.float32, device="cuda")
        for l in self.layers:
            m.layers[l] = dict(qkv=z, o=z, up=z, down=z, attn_norm=None, mlp_norm=None)
        m.embedding = z
        self._stage = Stage(m, self.layers[0], n_layers, capacity=self.capacity,
                            max_tokens=self.max_tokens, n_seq_ids=self.n_seq_ids)

    # -- storage ---------------------------------------------------------------
    def insert(self, pos: int, seqs: Iterable[int]) -> int:
        """Append one cell to every covered layer (metadata; K/V unset)."""
        seqs = sorted(set(int(s) for s in seqs))
        if not seqs:
            raise CacheError("cell must belong to at least one sequence")
        if not 0 <= pos < self.max_context:
            raise CacheError(f"position {pos} outside [0, {self.max_context})")
        for s in seqs:
            if not 0 <= s < self.n_seq_ids:
                raise CacheError(f"sequence id {s} outside [0, {self.n_seq_ids})")
        row = self.n_cells
        self.stage.insert_meta(encode_tokens([BatchToken(0, pos, frozenset(seqs))]))
        return row

    @property
    def n_cells(self) -> int:
        return 0 if self._stage is None else self._stage.n_cells()

    def keys(self, layer: int, rows) -> np.ndarray:
        return np.stack([self._stage.read_kv_sync(layer, int(r))[0] for r in rows])

    def values(self, layer: int, rows) -> np.ndarray:
        return np.stack([self._stage.read_kv_sync(layer, int(r))[1] for r in rows])

    # -- metadata operations (one table: all layers at once) --------------------
    def copy(self, src: int, dsts: Iterable[int], end_pos: int) -> None:
        self._check_seq(src)
        dsts = sorted(set(int(d) for d in dsts))
        for d in dsts:
            self._check_seq(d)
        if self.n_cells:
            self.stage.cache_copy(src, dsts, end_pos)

    def remove(self, seq: int, from_pos: int) -> None:
        self._check_seq(seq)
        if self.n_cells:
            self.stage.cache_remove(seq, from_pos)

    def free_sequence(self, seq: int) -> None:
        if seq == 0:
            raise CacheError("cannot free the canonical sequence")
        self.remove(seq, 0)

    def keep(self, seq: int) -> None:
        """llama.cpp seq_keep: drop every other sequence's membership."""
        self._check_seq(seq)
        if self.n_cells:
            self.stage.cache_keep(seq)

    def _check_seq(self, s: int) -> None:
        if not 0 <= s < self.n_seq_ids:
            raise CacheError(f"sequence id {s} outside [0, {self.n_seq_ids})")

    # -- queries (synchronous D2H of the metadata) -----------------------------
    def _meta(self):
        if self._stage is None or self.n_cells == 0:
            return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.uint32)
        return self._stage.meta_sync()

    def visible_rows(self, seq: int, query_pos: int, layer: int = None) -> np.ndarray:
        pos, mask = self._meta()
        vis = ((mask >> np.uint32(seq)) & 1).astype(bool) & (pos < query_pos)
        rows = np.where(vis)[0]
        return rows[np.argsort(pos[rows], kind="stable")]

    def visible_positions(self, seq: int, query_pos: int, layer: int = None) -> np.ndarray:
        pos, _ = self._meta()
        return pos[self.visible_rows(seq, query_pos)]

    def visible_cells(self, seq: int, query_pos: int, layer: int) -> List[KVCell]:
        pos, mask = self._meta()
        out = []
        for r in self.visible_rows(seq, query_pos):
            k, v = self._stage.read_kv_sync(layer, int(r))
            out.append(KVCell(layer, int(pos[r]), _mask_to_set(mask[r]), k, v))
        return out

    def snapshot(self, layer: int = None) -> CacheView:
        pos, mask = self._meta()
        rows = np.where(mask != 0)[0]
        return CacheView([(int(pos[r]), _mask_to_set(mask[r])) for r in rows], rows)

    def seq_positions(self, seq: int, layer: int = None) -> np.ndarray:
        pos, mask = self._meta()
        return np.sort(pos[((mask >> np.uint32(seq)) & 1).astype(bool)])


def free_sequence(cache: KVCache, allocator: SequenceAllocator, seq: int) -> None:
    """Release a partition (kvcache.py:286-289)."""
    allocator.free(seq)
    cache.free_sequence(seq)
