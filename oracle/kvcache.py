"""Oracle KV cache: restates ``specpipe/kvcache.py`` (TEST INFRASTRUCTURE).

Cells are appended per layer and carry a position plus a set of sequence ids;
copy/remove/free only edit membership (``kvcache.py:1-14``).  The restatement
keeps one table per covered layer exactly like the reference so that
``pad_dead`` alignment semantics (``kvcache.py:158-167``) can be replayed, and
adds ``keep`` (llama.cpp ``seq_keep``), which the reference does not have but
the north star names.
"""

from __future__ import annotations

from collections import deque

import numpy as np


class OracleCacheError(ValueError):
    pass


class OracleExhausted(Exception):
    pass


class OracleAllocator:
    """FIFO partition ids 1..P-1, id 0 canonical (``kvcache.py:33-66``)."""

    def __init__(self, partitions: int = 8):
        if partitions < 2:
            raise OracleCacheError("need >= 2 partitions")
        self.partitions = partitions
        self.free_ids = deque(range(1, partitions))
        self.live_ids = set()

    def alloc(self) -> int:
        if not self.free_ids:
            raise OracleExhausted("no free partition")
        s = self.free_ids.popleft()
        self.live_ids.add(s)
        return s

    def free(self, s: int) -> None:
        if s == 0 or s not in self.live_ids:
            raise OracleCacheError(f"bad free of {s}")
        self.live_ids.remove(s)
        self.free_ids.append(s)

    def available(self) -> int:
        return len(self.free_ids)

    def live(self):
        return sorted(self.live_ids)

    def all_ids(self):
        return list(range(1, self.partitions))


class _LayerTable:
    def __init__(self, dim: int, n_seq: int):
        self.pos: list = []
        self.member: list = []          # list of python sets
        self.k: list = []
        self.v: list = []
        self.dim = dim
        self.n_seq = n_seq


class OracleCache:
    """Per-layer append-only cells (``kvcache.py:94-283``)."""

    def __init__(self, dim: int, layers, max_context: int, n_seq_ids: int = 8):
        self.dim = dim
        self.layers = tuple(layers)
        if not self.layers:
            raise OracleCacheError("no layers")
        self.max_context = max_context
        self.n_seq_ids = n_seq_ids
        self.t = {l: _LayerTable(dim, n_seq_ids) for l in self.layers}

    # kvcache.py:135-156
    def insert(self, layer, pos, seqs, key, value) -> int:
        if layer not in self.t:
            raise OracleCacheError("layer not covered")
        seqs = set(int(s) for s in seqs)
        if not seqs:
            raise OracleCacheError("cell needs a sequence")
        if not 0 <= pos < self.max_context:
            raise OracleCacheError("position out of range")
        if any(not 0 <= s < self.n_seq_ids for s in seqs):
            raise OracleCacheError("sequence id out of range")
        tb = self.t[layer]
        tb.pos.append(int(pos))
        tb.member.append(seqs)
        tb.k.append(np.array(key, dtype=np.float64))
        tb.v.append(np.array(value, dtype=np.float64))
        return len(tb.pos) - 1

    # kvcache.py:158-167
    def pad_dead(self, layer, positions) -> None:
        tb = self.t[layer]
        for p in positions:
            tb.pos.append(int(p))
            tb.member.append(set())
            tb.k.append(np.zeros(self.dim))
            tb.v.append(np.zeros(self.dim))

    @property
    def n_cells(self) -> int:
        return len(self.t[self.layers[0]].pos)

    # kvcache.py:181-204: destination keeps any position it already holds;
    # the occupied set of each destination is taken before that destination
    # is updated, the candidate set once before the loop.
    def copy(self, src, dsts, end_pos) -> None:
        dsts = sorted(set(int(d) for d in dsts))
        for layer in self.layers:
            tb = self.t[layer]
            cand = [i for i, (p, m) in enumerate(zip(tb.pos, tb.member))
                    if src in m and p < end_pos]
            if not cand:
                continue
            for d in dsts:
                if d == src:
                    continue
                occupied = {p for p, m in zip(tb.pos, tb.member) if d in m}
                for i in cand:
                    if tb.pos[i] not in occupied:
                        tb.member[i].add(d)

    # kvcache.py:206-216
    def remove(self, seq, from_pos) -> None:
        for layer in self.layers:
            tb = self.t[layer]
            for p, m in zip(tb.pos, tb.member):
                if p >= from_pos:
                    m.discard(seq)

    # kvcache.py:218-222
    def free_sequence(self, seq) -> None:
        if seq == 0:
            raise OracleCacheError("cannot free canonical")
        self.remove(seq, 0)

    # llama.cpp seq_keep semantics (not in the reference): every cell that
    # belongs to ``seq`` keeps only ``seq``; every other cell dies.
    def keep(self, seq) -> None:
        for layer in self.layers:
            tb = self.t[layer]
            for i, m in enumerate(tb.member):
                tb.member[i] = {seq} if seq in m else set()

    # kvcache.py:230-238: rows visible to seq below query_pos, stable by pos
    def visible_rows(self, seq, query_pos, layer):
        tb = self.t[layer]
        rows = [i for i, (p, m) in enumerate(zip(tb.pos, tb.member))
                if seq in m and p < query_pos]
        rows.sort(key=lambda i: (tb.pos[i], i))
        return rows

    def visible_positions(self, seq, query_pos, layer):
        tb = self.t[layer]
        return [tb.pos[i] for i in self.visible_rows(seq, query_pos, layer)]

    # kvcache.py:260-276: live cells (position, frozenset) in row order
    def snapshot(self, layer=None):
        layer = self.layers[0] if layer is None else layer
        tb = self.t[layer]
        return [(p, frozenset(m)) for p, m in zip(tb.pos, tb.member) if m]

    def seq_positions(self, seq, layer=None):
        layer = self.layers[0] if layer is None else layer
        tb = self.t[layer]
        return sorted(p for p, m in zip(tb.pos, tb.member) if seq in m)

    def key(self, layer, row):
        return self.t[layer].k[row]

    def value(self, layer, row):
        return self.t[layer].v[row]
