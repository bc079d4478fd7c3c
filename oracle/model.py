"""Oracle decoder: float64 restatement of ``specpipe/model.py`` (TEST INFRASTRUCTURE).

Two architectures:

* ``ref``   — the reference's toy decoder, restated from ``model.py``:
  sinusoidal additive positions (``model.py:153-159``), gain-less RMSNorm with
  eps 1e-8 inside the mean (``model.py:188-189``), tanh-GELU MLP of width 4d
  (``model.py:192-194``), weights drawn from PCG64 in the documented order
  (``model.py:162-185``).  Pinned against the reference's own outputs.
* ``llama`` — RMSNorm with gain, rotate-half RoPE, GQA, SwiGLU.  Not in the
  reference; weights are supplied by the caller (the product's
  own bf16 weights, widened to float64) and parity is internal.

Evaluation is strictly per token with the reference's gather order: visible
cells sorted by (position, cache-before-batch, index) with the query itself
last (``model.py:287-323``, ``model.py:394-415``).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .kvcache import OracleCache


class OracleModelError(ValueError):
    pass


@dataclass(frozen=True)
class OracleConfig:
    vocab_size: int = 256
    embed_dim: int = 64
    n_layers: int = 12
    n_heads: int = 1
    max_context: int = 1024
    seed: int = 0
    arch: str = "ref"               # "ref" | "llama"
    n_kv_heads: Optional[int] = None
    ffn_dim: Optional[int] = None
    norm_eps: float = 1e-5          # llama only; ref uses 1e-8 inside the mean
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.n_heads

    @property
    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def hidden(self) -> int:
        return 4 * self.embed_dim if self.ffn_dim is None else self.ffn_dim


@dataclass
class OracleModel:
    cfg: OracleConfig
    embedding: np.ndarray                 # [V, d]
    pos_table: Optional[np.ndarray]       # [max_context, d] (ref only)
    layers: List[dict]                    # [d_in, d_out] matrices (h @ W)
    w_out: np.ndarray                     # [d, V]
    final_norm: Optional[np.ndarray] = None   # llama gain

    def checksum(self) -> str:
        """sha256 in the reference's order (``model.py:137-145``)."""
        h = hashlib.sha256()
        h.update(self.embedding.tobytes())
        h.update(self.pos_table.tobytes())
        for lw in self.layers:
            for name in ("wq", "wk", "wv", "wo", "w1", "w2"):
                h.update(lw[name].tobytes())
        h.update(self.w_out.tobytes())
        return h.hexdigest()


# -- ref architecture ---------------------------------------------------------

def position_table(max_context: int, dim: int) -> np.ndarray:
    """Sinusoidal table (``model.py:153-159``): column i uses frequency
    10000^(2*floor(i/2)/dim), sine on even columns and cosine on odd."""
    p = np.arange(max_context, dtype=np.float64).reshape(-1, 1)
    col = np.arange(dim, dtype=np.float64).reshape(1, -1)
    ang = p / np.power(10000.0, 2.0 * np.floor(col / 2.0) / dim)
    return np.where(col % 2 == 0, np.sin(ang), np.cos(ang)).astype(np.float64)


def build_ref_model(cfg: OracleConfig) -> OracleModel:
    """PCG64 draws: embedding, per layer wq wk wv wo w1 w2, then w_out
    (``model.py:162-185``); scaling 1/sqrt(fan_in), residual branches
    additionally 1/sqrt(2L)."""
    if cfg.vocab_size < 2 or cfg.n_layers < 1 or cfg.embed_dim % cfg.n_heads:
        raise OracleModelError("invalid config")
    g = np.random.Generator(np.random.PCG64(cfg.seed))
    d, hid = cfg.embed_dim, 4 * cfg.embed_dim
    r = 1.0 / math.sqrt(2.0 * cfg.n_layers)
    emb = g.standard_normal((cfg.vocab_size, d))
    pos = position_table(cfg.max_context, d)
    layers = []
    for _ in range(cfg.n_layers):
        lw = {}
        lw["wq"] = g.standard_normal((d, d)) / math.sqrt(d)
        lw["wk"] = g.standard_normal((d, d)) / math.sqrt(d)
        lw["wv"] = g.standard_normal((d, d)) / math.sqrt(d)
        lw["wo"] = g.standard_normal((d, d)) / math.sqrt(d) * r
        lw["w1"] = g.standard_normal((d, hid)) / math.sqrt(d)
        lw["w2"] = g.standard_normal((hid, d)) / math.sqrt(hid) * r
        layers.append(lw)
    w_out = g.standard_normal((d, cfg.vocab_size)) / math.sqrt(d)
    return OracleModel(cfg, emb, pos, layers, w_out)


def rmsnorm_ref(v: np.ndarray) -> np.ndarray:
    """``model.py:188-189``: v / sqrt(v.v/d + 1e-8), no gain."""
    return v / math.sqrt(float(v @ v) / v.shape[0] + 1e-8)


def gelu_tanh(v: np.ndarray) -> np.ndarray:
    """``model.py:192-194``."""
    return 0.5 * v * (1.0 + np.tanh(0.7978845608028654 * (v + 0.044715 * v * v * v)))


# -- llama architecture (extension, no reference counterpart) ------------------

def rmsnorm_gain(v: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    return v / math.sqrt(float(v @ v) / v.shape[0] + eps) * g


def rope_rotate_half(x: np.ndarray, pos: int, n_heads: int, hd: int,
                     theta: float) -> np.ndarray:
    half = hd // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    ang = pos * inv
    c, s = np.cos(ang), np.sin(ang)
    out = np.empty_like(x)
    for h in range(n_heads):
        a = x[h * hd: h * hd + half]
        b = x[h * hd + half: (h + 1) * hd]
        out[h * hd: h * hd + half] = a * c - b * s
        out[h * hd + half: (h + 1) * hd] = b * c + a * s
    return out


def silu(v: np.ndarray) -> np.ndarray:
    return v / (1.0 + np.exp(-v))


# -- shared evaluation ----------------------------------------------------------

def _plans(tokens, cache: OracleCache, layer: int):
    """Per query: merged visible entries (src, idx) ordered by
    (pos, cache-before-batch, index) — ``model.py:262-323``."""
    tb = cache.t[layer]
    out = []
    for i, (_, qpos, qseqs, _) in enumerate(tokens):
        ent = []
        for r, (p, m) in enumerate(zip(tb.pos, tb.member)):
            if p < qpos and not m.isdisjoint(qseqs):
                ent.append((p, 0, r))
        for j, (_, p, s, _) in enumerate(tokens):
            if j != i and p < qpos and not s.isdisjoint(qseqs):
                ent.append((p, 1, j))
        ent.sort()
        out.append([(src, idx) for (_, src, idx) in ent])
    return out


def visible_counts(tokens, cache: OracleCache, layer: Optional[int] = None):
    layer = cache.layers[0] if layer is None else layer
    return [len(p) for p in _plans(tokens, cache, layer)]


def eval_layers(model: OracleModel, lo: int, hi: int,
                x_in: Optional[np.ndarray], tokens: Sequence,
                cache: OracleCache, plans: Optional[list] = None) -> np.ndarray:
    """Layers [lo, hi) over a token batch (``model.py:326-421``).

    ``tokens``: sequence of (token_id, pos, frozenset(seqs), want_logits).
    ``plans``: a caller-supplied mask (``model.py:369-373``) as per-query
    ``[(src, idx)]`` lists (src 0 = raw cache row, 1 = batch index), in
    gather order; default: derived from cache membership.
    """
    cfg = model.cfg
    if not 0 <= lo < hi <= cfg.n_layers:
        raise OracleModelError("bad layer range")
    n, d = len(tokens), cfg.embed_dim
    if lo == 0:
        x = np.empty((n, d))
        for i, (t, p, _, _) in enumerate(tokens):
            if not 0 <= t < cfg.vocab_size or p >= cfg.max_context:
                raise OracleModelError("token/pos out of range")
            x[i] = model.embedding[t]
            if cfg.arch == "ref":
                x[i] = x[i] + model.pos_table[p]
    else:
        if x_in is None or x_in.shape != (n, d):
            raise OracleModelError("bad input activations")
        x = np.array(x_in, dtype=np.float64)
    if plans is None:
        plans = _plans(tokens, cache, lo)
    H, hd, KH = cfg.n_heads, cfg.head_dim, cfg.kv_heads
    grp = H // KH
    scale = 1.0 / math.sqrt(hd)
    for layer in range(lo, hi):
        lw = model.layers[layer]
        q = np.empty((n, H * hd))
        k = np.empty((n, KH * hd))
        v = np.empty((n, KH * hd))
        for i in range(n):
            if cfg.arch == "ref":
                h = rmsnorm_ref(x[i])
            else:
                h = rmsnorm_gain(x[i], lw["attn_norm"], cfg.norm_eps)
            q[i], k[i], v[i] = h @ lw["wq"], h @ lw["wk"], h @ lw["wv"]
            if cfg.arch == "llama":
                p = tokens[i][1]
                q[i] = rope_rotate_half(q[i], p, H, hd, cfg.rope_theta)
                k[i] = rope_rotate_half(k[i], p, KH, hd, cfg.rope_theta)
        for i, (_, p, s, _) in enumerate(tokens):
            cache.insert(layer, p, s, k[i], v[i])
        for i in range(n):
            ents = plans[i]
            keys = [cache.key(layer, j) if src == 0 else k[j] for src, j in ents]
            vals = [cache.value(layer, j) if src == 0 else v[j] for src, j in ents]
            K = np.array(keys + [k[i]]).reshape(len(ents) + 1, KH * hd)
            V = np.array(vals + [v[i]]).reshape(len(ents) + 1, KH * hd)
            attn = np.empty(H * hd)
            for h in range(H):
                kh = h // grp
                sc = K[:, kh * hd:(kh + 1) * hd] @ q[i, h * hd:(h + 1) * hd] * scale
                sc = sc - sc.max()
                w = np.exp(sc)
                w = w / w.sum()
                attn[h * hd:(h + 1) * hd] = w @ V[:, kh * hd:(kh + 1) * hd]
            x[i] = x[i] + attn @ lw["wo"]
            if cfg.arch == "ref":
                h2 = rmsnorm_ref(x[i])
                x[i] = x[i] + gelu_tanh(h2 @ lw["w1"]) @ lw["w2"]
            else:
                h2 = rmsnorm_gain(x[i], lw["mlp_norm"], cfg.norm_eps)
                x[i] = x[i] + (silu(h2 @ lw["wg"]) * (h2 @ lw["wu"])) @ lw["wd"]
        if not np.all(np.isfinite(x)):
            raise OracleModelError(f"non-finite activations after layer {layer}")
    return x


def logits(model: OracleModel, x: np.ndarray, tokens: Sequence) -> np.ndarray:
    """Rows for flagged tokens in batch order (``model.py:424-435``)."""
    idx = [i for i, t in enumerate(tokens) if t[3]]
    if not idx:
        raise OracleModelError("no tokens flagged for logits")
    rows = []
    for i in idx:
        if model.cfg.arch == "ref":
            h = rmsnorm_ref(x[i])
        else:
            h = rmsnorm_gain(x[i], model.final_norm, model.cfg.norm_eps)
        rows.append(h @ model.w_out)
    return np.array(rows)


def greedy_sample(vec) -> int:
    """Lowest-id argmax; NaN rejected (``model.py:438-443``)."""
    v = np.asarray(vec)
    if np.isnan(v).any():
        raise OracleModelError("NaN in logits")
    return int(np.argmax(v))


def max_softmax(vec) -> float:
    """``model.py:446-450``."""
    v = np.asarray(vec, dtype=np.float64)
    e = np.exp(v - v.max())
    return float(e.max() / e.sum())


def second_best(vec) -> int:
    """Runner-up id, lowest id on ties (``model.py:453-457``)."""
    v = np.array(vec, dtype=np.float64)
    v[greedy_sample(v)] = -np.inf
    return int(np.argmax(v))


def sample_prompt(seed: int, length: int, vocab_size: int) -> list:
    """``model.py:530-533``."""
    g = np.random.Generator(np.random.PCG64(seed))
    return [int(t) for t in g.integers(0, vocab_size, size=length)]


class OracleDecoder:
    """Single-context greedy decoder (``model.py:460-522``)."""

    def __init__(self, model: OracleModel, seq_id: int = 0):
        self.model = model
        self.seq = seq_id
        c = model.cfg
        self.cache = OracleCache(c.kv_dim, range(c.n_layers), c.max_context,
                                 max(1, seq_id + 1))
        self.tokens: list = []
        self.tip: Optional[np.ndarray] = None

    def feed(self, toks) -> np.ndarray:
        toks = list(toks)
        if not toks:
            if self.tip is None:
                raise OracleModelError("no tokens fed yet")
            return self.tip
        base = len(self.tokens)
        batch = [(t, base + i, frozenset([self.seq]), i == len(toks) - 1)
                 for i, t in enumerate(toks)]
        x = eval_layers(self.model, 0, self.model.cfg.n_layers, None, batch,
                        self.cache)
        self.tokens.extend(toks)
        self.tip = logits(self.model, x, batch)[0]
        return self.tip

    def truncate(self, n: int) -> None:
        if n < len(self.tokens):
            self.cache.remove(self.seq, n)
            del self.tokens[n:]
            self.tip = None

    def greedy_decode(self, prompt, n_tokens: int) -> list:
        tip = self.feed(prompt)
        out = []
        for _ in range(n_tokens):
            t = greedy_sample(tip)
            out.append(t)
            tip = self.feed([t])
        return out
