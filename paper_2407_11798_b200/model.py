"""Model API mirror of ``specpipe/model.py`` backed by the sm_100a library.

Same names and semantics as the reference (``ModelConfig``, ``BatchToken``,
``Batch``, ``build_model``, ``eval_layers``, ``logits``, ``greedy_sample``,
``max_softmax``, ``second_best``, ``SerialDecoder``, ``reference_decode``,
``sample_prompt``), extended with the ``llama`` architecture (RMSNorm gain,
RoPE, GQA, SwiGLU, bf16) that configs 2-5 need.  Weights live on the GPU in
the streaming layout the GEMV kernels read (``[d_out, d_in]``, K
contiguous); evaluation runs through ``runtime.Stage``.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, replace
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ModelError

SPECULATIVE = "speculative"
NON_SPECULATIVE = "non-speculative"
PREFILL = "prefill"

KIND_CODE = {PREFILL: _lib.SP_KIND_PREFILL, NON_SPECULATIVE: _lib.SP_KIND_NONSPEC,
             SPECULATIVE: _lib.SP_KIND_SPEC}


@dataclass(frozen=True)
class ModelConfig:
    """Shape and seed (model.py:39-64) plus the B200 architecture fields."""

    vocab_size: int = 256
    embed_dim: int = 64
    n_layers: int = 12
    n_heads: int = 1
    max_context: int = 1024
    seed: int = 0
    arch: str = "ref"                 # "ref" (reference toy) | "llama"
    n_kv_heads: Optional[int] = None  # GQA (llama)
    ffn_dim: Optional[int] = None     # ref: 4*d; llama: SwiGLU width
    dtype: Optional[str] = None       # "fp32" | "bf16" (default: ref fp32, llama bf16)
    norm_eps: float = 1e-5            # llama; the ref arch uses 1e-8 (model.py:189)
    rope_theta: float = 10000.0

    def validate(self) -> None:
        if self.vocab_size < 2:
            raise ModelError(f"vocab_size must be >= 2, got {self.vocab_size}")
        if self.n_layers < 1:
            raise ModelError(f"n_layers must be >= 1, got {self.n_layers}")
        if self.embed_dim % self.n_heads != 0:
            raise ModelError(
                f"embed_dim {self.embed_dim} not divisible by n_heads {self.n_heads}")
        if self.max_context < 1:
            raise ModelError("max_context must be positive")
        if self.arch not in ("ref", "llama"):
            raise ModelError(f"unknown arch {self.arch!r}")
        if self.n_heads % self.kv_heads:
            raise ModelError("n_heads must be a multiple of n_kv_heads")
        if self.weight_dtype not in ("fp32", "bf16"):
            raise ModelError(f"unknown dtype {self.dtype!r}")

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

    @property
    def weight_dtype(self) -> str:
        if self.dtype is not None:
            return self.dtype
        return "fp32" if self.arch == "ref" else "bf16"

    @property
    def eps(self) -> float:
        return 1e-8 if self.arch == "ref" else self.norm_eps

    def dims(self, tiled: Optional[bool] = None, swz: bool = False) -> _lib.sp_model_dims:
        if tiled is None:
            tiled = self.arch == "llama"
        return _lib.sp_model_dims(
            _lib.SP_ARCH_REF if self.arch == "ref" else _lib.SP_ARCH_LLAMA,
            self.vocab_size, self.embed_dim, self.n_layers, self.n_heads,
            self.kv_heads, self.head_dim, self.hidden, self.max_context,
            _lib.SP_DTYPE_F32 if self.weight_dtype == "fp32" else _lib.SP_DTYPE_BF16,
            self.eps, self.rope_theta,
            _lib.SP_LAYOUT_TC_TILED if tiled else
            (_lib.SP_LAYOUT_SWZ8 if swz else _lib.SP_LAYOUT_NATURAL))

    def weight_bytes(self, layers: Optional[int] = None, head: bool = True,
                     embedding: bool = True) -> int:
        """Bytes streamed per token (weights only) — the roofline numerator."""
        wb = 4 if self.weight_dtype == "fp32" else 2
        d, f = self.embed_dim, self.hidden
        q, kv = self.n_heads * self.head_dim, self.kv_dim
        up = 2 * f if self.arch == "llama" else f
        per_layer = (q + 2 * kv) * d + d * q + up * d + d * f
        n = self.n_layers if layers is None else layers
        total = n * per_layer * wb
        if head:
            total += self.vocab_size * d * wb
        return total


# Named target/draft shapes used by BASELINE.json's configs.
LLAMA_SHAPES = {
    "llama2-7b": dict(vocab_size=32000, embed_dim=4096, n_layers=32, n_heads=32,
                      n_kv_heads=32, ffn_dim=11008),
    "llama2-13b": dict(vocab_size=32000, embed_dim=5120, n_layers=40, n_heads=40,
                       n_kv_heads=40, ffn_dim=13824),
    "llama2-70b": dict(vocab_size=32000, embed_dim=8192, n_layers=80, n_heads=64,
                       n_kv_heads=8, ffn_dim=28672),
    "tinyllama-1.1b": dict(vocab_size=32000, embed_dim=2048, n_layers=22, n_heads=32,
                           n_kv_heads=4, ffn_dim=5632),
    "llama-160m": dict(vocab_size=32000, embed_dim=768, n_layers=12, n_heads=12,
                       n_kv_heads=12, ffn_dim=3072),
}


def llama_config(shape: str, max_context: int = 1024, seed: int = 0,
                 **overrides) -> ModelConfig:
    kw = dict(LLAMA_SHAPES[shape])
    kw.update(overrides)
    return ModelConfig(arch="llama", max_context=max_context, seed=seed, **kw)


@dataclass(frozen=True)
class BatchToken:
    """One token in a batch: id, absolute position, sequence memberships."""

    token: int
    pos: int
    seqs: frozenset
    want_logits: bool = False


@dataclass(frozen=True)
class Batch:
    """Unit of work fed into a pipeline run (model.py:77-114)."""

    tokens: tuple
    kind: str = NON_SPECULATIVE
    run_id: int = -1

    def __post_init__(self):
        if not self.tokens:
            raise ModelError("empty batch")
        if self.kind == NON_SPECULATIVE and len(self.tokens) != 1:
            raise ModelError("non-speculative batches carry exactly one token")
        last = {}
        for t in self.tokens:
            for s in t.seqs:
                p = last.get(s)
                if p is not None and t.pos <= p:
                    raise ModelError(
                        f"positions not strictly increasing along sequence {s}")
                last[s] = t.pos

    @property
    def positions(self) -> tuple:
        return tuple(t.pos for t in self.tokens)

    @property
    def logit_indices(self) -> tuple:
        return tuple(i for i, t in enumerate(self.tokens) if t.want_logits)


TOKEN_DTYPE = np.dtype([("token", "<i4"), ("pos", "<i4"), ("seq_mask", "<u4"),
                        ("want_logits", "<i4")])


def seq_mask(seqs: Iterable[int]) -> int:
    m = 0
    for s in seqs:
        if not 0 <= s < 32:
            raise ModelError(f"sequence id {s} outside [0, 32)")
        m |= 1 << int(s)
    return m


def encode_tokens(tokens: Sequence) -> np.ndarray:
    """BatchTokens -> the C ABI's sp_token array."""
    arr = np.empty(len(tokens), dtype=TOKEN_DTYPE)
    for i, t in enumerate(tokens):
        arr[i] = (t.token, t.pos, seq_mask(t.seqs), 1 if t.want_logits else 0)
    return arr


def _position_table(max_context: int, dim: int) -> np.ndarray:
    """Sinusoidal additive position table of the ref arch (model.py:153-159)."""
    p = np.arange(max_context, dtype=np.float64)[:, None]
    c = np.arange(dim, dtype=np.float64)[None, :]
    ang = p / np.power(10000.0, (2.0 * np.floor(c / 2.0)) / dim)
    return np.where(c % 2 == 0, np.sin(ang), np.cos(ang)).astype(np.float64)


class DeviceModel:
    """Immutable weights resident in HBM (LayeredModel, model.py:127-145).

    ``layers`` holds only the layer range this process serves (a pipeline
    stage materialises its own slice of a 70B model); ``embedding`` exists
    on the stage holding layer 0 and ``w_out`` on the one holding the last
    layer.  ``host`` keeps the reference-order float64 arrays for the ref
    arch (checksum parity, oracle comparisons).
    """

    def __init__(self, config: ModelConfig, device, layer_range=None):
        self.config = config
        self.device = device
        lo, hi = (0, config.n_layers) if layer_range is None else layer_range
        self.layer_range = (lo, hi)
        self.embedding = None     # [V, d]
        self.pos_table = None     # [max_context, d] fp32 (ref)
        self.w_out = None         # [V, d]
        self.w_out_tc = None      # the same, tensor-core tiled (llama, V % 128 == 0)
        self.final_norm = None    # [d] fp32 (llama)
        self.layers = {}          # layer -> dict of device tensors
        self.host = None
        self.tiled = config.arch == "llama"    # tensor-core weight layout
        self.swz = False                        # row-major bf16 in the SWZ8 layout
        self._head_stage = None

    @property
    def has_head(self) -> bool:
        return self.w_out is not None

    def checksum(self) -> str:
        """sha256 in the reference's tensor order (model.py:137-145)."""
        if self.host is None:
            raise ModelError("checksum needs the host copy (ref arch only)")
        h = hashlib.sha256()
        h.update(self.host["embedding"].tobytes())
        h.update(self.host["pos_table"].tobytes())
        for lw in self.host["layers"]:
            for name in ("wq", "wk", "wv", "wo", "w1", "w2"):
                h.update(lw[name].tobytes())
        h.update(self.host["w_out"].tobytes())
        return h.hexdigest()

    def natural_weights(self) -> dict:
        """Float64 host copy in the reference's [d_in, d_out] layout (tests)."""
        import torch  # noqa: F401  (device tensors)
        cfg = self.config
        out = dict(layers=[])
        H, KH, hd = cfg.n_heads, cfg.kv_heads, cfg.head_dim
        f64 = lambda t: t.detach().float().cpu().numpy().astype(np.float64)  # noqa: E731
        out["embedding"] = f64(self.embedding) if self.embedding is not None else None
        out["pos_table"] = None if self.pos_table is None else f64(self.pos_table)
        w_out = self.w_out if (self.w_out is None or not self.swz) else swz8_weight(self.w_out)
        out["w_out"] = None if w_out is None else f64(w_out).T.copy()
        out["final_norm"] = None if self.final_norm is None else f64(self.final_norm)
        lo, hi = self.layer_range
        lay = (lambda t: untile_weight(t)) if self.tiled else (
            (lambda t: swz8_weight(t)) if self.swz else (lambda t: t))
        for l in range(lo, hi):
            L = {k: (lay(v) if k in ("qkv", "o", "up", "down") else v)
                 for k, v in self.layers[l].items()}
            qkv = f64(L["qkv"])
            q, k, v = qkv[:H * hd], qkv[H * hd:H * hd + KH * hd], qkv[H * hd + KH * hd:]
            if cfg.arch == "llama":
                q, k = unpermute_rope_rows(q, H, hd), unpermute_rope_rows(k, KH, hd)
            d = dict(wq=q.T.copy(), wk=k.T.copy(), wv=v.T.copy(), wo=f64(L["o"]).T.copy())
            up = f64(L["up"])
            if cfg.arch == "llama":
                d["wg"], d["wu"] = up[0::2].T.copy(), up[1::2].T.copy()
                d["wd"] = f64(L["down"]).T.copy()
                d["attn_norm"], d["mlp_norm"] = f64(L["attn_norm"]), f64(L["mlp_norm"])
            else:
                d["w1"], d["w2"] = up.T.copy(), f64(L["down"]).T.copy()
            out["layers"].append(d)
        return out


def _swizzle_gather(t):
    """Within each 128x64 tile, 16-byte chunk p of row r holds logical chunk
    p ^ (r % 8) (the 128B swizzle); XOR is an involution, so the same gather
    both applies and removes it.  ``t``: [Tr, Tc, 128, 8, 8]."""
    import torch
    r = torch.arange(128, device=t.device).view(128, 1)
    j = torch.arange(8, device=t.device).view(1, 8)
    idx = (j ^ (r % 8)).view(1, 1, 128, 8, 1).expand(t.shape)
    return torch.gather(t, 3, idx)


def tile_weight(w):
    """Row-major [N, K] bf16 -> the tensor-core layout: [N/128][K/64] tiles
    of 128 x 64, each the 128B-swizzled K-major image a UMMA descriptor
    reads, so one tile is one contiguous 16 KB bulk copy and a CTA's K range
    is one sequential run of HBM (tcgemm.cu)."""
    N, K = w.shape
    if N % 128 or K % 64:
        raise ModelError(f"tensor-core weights need N % 128 == 0 and K % 64 == 0, got {N}x{K}")
    t = w.reshape(N // 128, 128, K // 64, 8, 8).permute(0, 2, 1, 3, 4)
    return _swizzle_gather(t).contiguous().reshape(N, K)


def swz8_weight(w):
    """SWZ8 layout (include/specpipe_b200.h): unit u (8 bf16) of row r goes to
    u ^ (r & 7).  An involution: applying it twice restores the rows."""
    import torch
    R, K = w.shape
    assert K % 64 == 0, "SWZ8 needs K % 64 == 0"
    w3 = w.reshape(R, K // 8, 8)
    out = torch.empty_like(w3)
    units = torch.arange(K // 8, device=w.device)
    for j in range(8):
        out[j::8] = w3[j::8][:, units ^ j]
    return out.reshape(R, K).contiguous()


def untile_weight(w):
    N, K = w.shape
    t = _swizzle_gather(w.reshape(N // 128, K // 64, 128, 8, 8))
    return t.permute(0, 2, 1, 3, 4).contiguous().reshape(N, K)


def permute_rope_rows(w: np.ndarray, n_heads: int, hd: int):
    """Natural head rows [dims 0..hd) -> pair-interleaved (j, j+hd/2)."""
    idx = rope_row_order(n_heads, hd)
    return w[idx]


def unpermute_rope_rows(w: np.ndarray, n_heads: int, hd: int):
    idx = rope_row_order(n_heads, hd)
    out = np.empty_like(w)
    out[idx] = w
    return out


def rope_row_order(n_heads: int, hd: int) -> np.ndarray:
    half = hd // 2
    per = np.empty(hd, dtype=np.int64)
    per[0::2] = np.arange(half)
    per[1::2] = np.arange(half) + half
    return np.concatenate([h * hd + per for h in range(n_heads)])


def _ref_host_weights(config: ModelConfig) -> dict:
    """PCG64 draws in the reference's documented order (model.py:162-185)."""
    rng = np.random.Generator(np.random.PCG64(config.seed))
    d, hid = config.embed_dim, 4 * config.embed_dim
    resid = 1.0 / math.sqrt(2.0 * config.n_layers)
    host = dict(embedding=rng.standard_normal((config.vocab_size, d)),
                pos_table=_position_table(config.max_context, d), layers=[])
    for _ in range(config.n_layers):
        wq = rng.standard_normal((d, d)) / math.sqrt(d)
        wk = rng.standard_normal((d, d)) / math.sqrt(d)
        wv = rng.standard_normal((d, d)) / math.sqrt(d)
        wo = rng.standard_normal((d, d)) / math.sqrt(d) * resid
        w1 = rng.standard_normal((d, hid)) / math.sqrt(d)
        w2 = rng.standard_normal((hid, d)) / math.sqrt(hid) * resid
        host["layers"].append(dict(wq=wq, wk=wk, wv=wv, wo=wo, w1=w1, w2=w2))
    host["w_out"] = rng.standard_normal((d, config.vocab_size)) / math.sqrt(d)
    for a in (host["embedding"], host["pos_table"], host["w_out"]):
        a.flags.writeable = False
    return host


def build_model(config: ModelConfig, device=None, layer_range=None,
                embedding: Optional[bool] = None,
                head: Optional[bool] = None, tiled: Optional[bool] = None) -> DeviceModel:
    """Seeded weights on the GPU (model.py:162-185).

    ref arch: the exact PCG64 float64 draws of the reference, stored fp32
    (or bf16) on the device.  llama arch: N(0,1)/sqrt(fan_in) with the
    residual-branch factor 1/sqrt(2L) (mirroring model.py:171-184), drawn on
    the device by a torch generator seeded per tensor, so every pipeline
    rank can materialise just its own layers.  ``tiled`` (llama default
    True): store the layer weights in the tcgen05 tile layout; False keeps
    them row-major for the CUDA-core GEMV path (small, latency-bound drafts).
    """
    import torch

    config.validate()
    device = torch.device("cuda" if device is None else device)
    lo, hi = (0, config.n_layers) if layer_range is None else layer_range
    if not 0 <= lo < hi <= config.n_layers:
        raise ModelError(f"layer range [{lo},{hi}) outside [0,{config.n_layers})")
    want_emb = (lo == 0) if embedding is None else embedding
    want_head = (hi == config.n_layers) if head is None else head
    m = DeviceModel(config, device, (lo, hi))
    if tiled is not None:
        if tiled and config.arch != "llama":
            raise ModelError("tensor-core tiling needs the llama arch")
        m.tiled = bool(tiled)
    tdt = torch.float32 if config.weight_dtype == "fp32" else torch.bfloat16

    def dev(a):
        # order="C": the kernels stream [d_out, d_in] rows; a transposed
        # (F-ordered) host array must be physically re-laid out
        return torch.from_numpy(np.array(a, order="C", copy=True)).to(
            device=device, dtype=tdt).contiguous()

    if config.arch == "ref":
        host = _ref_host_weights(config)
        m.host = host
        if want_emb:
            m.embedding = dev(host["embedding"])
            m.pos_table = torch.from_numpy(np.array(host["pos_table"], order="C")).to(
                device, torch.float32).contiguous()
        for l in range(lo, hi):
            lw = host["layers"][l]
            m.layers[l] = dict(
                qkv=dev(np.concatenate([lw["wq"].T, lw["wk"].T, lw["wv"].T], 0)),
                o=dev(lw["wo"].T), up=dev(lw["w1"].T), down=dev(lw["w2"].T),
                attn_norm=None, mlp_norm=None)
        if want_head:
            m.w_out = dev(host["w_out"].T)
        return m

    # llama arch: deterministic per-tensor device generation
    d, f = config.embed_dim, config.hidden
    H, KH, hd = config.n_heads, config.kv_heads, config.head_dim
    resid = 1.0 / math.sqrt(2.0 * config.n_layers)
    gen = torch.Generator(device=device)

    def draw(idx, shape, scale):
        gen.manual_seed(config.seed * 1_000_003 + idx)
        t = torch.empty(shape, device=device, dtype=torch.float32)
        t.normal_(0.0, 1.0, generator=gen)
        return (t * scale).to(tdt)

    perm_q = torch.from_numpy(rope_row_order(H, hd)).to(device)
    perm_k = torch.from_numpy(rope_row_order(KH, hd)).to(device)
    if want_emb:
        m.embedding = draw(0, (config.vocab_size, d), 1.0)
    ones = torch.ones(d, device=device, dtype=torch.float32)
    for l in range(lo, hi):
        b = 16 + 8 * l
        wq = draw(b + 0, (H * hd, d), 1 / math.sqrt(d))[perm_q]
        wk = draw(b + 1, (KH * hd, d), 1 / math.sqrt(d))[perm_k]
        wv = draw(b + 2, (KH * hd, d), 1 / math.sqrt(d))
        wo = draw(b + 3, (d, H * hd), resid / math.sqrt(H * hd))
        wg = draw(b + 4, (f, d), 1 / math.sqrt(d))
        wu = draw(b + 5, (f, d), 1 / math.sqrt(d))
        wd = draw(b + 6, (d, f), resid / math.sqrt(f))
        up = torch.empty((2 * f, d), device=device, dtype=tdt)
        up[0::2] = wg
        up[1::2] = wu
        del wg, wu
        if not m.tiled and config.weight_dtype == "bf16" and d % 64 == 0 and f % 64 == 0 \
                and (H * hd) % 64 == 0:
            m.swz = True     # row-major for the CUDA-core / persistent draft kernels
        lay = tile_weight if m.tiled else (swz8_weight if m.swz else (lambda t: t.contiguous()))
        m.layers[l] = dict(qkv=lay(torch.cat([wq, wk, wv], 0)), o=lay(wo),
                           up=lay(up), down=lay(wd), attn_norm=ones.clone(),
                           mlp_norm=ones.clone())
        del wq, wk, wv, wo, up, wd
    if want_head:
        m.w_out = draw(1, (config.vocab_size, d), 1 / math.sqrt(d))
        if m.swz:
            m.w_out = swz8_weight(m.w_out)
        elif m.tiled and config.vocab_size % 128 == 0 and d % 64 == 0:
            # the tensor-core head's copy (stage steps); the row-major one
            # serves the CUDA-core head entry points and the host views
            m.w_out_tc = tile_weight(m.w_out)
        m.final_norm = ones.clone()
    return m


# ---------------------------------------------------------------------------
# host-side sampling helpers (model.py:438-457) — also accept device results
# ---------------------------------------------------------------------------

class RowResult:
    """One fused LM-head record (argmax/second/conf) standing in for a row."""

    __slots__ = ("argmax", "second", "conf", "max_logit")

    def __init__(self, argmax, second, conf, max_logit=0.0):
        self.argmax, self.second = int(argmax), int(second)
        self.conf, self.max_logit = float(conf), float(max_logit)

    def __repr__(self):
        return f"RowResult(argmax={self.argmax}, second={self.second}, conf={self.conf:.4g})"


def greedy_sample(vec) -> int:
    """Argmax with ties broken by lowest token id (model.py:438-443)."""
    if isinstance(vec, RowResult):
        return vec.argmax
    v = np.asarray(vec)
    if np.isnan(v).any():
        raise ModelError("NaN in logits")
    return int(np.argmax(v))


def max_softmax(vec) -> float:
    """Highest softmax probability (model.py:446-450)."""
    if isinstance(vec, RowResult):
        return vec.conf
    v = np.asarray(vec, dtype=np.float64)
    e = np.exp(v - v.max())
    return float(e.max() / e.sum())


def second_best(vec) -> int:
    """Runner-up token id, lowest id on ties (model.py:453-457)."""
    if isinstance(vec, RowResult):
        return vec.second
    v = np.array(vec, dtype=np.float64)
    v[greedy_sample(v)] = -np.inf
    return int(np.argmax(v))


def sample_prompt(seed: int, length: int, vocab_size: int) -> list:
    """Seeded random prompt tokens (model.py:530-533)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return [int(t) for t in rng.integers(0, vocab_size, size=length)]


# ---------------------------------------------------------------------------
# evaluation entry points (the reference's function signatures)
# ---------------------------------------------------------------------------

def _validate_batch(model: DeviceModel, batch: Batch, lo: int) -> None:
    cfg = model.config
    for t in batch.tokens:
        if lo == 0 and not 0 <= t.token < cfg.vocab_size:
            raise ModelError(f"token id {t.token} outside vocab")
        if lo == 0 and t.pos >= cfg.max_context:
            raise ModelError(f"position {t.pos} exceeds max_context")
        if t.pos < 0:
            raise ModelError("negative position")


@dataclass
class TreeAttentionMask:
    """Per-query visibility (model.py:197-259): which cache cells and which
    batch tokens each query attends to, in ascending position order.

    ``plans[i] = (sel, cache_rows, batch_rows)``: ``sel`` marks, entry by
    entry of query i's gather order, whether it is a cache cell (True, the
    next of ``cache_rows``, raw cell rows) or a batch token (False, the next
    of ``batch_rows``, indices into the batch); every query also sees itself
    (appended last, model.py:394-415).  ``order`` is the unmerged form
    ``[(source, index)]`` (source 0 = cache-view index, 1 = batch index) that
    ``build_tree_mask`` produces; ``cache_rows`` maps view indices to rows.
    """

    n_tokens: int
    n_cells: int
    order: Optional[list] = None
    cache_rows: Optional[np.ndarray] = None
    plans: Optional[list] = None

    def gather_plans(self) -> list:
        if self.plans is None:
            out = []
            for entries in self.order:
                sel = np.array([src == 0 for src, _ in entries], dtype=bool)
                crow = np.array([j for src, j in entries if src == 0], dtype=np.int64)
                if self.cache_rows is not None and crow.size:
                    crow = np.asarray(self.cache_rows, dtype=np.int64)[crow]
                brow = np.array([j for src, j in entries if src == 1], dtype=np.int64)
                out.append((sel, crow, brow))
            self.plans = out
        return self.plans

    def visible_counts(self) -> list:
        return [int(sel.size) for sel, _, _ in self.gather_plans()]

    def cache_matrix(self) -> np.ndarray:
        m = np.zeros((self.n_tokens, self.n_cells), dtype=bool)
        if self.order is not None:
            for i, entries in enumerate(self.order):
                for src, j in entries:
                    if src == 0:
                        m[i, j] = True
        return m

    def batch_matrix(self) -> np.ndarray:
        m = np.eye(self.n_tokens, dtype=bool)
        for i, (_, _, brow) in enumerate(self.gather_plans()):
            m[i, brow] = True
        return m


def _batch_visibility(tokens, i):
    q = tokens[i]
    return [j for j, o in enumerate(tokens)
            if j != i and o.pos < q.pos and not q.seqs.isdisjoint(o.seqs)]


def build_tree_mask(batch: Batch, cache_view: Sequence) -> TreeAttentionMask:
    """Causal, branch-exclusive mask from a ``(position, sequence_set)`` view
    of the live cells (model.py:262-284): a query sees an entry iff the
    entry's position is lower and their sequence sets intersect; entries are
    merged by position, cache before batch on ties, then by index."""
    toks = batch.tokens
    order = []
    for i, q in enumerate(toks):
        ent = [(cp, 0, j) for j, (cp, cs) in enumerate(cache_view)
               if cp < q.pos and not q.seqs.isdisjoint(cs)]
        ent += [(toks[j].pos, 1, j) for j in _batch_visibility(toks, i)]
        ent.sort()
        order.append([(src, j) for _, src, j in ent])
    return TreeAttentionMask(n_tokens=len(toks), n_cells=len(cache_view), order=order,
                             cache_rows=getattr(cache_view, "rows", None))


def build_mask_from_cache(batch: Batch, cache, layer: Optional[int] = None
                          ) -> TreeAttentionMask:
    """The same mask straight off the cache's cell table (model.py:287-323);
    one table serves every layer of a stage, so ``layer`` is accepted for
    signature compatibility only."""
    pos, mask = cache._meta()
    toks = batch.tokens
    plans = []
    for i, q in enumerate(toks):
        qm = np.uint32(seq_mask(q.seqs))
        rows = np.where(((mask & qm) != 0) & (pos < q.pos))[0]
        brow = np.array(_batch_visibility(toks, i), dtype=np.int64)
        merged = np.concatenate([pos[rows], np.array([toks[j].pos for j in brow],
                                                     dtype=np.int64)])
        o = np.argsort(merged, kind="stable")
        idx = np.concatenate([rows.astype(np.int64), brow])[o]
        sel = o < rows.size
        plans.append((sel, idx[sel], idx[~sel]))
    return TreeAttentionMask(n_tokens=len(toks), n_cells=int(len(pos)), plans=plans)


def _plan_rows(mask: TreeAttentionMask, n: int, n_old: int, ld: int):
    """TreeAttentionMask -> the device plan (rows per query in gather order,
    own row last; batch token j lives in row n_old + j)."""
    plans = mask.gather_plans()
    if len(plans) != n:
        raise ModelError(f"mask covers {len(plans)} tokens, batch has {n}")
    vis = np.zeros((n, ld), dtype=np.int32)
    ln = np.zeros(n, dtype=np.int32)
    for i, (sel, crow, brow) in enumerate(plans):
        sel = np.asarray(sel, dtype=bool)
        if sel.size + 1 > ld:
            raise ModelError("mask entry list longer than the stage's plan row")
        row = np.empty(sel.size + 1, dtype=np.int64)
        row[:-1][sel] = np.asarray(crow, dtype=np.int64)
        row[:-1][~sel] = n_old + np.asarray(brow, dtype=np.int64)
        row[-1] = n_old + i
        if (row[:-1][sel] >= n_old).any() or (row < 0).any():
            raise ModelError("mask references a cache row that does not exist")
        vis[i, :row.size] = row
        ln[i] = row.size
    return vis, ln


def eval_layers(model: DeviceModel, layer_range: tuple, input_acts, batch: Batch,
                cache, mask: Optional[TreeAttentionMask] = None) -> np.ndarray:
    """Evaluate decoder layers ``[lo, hi)`` for a batch (model.py:326-421).

    ``cache`` is a ``kvcache.KVCache`` covering (at least) the range; one
    cell per token is appended on its first evaluated range and later
    sub-ranges of the same batch continue it (split == full).  ``mask``
    (a ``TreeAttentionMask``) replaces the visibility derived from cache
    membership, as in the reference (model.py:369-373); its plan is uploaded
    to the device once and shared by every layer of the range.  Returns the
    float64 host copy of the activations, like the reference.
    """
    import torch

    lo, hi = layer_range
    cfg = model.config
    if not (0 <= lo < hi <= cfg.n_layers):
        raise ModelError(f"layer range [{lo},{hi}) outside [0,{cfg.n_layers})")
    n = len(batch.tokens)
    d = cfg.embed_dim
    _validate_batch(model, batch, lo)
    if lo > 0:
        if input_acts is None:
            raise ModelError("mid-model range requires input activations")
        if tuple(np.shape(input_acts)) != (n, d):
            raise ModelError(f"activation shape {np.shape(input_acts)} != ({n}, {d})")
    stage = cache._bind(model)
    x_in = None
    if lo > 0:
        x_in = torch.as_tensor(np.asarray(input_acts, dtype=np.float32)).to(model.device)
    plan = None
    if mask is not None and not stage.continues(batch, lo):
        plan = _plan_rows(mask, n, stage.n_cells(), stage.ld_vis())
    x = stage.eval_batch(batch, lo, hi, x_in, plan=plan)
    if not np.all(np.isfinite(x)):
        raise ModelError("non-finite activations")
    return x.astype(np.float64)


def logits(model: DeviceModel, final_acts, batch: Batch) -> np.ndarray:
    """Vocab logits for flagged tokens, in batch order (model.py:424-435)."""
    idx = batch.logit_indices
    if not idx:
        raise ModelError("no tokens flagged for logits")
    from .runtime import head_logits
    return head_logits(model, np.asarray(final_acts, dtype=np.float32), list(idx))


class SerialDecoder:
    """Single-context incremental greedy decoder (model.py:460-522) on GPU.

    ``feed`` returns the tip as a ``RowResult`` (fused argmax / runner-up /
    max-softmax) unless ``full_logits`` is set, in which case the float64
    logits row is returned like the reference.
    """

    def __init__(self, model: DeviceModel, seq_id: int = 0, n_seq_ids: int = 1,
                 capacity: Optional[int] = None, full_logits: bool = False,
                 stream=None):
        from .runtime import Stage
        self.model = model
        self.seq_id = seq_id
        self.full_logits = full_logits
        cap = capacity or max(64, model.config.max_context + 64)
        self.stage = Stage(model, 0, model.config.n_layers, capacity=cap,
                           max_tokens=min(cap, max(256, model.config.max_context)),
                           n_seq_ids=max(n_seq_ids, seq_id + 1), stream=stream)
        self.tokens: list = []
        self.tip_logits = None

    def __len__(self) -> int:
        return len(self.tokens)

    def feed(self, tokens: Iterable[int]):
        toks = list(tokens)
        if not toks:
            if self.tip_logits is None:
                raise ModelError("no tokens fed yet")
            return self.tip_logits
        base = len(self.tokens)
        cfg = self.model.config
        for i, t in enumerate(toks):
            if not 0 <= t < cfg.vocab_size:
                raise ModelError(f"token id {t} outside vocab")
            if base + i >= cfg.max_context:
                raise ModelError(f"position {base + i} exceeds max_context")
        batch = Batch(tokens=tuple(
            BatchToken(t, base + i, frozenset([self.seq_id]), i == len(toks) - 1)
            for i, t in enumerate(toks)), kind=PREFILL)
        self.tip_logits = self.stage.decode_step(batch, full_logits=self.full_logits)
        self.tokens.extend(toks)
        return self.tip_logits

    def truncate(self, length: int) -> None:
        if length < len(self.tokens):
            self.stage.cache_remove(self.seq_id, length)
            del self.tokens[length:]
            self.tip_logits = None

    def greedy_decode(self, prompt: Sequence, n_tokens: int) -> list:
        tip = self.feed(prompt)
        out = []
        for _ in range(n_tokens):
            t = greedy_sample(tip)
            out.append(t)
            tip = self.feed([t])
        return out


def reference_decode(config: ModelConfig, prompt: Sequence, n_tokens: int) -> list:
    """Fresh model + serial greedy decode (model.py:525-527), on the GPU."""
    return SerialDecoder(build_model(config)).greedy_decode(prompt, n_tokens)
