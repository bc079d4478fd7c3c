"""TEST INFRASTRUCTURE / CPU BASELINE ONLY -- never imported by the product.

Runs the UNMODIFIED reference (``specpipe``, installed into ``oracle/_ref``
by ``oracle/vendor_ref.sh``) on the host cores, for bench.py's reference arm
(``--impl reference``) and its ``cpu_baseline``:

1. cfg1 serial oracle: ``reference_decode`` tok/s (model.py:525-527);
2. cfg1 in all four modes: ``simulate(clock="wall")`` with zero injected
   delays (engine.py:1293-1356) -- generation speed, TTFT, ITL;
3. the reference's own architecture at a Llama width (2 layers + the LM
   head at V=32000, timed per token and extrapolated to the target's layer
   count, labelled "extrapolated"; the reference cannot run Llama).

The reference's two latent async-head bugs are patched at run
time, never edited: F4(a) a speculative launch whose frontier is carried by
an in-flight run copies its prefix from that run's partition (engine.py:
1070-1079 vs 1127-1143); F4(b) a draft request that would truncate without
feeding backs off one token (engine.py:1019-1045, model.py:507-512).
"""

from __future__ import annotations

import dataclasses
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "specpipe"))


def load():
    """Import the vendored reference and apply the F4 shims (idempotent)."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import specpipe
    from specpipe import engine as E
    C = E._Controller
    if getattr(C, "_f4_shimmed", False):
        return specpipe

    orig_launch_spec = C._launch_spec

    def _carrier(self):
        pos, tok = len(self.accepted) - 1, self.accepted[-1]
        for rec in self.fifo:
            if (rec.status == E.IN_FLIGHT and rec.min_pos <= pos <= rec.max_pos
                    and rec.tokens[pos - rec.min_pos] == tok):
                return rec.seq_id
        return 0

    def launch_spec(self, props):                      # F4(a)
        carrier = 0 if self.pending else _carrier(self)
        if not carrier:
            return orig_launch_spec(self, props)
        real = self._emit_copy
        self._emit_copy = lambda src, dsts, end: real(carrier if src == 0 else src, dsts, end)
        try:
            return orig_launch_spec(self, props)
        finally:
            del self._emit_copy

    orig_send = C._send_draft_request

    def send_draft_request(self):                      # F4(b)
        real = self.net.send_txn
        mirror_len = len(self.mirror)
        ctx = self.accepted + [t for _, t in self.pending]

        def send(src, dst, tag, payload, *rest):
            if (tag == E.Tag.DRAFT_REQUEST and not payload.feed
                    and 0 < payload.truncate_to < mirror_len):
                cp = payload.truncate_to
                payload = dataclasses.replace(payload, truncate_to=cp - 1,
                                              feed=tuple(ctx[cp - 1:cp]))
            return real(src, dst, tag, payload, *rest)

        self.net.send_txn = send
        try:
            return orig_send(self)
        finally:
            self.net.send_txn = real

    C._launch_spec = launch_spec
    C._send_draft_request = send_draft_request
    C._f4_shimmed = True
    return specpipe


# cfg1 (BASELINE.json configs[0]; BASELINE.md §2's setting)
CFG1 = dict(vocab_size=256, embed_dim=64, target_layers=8, draft_layers=1, n_heads=1,
            max_context=512, prompt_len=32, gen_len=128)


def cfg1_decode(sp, seed: int = 1234) -> dict:
    c = sp.ModelConfig(vocab_size=CFG1["vocab_size"], embed_dim=CFG1["embed_dim"],
                       n_layers=CFG1["target_layers"], n_heads=CFG1["n_heads"],
                       max_context=CFG1["max_context"], seed=1)
    prompt = sp.sample_prompt(seed, CFG1["prompt_len"], CFG1["vocab_size"])
    t0 = time.perf_counter()
    out = sp.reference_decode(c, prompt, CFG1["gen_len"])
    dt = time.perf_counter() - t0
    return {"tokens_per_s": round(len(out) / dt, 1), "tokens": len(out),
            "note": "reference_decode incl. model build + prefill (model.py:525-527)"}


def cfg1_modes(sp, stages: int = 4, alpha: float = 0.8) -> dict:
    """simulate(clock='wall') with zero injected delays."""
    out = {}
    for mode in ("iterative", "pipeline-iterative", "sync-speculative", "async-speculative"):
        nodes = 1 if mode == "iterative" else (stages if mode == "pipeline-iterative"
                                               else stages + 1)
        cfg = sp.ExperimentConfig(mode=mode, nodes=nodes, clock="wall", per_layer_delay=0.0,
                                  link_latency=0.0, draft_token_delay=0.0,
                                  draft_backend="synthetic", alpha=alpha, **CFG1)
        t0 = time.perf_counter()
        m = sp.simulate(cfg).metrics
        out[mode] = {"generation_speed": round(m.generation_speed, 1),
                     "ttft_ms": round(m.ttft * 1e3, 3), "itl_ms": round(m.itl * 1e3, 3),
                     "nodes": nodes, "wall_s": round(time.perf_counter() - t0, 2)}
    return out


def width_extrapolated(sp, d: int, n_heads: int, n_layers: int, vocab: int = 32000,
                       layers: int = 2, n_decode: int = 2, prompt_len: int = 8) -> dict:
    """The reference's own decoder (``ref`` arch) at a Llama width: per-token
    time of ``layers`` layers + the LM head, extrapolated to ``n_layers``."""
    import numpy as np  # noqa: F401
    from specpipe.kvcache import KVCache
    c = sp.ModelConfig(vocab_size=vocab, embed_dim=d, n_layers=layers, n_heads=n_heads,
                       max_context=prompt_len + n_decode + 8, seed=3)
    t0 = time.perf_counter()
    m = sp.build_model(c)
    build_s = time.perf_counter() - t0
    cache = KVCache(d, range(layers), c.max_context, 1)
    prompt = sp.sample_prompt(1, prompt_len, vocab)
    b = sp.Batch(tokens=tuple(sp.BatchToken(t, i, frozenset([0]), i == prompt_len - 1)
                              for i, t in enumerate(prompt)), kind="prefill", run_id=1)
    sp.eval_layers(m, (0, layers), None, b, cache)
    per, head = [], []
    for i in range(n_decode):
        bt = sp.Batch(tokens=(sp.BatchToken(int(prompt[i % prompt_len]), prompt_len + i,
                                            frozenset([0]), True),),
                      kind="non-speculative", run_id=2 + i)
        t0 = time.perf_counter()
        x = sp.eval_layers(m, (0, layers), None, bt, cache)
        per.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        sp.logits(m, x, bt)
        head.append(time.perf_counter() - t0)
    per_layer = statistics.median(per) / layers
    t_head = statistics.median(head)
    per_token = per_layer * n_layers + t_head
    return {"tokens_per_s": 1.0 / per_token, "ms_per_token": per_token * 1e3,
            "per_layer_ms": per_layer * 1e3, "head_ms": t_head * 1e3, "build_s": build_s,
            "sample": (f"reference ref-arch decoder (specpipe.eval_layers + logits, fp64) at "
                       f"d={d}, {n_heads} heads, V={vocab}: {layers} layers timed over "
                       f"{n_decode} decode tokens after a {prompt_len}-token prompt, "
                       f"extrapolated to {n_layers} layers + LM head")}
