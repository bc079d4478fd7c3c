"""Long-context decode (max_context >= 4096 selects the flash-decoding
attention kernel, attention_fd.cu): logits vs the fp64 oracle after a
~1500-token context, and bitwise batch/split invariance of a 5-token
verification run against 5 single-token runs (model.py:326-457)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


@pytest.fixture(scope="module")
def sp():
    import torch
    assert torch.cuda.is_available()
    import paper_2407_11798_b200 as sp
    return sp


CFG = dict(vocab_size=512, embed_dim=256, n_layers=2, n_heads=4, n_kv_heads=2, ffn_dim=512,
           max_context=4096, seed=13, arch="llama")


def _prefill(sp, m, cache, toks, chunk=200):
    x = None
    for c0 in range(0, len(toks), chunk):
        part = toks[c0:c0 + chunk]
        b = sp.Batch(tokens=tuple(sp.BatchToken(t, c0 + i, frozenset([0]), True)
                                  for i, t in enumerate(part)), kind=sp.PREFILL)
        x = sp.eval_layers(m, (0, m.config.n_layers), None, b, cache)
    return sp.logits(m, x, b)[-1]


def test_long_context_matches_oracle(sp):
    from oracle import model as OM
    cfg = sp.ModelConfig(**CFG)
    m = sp.build_model(cfg)
    nat = m.natural_weights()
    om = OM.OracleModel(OM.OracleConfig(**{k: v for k, v in CFG.items()}), nat["embedding"],
                        None, nat["layers"], nat["w_out"], nat["final_norm"])
    prompt = sp.sample_prompt(4, 1500, cfg.vocab_size)
    cache = sp.KVCache(cfg.kv_dim, range(cfg.n_layers), cfg.max_context)
    g = _prefill(sp, m, cache, prompt)
    odec = OM.OracleDecoder(om)
    o = odec.feed(prompt)
    errs = [np.abs(g - o).max()]
    pos = len(prompt)
    for _ in range(3):
        t = int(np.argmax(o))
        b = sp.Batch(tokens=(sp.BatchToken(t, pos, frozenset([0]), True),), kind=sp.NON_SPECULATIVE)
        g = sp.logits(m, sp.eval_layers(m, (0, cfg.n_layers), None, b, cache), b)[0]
        o = odec.feed([t])
        errs.append(np.abs(g - o).max())
        pos += 1
    assert max(errs) < BF16_TOL, errs


def test_long_context_batch_equals_serial_bitwise(sp):
    cfg = sp.ModelConfig(**CFG)
    m = sp.build_model(cfg)
    prompt = sp.sample_prompt(5, 1300, cfg.vocab_size)
    run = [7, 100, 3, 42, 9]
    ca = sp.KVCache(cfg.kv_dim, range(cfg.n_layers), cfg.max_context)
    cb = sp.KVCache(cfg.kv_dim, range(cfg.n_layers), cfg.max_context)
    _prefill(sp, m, ca, prompt)
    _prefill(sp, m, cb, prompt)
    p0 = len(prompt)
    b = sp.Batch(tokens=tuple(sp.BatchToken(t, p0 + i, frozenset([0]), True)
                              for i, t in enumerate(run)), kind=sp.SPECULATIVE)
    batched = sp.logits(m, sp.eval_layers(m, (0, cfg.n_layers), None, b, ca), b)
    rows = []
    for i, t in enumerate(run):
        bi = sp.Batch(tokens=(sp.BatchToken(t, p0 + i, frozenset([0]), True),),
                      kind=sp.NON_SPECULATIVE)
        rows.append(sp.logits(m, sp.eval_layers(m, (0, cfg.n_layers), None, bi, cb), bi)[0])
    assert np.array_equal(batched, np.stack(rows))
