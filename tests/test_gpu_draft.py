"""K15 persistent draft kernel: a whole draft request (feed + chained
proposals, speculation.py:142-195 with microbatch 1) in one launch must
reproduce the per-forward path (graph-replayed sp_stage_step + fused LM
head) — same proposals, same stop decisions, same K/V rows — and the
synthetic draft's explicit-token mode must leave the same cache behind."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import torch
    assert torch.cuda.is_available()
    import paper_2407_11798_b200 as sp
    return sp


SHAPES = {
    # (hd 64, GQA, 3 layers) and (hd 128, MHA) — small, fast to build
    "gqa64": dict(arch="llama", vocab_size=1000, embed_dim=512, n_layers=3, n_heads=8,
                  n_kv_heads=2, ffn_dim=1024, max_context=512, seed=3),
    "mha128": dict(arch="llama", vocab_size=777, embed_dim=256, n_layers=2, n_heads=2,
                   ffn_dim=768, max_context=512, seed=4),
    # the 160M draft's widths (long down rows: 4-row ring chunks, parity ABA
    # guard), two layers
    "wide": dict(arch="llama", vocab_size=2000, embed_dim=768, n_layers=2, n_heads=12,
                 ffn_dim=3072, max_context=512, seed=5),
}


def _servers(sp, shape):
    import torch
    from paper_2407_11798_b200.drafting import ModelDraftServer
    cfg = sp.ModelConfig(**SHAPES[shape])
    m = sp.build_model(cfg, torch.device("cuda", 0), tiled=False)
    a = ModelDraftServer(m, capacity=2048)
    b = ModelDraftServer(m, capacity=2048)
    assert a.fused_ok
    a.fused = True
    b.fused = False
    return a, b


def _drive(srv, prompt, script):
    srv.request(0, prompt, 0, 0.0)
    srv.reply()
    out = []
    for trunc, feed, budget, cutoff in script:
        t = len(srv) if trunc is None else min(trunc, len(srv))
        srv.request(t, feed, budget, cutoff)
        out.append(srv.reply())
    return out


SCRIPT = [(None, [5], 4, 0.0), (None, [17, 3], 4, 0.0), (-1, [9], 3, 0.0),
          (None, [], 4, 0.0), (None, [1, 2, 3, 4], 2, 0.0), (None, [8], 4, 0.5),
          (None, [8], 1, 0.0), (None, [11, 12, 13, 14, 15, 16], 4, 0.0),
          (None, [2], 0, 0.0), (None, [7], 4, 0.02)]


@pytest.mark.parametrize("shape", list(SHAPES))
def test_fused_chain_matches_per_forward(sp, shape):
    fused, ref = _servers(sp, shape)
    rng = np.random.default_rng(1)
    prompt = rng.integers(0, SHAPES[shape]["vocab_size"], 37).tolist()
    script = []
    for trunc, feed, budget, cut in SCRIPT:
        script.append((None if trunc is None else 30 if trunc == -1 else trunc,
                       feed, budget, cut))
    got = _drive(fused, prompt, script)
    want = _drive(ref, prompt, script)
    for (gt, gc), (wt, wc) in zip(got, want):
        assert gt == wt
        np.testing.assert_allclose(gc, wc, rtol=2e-3, atol=1e-5)
    assert fused.tokens == ref.tokens
    # the caches agree on every live row of every layer
    L = SHAPES[shape]["n_layers"]
    for layer in range(L):
        for row in range(len(fused.tokens)):
            k1, v1 = fused.stage.read_kv_sync(layer, row)
            k2, v2 = ref.stage.read_kv_sync(layer, row)
            np.testing.assert_allclose(k1, k2, rtol=3e-2, atol=3e-2)
            np.testing.assert_allclose(v1, v2, rtol=3e-2, atol=3e-2)


def test_fused_gate_closes_like_per_forward(sp):
    fused, ref = _servers(sp, "gqa64")
    prompt = list(range(10, 40))
    script = [(None, [4], 4, c) for c in (0.0, 1.0, 0.001, 0.9, 0.0)]
    got = _drive(fused, prompt, script)
    want = _drive(ref, prompt, script)
    assert [g[0] for g in got] == [w[0] for w in want]
    # cutoff 1.0 stops the chain before any proposal
    assert got[1][0] == ()


def test_fused_reproducible(sp):
    a, _ = _servers(sp, "gqa64")
    b, _ = _servers(sp, "gqa64")
    prompt = list(range(50, 70))
    assert _drive(a, prompt, SCRIPT[:5]) == _drive(b, prompt, SCRIPT[:5])


def test_table_draft_fused_cache(sp):
    """The synthetic draft pays its forwards through the fused kernel with
    explicit tokens; its cache must equal the per-forward path's."""
    import torch
    from paper_2407_11798_b200.drafting import TableDraftServer
    cfg = sp.ModelConfig(**SHAPES["gqa64"])
    m = sp.build_model(cfg, torch.device("cuda", 0), tiled=False)
    truth = list(range(100, 400))
    runner = list(range(400, 700))
    a = TableDraftServer(m, truth, runner, 0.7, 5, capacity=2048)
    b = TableDraftServer(m, truth, runner, 0.7, 5, capacity=2048)
    assert a.fused_ok
    a.fused = True
    b.fused = False
    for s in (a, b):
        s.request(0, truth[:20], 0, 0.0)
        s.reply()
        for i in range(12):
            t = len(s) - (i % 3)
            s.request(t, [truth[t]] if t < len(truth) else [1], 4, 0.0)
            s.reply()
    assert a.tokens == b.tokens
    # the fused path leaves at most the last proposal unforwarded (the next
    # request forwards it together with its own feed)
    assert len(a.tokens) - 1 <= a.cached <= len(a.tokens) and b.cached == len(b.tokens)
    for layer in range(cfg.n_layers):
        for row in range(a.cached):
            k1, v1 = a.stage.read_kv_sync(layer, row)
            k2, v2 = b.stage.read_kv_sync(layer, row)
            np.testing.assert_allclose(k1, k2, rtol=3e-2, atol=3e-2)
            np.testing.assert_allclose(v1, v2, rtol=3e-2, atol=3e-2)


def test_decode_chain_rejects_bad_use(sp):
    import torch
    from paper_2407_11798_b200 import errors
    cfg = sp.ModelConfig(**SHAPES["gqa64"])
    m = sp.build_model(cfg, torch.device("cuda", 0), tiled=False)
    from paper_2407_11798_b200.runtime import Stage
    st = Stage(m, 0, cfg.n_layers, capacity=256, max_tokens=32, n_seq_ids=1)
    out = torch.zeros((66, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(errors.ProtocolError):      # rows must equal positions
        st.decode_chain([1], 5, 2, 0.0, out.data_ptr(), out[65].data_ptr())
    with pytest.raises(errors.ModelError):         # token outside the vocab
        st.decode_chain([cfg.vocab_size], 0, 0, 0.0, out.data_ptr(), out[65].data_ptr())
    st.decode_chain([1, 2], 0, 3, 0.0, out.data_ptr(), out[65].data_ptr())
    st.synchronize()
    assert st.n_cells() == 5
    st.truncate(2)
    assert st.n_cells() == 2
