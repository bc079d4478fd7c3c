"""Parity on the path bench.py measures (VERDICT r01 "what's weak" 1):

* the headline's own widths -- the 7B target (d=4096, 32 heads, ffn 11008) on
  the tcgen05 path and the 160M draft (d=768, 12 heads, ffn 3072) on both the
  SWZ8 GEMV path and tiled -- against the fp64 oracle (model.py:326-457);
* the persistent draft kernels the bench runs by default (cluster form at
  N<=2, grid form on a dedicated draft GPU), per chained proposal, against the
  oracle's greedy step on the same context (speculation.py:185-211 with
  microbatch 1, engine.py:663-688);
* the synthetic draft's emissions against the reference's own SyntheticDraft
  draw sequence (speculation.py:98-139, golden misc.synthetic).

Tolerances: logits max-abs 2e-2 (bf16, north star); proposal tokens exact
wherever the fp64 top-1/top-2 gap exceeds 10x that tolerance; confidence
(max softmax) within 2e-2.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


@pytest.fixture(scope="module")
def sp():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_11798_b200 as sp
    return sp


def _oracle_for(sp, m, cfg):
    from oracle import model as OM
    nat = m.natural_weights()
    oc = OM.OracleConfig(vocab_size=cfg.vocab_size, embed_dim=cfg.embed_dim,
                         n_layers=cfg.n_layers, n_heads=cfg.n_heads,
                         max_context=cfg.max_context, seed=cfg.seed, arch="llama",
                         n_kv_heads=cfg.n_kv_heads, ffn_dim=cfg.ffn_dim)
    om = OM.OracleModel(oc, nat["embedding"], None, nat["layers"], nat["w_out"],
                        nat["final_norm"])
    return OM, om


@pytest.mark.parametrize("shape,tiled,layers", [("llama2-7b", True, 1),
                                                ("llama2-7b", True, 2),
                                                ("llama-160m", False, 2),
                                                ("llama-160m", True, 2)])
def test_headline_widths_match_oracle(sp, shape, tiled, layers):
    """Prompt logits + 3 greedy decode steps of a layer slice at the real
    width, vocabulary and head layout of the benchmarked pair."""
    cfg = sp.llama_config(shape, max_context=64, seed=9, n_layers=layers)
    m = sp.build_model(cfg, tiled=tiled)
    OM, om = _oracle_for(sp, m, cfg)
    prompt = sp.sample_prompt(6, 7, cfg.vocab_size)
    dec = sp.SerialDecoder(m, full_logits=True)
    odec = OM.OracleDecoder(om)
    g, o = dec.feed(prompt), odec.feed(prompt)
    errs = [np.abs(g - o).max()]
    for _ in range(3):
        t = int(np.argmax(o))
        g, o = dec.feed([t]), odec.feed([t])
        errs.append(np.abs(g - o).max())
    assert max(errs) < BF16_TOL, errs


def _draft_vs_oracle(sp, kernel, shape_kw, n_req=8, budget=4, seed=2, fused=True):
    """Drive a ModelDraftServer with ``SP_DRAFT_KERNEL=kernel`` and check each
    chained proposal against the oracle's step on the same context.  ``fused``
    says which path the shape takes: the persistent kernels, or (widths past
    their shared-memory plan, sp_stage_decode_chain_ok == 0) one graph-replayed
    stage step per forward."""
    import torch
    from paper_2407_11798_b200.drafting import ModelDraftServer
    old = os.environ.get("SP_DRAFT_KERNEL")
    os.environ["SP_DRAFT_KERNEL"] = kernel
    try:
        cfg = sp.ModelConfig(**shape_kw)
        m = sp.build_model(cfg, torch.device("cuda", 0), tiled=False)
        srv = ModelDraftServer(m, capacity=1024)
        assert srv.fused == fused, "the path under test must be the one the product takes"
        OM, om = _oracle_for(sp, m, cfg)
        rng = np.random.default_rng(seed)
        prompt = rng.integers(0, cfg.vocab_size, 12).tolist()
        srv.request(0, prompt, 0, 1.0)
        srv.reply()
        exact = checked = 0
        for r in range(n_req):
            # feed one fresh token (as a head does after an acceptance), and
            # every few requests roll back two tokens first (rejection)
            trunc = len(srv) - (2 if r % 3 == 2 else 0)
            feed = [int(rng.integers(0, cfg.vocab_size))]
            srv.request(trunc, feed, budget, 0.0)
            toks, confs = srv.reply()
            assert len(toks) == budget
            ctx = list(srv.tokens)             # prefix + feed + proposals
            base = len(ctx) - len(toks)
            odec = OM.OracleDecoder(om)
            row = odec.feed(ctx[:base])
            for j, (t, c) in enumerate(zip(toks, confs)):
                srt = np.sort(row)
                gap = srt[-1] - srt[-2]
                checked += 1
                if gap > 10 * BF16_TOL:
                    exact += 1
                    assert t == int(np.argmax(row)), (kernel, r, j, gap)
                else:      # near-tie: the GPU may take either of the top two
                    assert t in (int(np.argmax(row)), int(OM.second_best(row))), (r, j)
                ref_c = OM.max_softmax(row)
                assert abs(c - ref_c) < BF16_TOL, (kernel, r, j, c)
                # V=32000 makes conf tiny; also bound it relatively (a logit
                # error e moves log-softmax by at most 2e)
                assert abs(np.log(c) - np.log(ref_c)) < 2.5 * BF16_TOL, (kernel, r, j, c, ref_c)
                row = odec.feed([t])
        assert exact >= checked // 4, (exact, checked)
    finally:
        if old is None:
            os.environ.pop("SP_DRAFT_KERNEL", None)
        else:
            os.environ["SP_DRAFT_KERNEL"] = old


# the 160M draft's real widths (d=768, 12 heads of 128, ffn 3072, V=32000) in
# two layers, and TinyLlama-1.1B's (d=2048, GQA 32/4 heads of 64, ffn 5632)
DRAFT_SHAPES = {
    "160m": dict(arch="llama", vocab_size=32000, embed_dim=768, n_layers=2, n_heads=12,
                 ffn_dim=3072, max_context=256, seed=7),
    "1.1b": dict(arch="llama", vocab_size=32000, embed_dim=2048, n_layers=2, n_heads=32,
                 n_kv_heads=4, ffn_dim=5632, max_context=256, seed=8),
}


@pytest.mark.parametrize("kernel", ["cluster", "grid"])
def test_persistent_draft_kernels_match_oracle(sp, kernel):
    _draft_vs_oracle(sp, kernel, DRAFT_SHAPES["160m"])


def test_per_forward_draft_1b_matches_oracle(sp):
    """TinyLlama-1.1B widths (configs[2]/[3]'s draft): ffn 5632 exceeds the
    persistent kernels' per-CTA slice plan, so the product drafts with one
    stage step per forward; same oracle check."""
    _draft_vs_oracle(sp, "cluster", DRAFT_SHAPES["1.1b"], fused=False)


def test_synthetic_emissions_match_reference(sp, golden):
    """TableDraftServer draws exactly the reference SyntheticDraft sequence:
    one PCG64 draw per emission, truth with probability alpha else the
    runner-up (golden: the reference run with the context on the true path,
    tests/golden/make_golden.py)."""
    from paper_2407_11798_b200.drafting import TableDraftServer
    from paper_2407_11798_b200.engine import truth_table
    m = golden["misc"]
    c = m["synth_config"]
    cfg = sp.ModelConfig(c["vocab_size"], c["embed_dim"], c["n_layers"], c["n_heads"],
                         c["max_context"], c["seed"])
    model = sp.build_model(cfg)
    prompt = m["synth_prompt"]
    truth, runner = truth_table(model, prompt, 26)
    assert truth[len(prompt):len(prompt) + 24] == m["synth_truth"]
    for case in m["synthetic"]:
        srv = TableDraftServer(model, truth, runner, case["alpha"], case["seed"],
                               charge=False, capacity=512)
        srv.request(0, prompt, 0, 0.0)
        srv.reply()
        emitted = []
        for i in range(24):
            # context before emission i = prompt + truth[:i] (the reference
            # truncates its own emission away and feeds the true token)
            if i == 0:
                srv.request(len(prompt), [], 1, 0.0)
            else:
                srv.request(len(prompt) + i - 1, [m["synth_truth"][i - 1]], 1, 0.0)
            toks, confs = srv.reply()
            assert confs == (case["alpha"],) * len(toks)
            emitted.extend(toks)
        assert emitted == case["emitted"], case["alpha"]
