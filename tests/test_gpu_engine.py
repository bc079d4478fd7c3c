"""GPU engine: every decoding mode reproduces the reference's serial greedy
stream (tests/test_engine.py + criterion 1/2 of test_acceptance.py, re-pointed
at the B200 pipeline), with the reference's invariants on cancellation,
FIFO completion and partition exhaustion."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import torch
    assert torch.cuda.is_available()
    import paper_2407_11798_b200 as sp
    return sp


BASE = dict(mode="async-speculative", nodes=4, vocab_size=64, embed_dim=32,
            target_layers=6, draft_layers=2, max_context=512, prompt_len=16,
            gen_len=20, prompt_seed=5, target_seed=7, draft_seed=11,
            cutoff=0.0, cutoff_decay=0.0)


def cfg(sp, **kw):
    return sp.ExperimentConfig(**{**BASE, **kw})


# Speculation only pays when a draft request is cheaper than a target run.
# The reference's tests get that from their simulated delays.  On the GPU a
# tiny target is host-bound (the head finds every run already finished, and
# LOGITS take priority over new draft requests, engine.py:976-989), so these
# tests use a GPU-bound target (48 llama layers at d=1024, ~1 ms per run) and
# an uncharged synthetic draft (the analogue of draft_token_delay = 0).
DEEP = dict(arch="llama", vocab_size=512, embed_dim=1024, n_heads=8, target_layers=48,
            draft_layers=1, draft_embed_dim=128, draft_charge=False)


def deep(sp, **kw):
    return cfg(sp, **{**DEEP, **kw})


def _golden_stream(golden, seed):
    for e in golden["engine"]:
        if e["mode"] == "iterative" and e["prompt_seed"] == seed:
            return e["tokens"]
    raise KeyError(seed)


@pytest.mark.parametrize("seed", [5, 21])
def test_all_modes_byte_identical(sp, golden, seed):
    want = _golden_stream(golden, seed)
    for mode, nodes in [("iterative", 1), ("pipeline-iterative", 3),
                        ("sync-speculative", 4), ("async-speculative", 4)]:
        res = sp.simulate(cfg(sp, mode=mode, nodes=nodes, prompt_seed=seed))
        assert res.tokens == want, f"{mode} diverged"
        assert res.metrics.token_checksum == sp.token_checksum(want)


@pytest.mark.parametrize("alpha", [0.0, 0.35, 0.8, 1.0])
def test_synthetic_alpha_equivalence(sp, golden, alpha):
    res = sp.simulate(cfg(sp, draft_backend="synthetic", alpha=alpha))
    assert res.tokens == _golden_stream(golden, 5)


def test_weighted_pipeline_equivalence(sp, golden):
    res = sp.simulate(cfg(sp, mode="pipeline-iterative", nodes=3, node_weights=(2, 1, 3)))
    assert res.tokens == _golden_stream(golden, 5)


def test_alpha_one_no_rejections(sp):
    m = sp.simulate(deep(sp, draft_backend="synthetic", alpha=1.0, gen_len=48)).metrics
    assert m.examined > 0
    assert m.matched == m.examined
    assert m.acceptance_rate == 1.0
    assert m.cancelled_runs == 0


def test_alpha_zero_equals_iterative(sp):
    res = sp.simulate(cfg(sp, draft_backend="synthetic", alpha=0.0, gen_len=16))
    it = sp.simulate(cfg(sp, mode="iterative", nodes=1, gen_len=16))
    assert res.tokens == it.tokens
    assert res.metrics.matched == 0


def test_cancelled_runs_provably_stale(sp):
    res = sp.simulate(deep(sp, draft_backend="synthetic", alpha=0.4, gen_len=64))
    assert res.cancel_log, "expected cancellations at alpha=0.4"
    # early cancellation (skip / mid-stage abandon) never perturbs later runs
    assert res.tokens == sp.simulate(deep(sp, mode="iterative", nodes=1, gen_len=64)).tokens
    truth = res.accepted_full
    for e in res.cancel_log:
        if e.reason == "superfluous":
            assert e.max_pos < e.accepted_len_at_cancel - 1
        else:
            assert [p for p, t in e.chain
                    if p < e.accepted_len_at_cancel and t != truth[p]], e


def test_pipeline_integrity(sp):
    res = sp.simulate(deep(sp, draft_backend="synthetic", alpha=0.5, gen_len=32))
    assert all(r.status != "in-flight" for r in res.records)
    times = [t for t, _ in res.accept_events]
    assert times == sorted(times)
    assert res.metrics.msgs_by_tag["LOGITS"] == res.metrics.runs_started
    kinds = {"run-config", "cache-copy", "cache-remove"}
    proj = [[e for e in res.node_logs[s] if e[0] in kinds] for s in (1, 2, 3)]
    assert proj[0] == proj[1] == proj[2]


def test_partition_exhaustion_stalls_not_crashes(sp, golden):
    res = sp.simulate(deep(sp, draft_backend="synthetic", alpha=1.0, partitions=2,
                           gen_len=16))
    assert res.tokens == sp.simulate(deep(sp, mode="iterative", nodes=1, gen_len=16)).tokens
    assert res.metrics.spec_runs > 0


def test_eos_halts(sp):
    probe = sp.simulate(cfg(sp, mode="iterative", nodes=1, gen_len=12))
    eos = probe.tokens[4]
    res = sp.simulate(cfg(sp, mode="iterative", nodes=1, gen_len=12, eos_token=eos))
    assert res.tokens == probe.tokens[:5]
    res = sp.simulate(cfg(sp, gen_len=12, eos_token=probe.tokens[5]))
    idx = res.tokens.index(probe.tokens[5])
    assert res.tokens == probe.tokens[:idx + 1]


def test_metric_identity(sp):
    m = sp.simulate(deep(sp, draft_backend="synthetic", alpha=0.7, gen_len=24)).metrics
    k = m.tokens_generated - 1
    assert k / (m.ttft + m.itl * (k - 1)) == pytest.approx(m.generation_speed, rel=1e-9)


def test_criterion1_cfg1_streams(sp, golden):
    """256 generated tokens on the reference's criterion-1 model, 4 modes."""
    for s in golden["streams"][:3]:
        c = s["config"]
        for mode, nodes in [("iterative", 1), ("pipeline-iterative", 4),
                            ("sync-speculative", 5), ("async-speculative", 5)]:
            res = sp.simulate(sp.ExperimentConfig(
                mode=mode, nodes=nodes, vocab_size=c["vocab_size"],
                embed_dim=c["embed_dim"], target_layers=c["n_layers"],
                n_heads=c["n_heads"], draft_layers=2, max_context=c["max_context"],
                prompt_len=128, gen_len=256, target_seed=c["seed"], draft_seed=2,
                prompt_seed=s["prompt_seed"], cutoff=0.0, cutoff_decay=0.0))
            assert res.tokens == s["tokens"], (mode, s["prompt_seed"])


def test_randomized_stress_matches_serial(sp):
    """Criterion-2 style: randomized speculation settings never change output."""
    r = np.random.Generator(np.random.PCG64(99))
    for i in range(24):
        seed = int(r.integers(0, 4))
        c = sp.ExperimentConfig(
            mode="async-speculative", nodes=int(r.integers(2, 6)), vocab_size=16,
            embed_dim=16, target_layers=4, draft_layers=1, draft_embed_dim=16,
            max_context=128, prompt_len=8, gen_len=int(r.integers(8, 33)),
            target_seed=3, prompt_seed=seed,
            draft_backend=["toy", "synthetic"][int(r.integers(0, 2))],
            alpha=float(r.choice([0.0, 0.3, 0.6, 0.9, 1.0])),
            microbatch=int(r.integers(1, 5)), partitions=int(r.integers(2, 9)),
            continuous=bool(r.integers(0, 2)), spec_ramp=bool(i % 3),
            cutoff=float(r.choice([0.0, 0.2, 0.5])),
            cutoff_recovery=float(r.choice([0.0, 0.05])),
            cutoff_decay=float(r.choice([0.0, 0.05])))
        res = sp.simulate(c)
        ref = sp.reference_decode(c.target_config(),
                                  sp.sample_prompt(seed, 8, 16), c.gen_len)
        assert res.tokens == ref, c


def test_device_draft_loop_matches_host_speculation(sp):
    """The device-side speculate_microbatch loop (gate words in HBM) proposes
    exactly what the host loop over the same GPU draft proposes."""
    from paper_2407_11798_b200.drafting import ModelDraftServer
    cfgm = sp.ModelConfig(64, 32, 2, 4, 256, 11)
    dm = sp.build_model(cfgm)
    srv = ModelDraftServer(dm)
    host = sp.ToyDraft(dm)
    prompt = sp.sample_prompt(5, 16, 64)
    srv.request(0, prompt, 0, 1.0)
    assert srv.reply() == ((), ())
    host.feed(prompt)
    for cut in (0.0, 0.05, 0.1, 0.2, 0.0):
        srv.request(len(srv), (), 4, cut)
        toks, confs = srv.reply()
        st = sp.SpeculationState(host, sp.CutoffController(base=cut, recovery=0, decay=0), 1)
        props = sp.speculate_microbatch(st, max_tokens=4)
        assert list(toks) == [t for t, _ in props]
        assert np.allclose(confs, [c for _, c in props], rtol=1e-6)


@pytest.mark.parametrize("seed", [5, 21])
def test_bounded_cell_pool_compaction(sp, seed):
    """A pool far smaller than the cells a generation appends: the pipeline
    reclaims dead cells (stable compaction) and the stream still equals the
    serial greedy decode."""
    from paper_2407_11798_b200.engine import Engine
    for mode, nodes in [("async-speculative", 4), ("sync-speculative", 3)]:
        c = cfg(sp, mode=mode, nodes=nodes, prompt_seed=seed, gen_len=96, capacity=136,
                partitions=3,
                max_run_tokens=32, draft_backend="synthetic", alpha=0.5)
        eng = Engine(c)
        res = eng.run()
        ref = sp.reference_decode(c.target_config(), sp.sample_prompt(seed, c.prompt_len,
                                                                      c.vocab_size), 96)
        assert res.tokens == ref, mode
        assert eng.pipe.compactions > 0, mode


def test_stage_compact_moves_live_rows(sp):
    """Stage-level: compaction keeps live cells in row order with their K/V."""
    import numpy as np
    from paper_2407_11798_b200.runtime import Stage
    from paper_2407_11798_b200.model import BatchToken, encode_tokens
    c = sp.ModelConfig(vocab_size=64, embed_dim=32, n_layers=2, n_heads=2, max_context=256, seed=3)
    m = sp.build_model(c)
    st = Stage(m, 0, 2, capacity=64, max_tokens=16, n_seq_ids=4)
    toks = [BatchToken(5 + i, i, frozenset([0]), i == 9) for i in range(10)]
    st.forward(encode_tokens(toks), 0, 0, 0)
    spec = [BatchToken(7, 10 + i, frozenset([1]), True) for i in range(4)]
    st.forward(encode_tokens(spec), 1, 1, 0)
    st.synchronize()
    pos0, mask0 = st.meta_sync()
    kv0 = {r: st.read_kv_sync(1, r) for r in range(14)}
    st.cache_remove(1, 0)          # the speculative run's cells die
    st.cache_remove(0, 6)          # and the tail of seq 0
    assert st.compact() == 6
    pos1, mask1 = st.meta_sync()
    assert list(pos1[:6]) == list(pos0[:6]) and all(mask1[:6] == mask0[:6])
    for r in range(6):
        k, v = st.read_kv_sync(1, r)
        assert np.array_equal(k, kv0[r][0]) and np.array_equal(v, kv0[r][1])


def test_persistent_stage_kernel_streams(sp):
    """The opt-in persistent decode stage (SP_STAGE_MK=1, one launch per
    stage-run, grid barriers between phases, stream-K GEMMs) reproduces the
    greedy stream of the default kernel chain in every mode.  The expected
    stream is computed HERE (this process never sets SP_STAGE_MK, so it runs
    the chain); the subprocess runs everything -- serial decode included --
    on the persistent kernel and must reproduce it."""
    import os
    import subprocess
    import sys
    assert os.environ.get("SP_STAGE_MK") in (None, "", "0")
    c0 = sp.ExperimentConfig(**{**DEEP, "mode": "iterative", "nodes": 1, "gen_len": 24,
                                "prompt_len": 16, "max_context": 512, "prompt_seed": 5,
                                "target_seed": 7, "draft_seed": 11})
    want = sp.reference_decode(c0.target_config(), sp.sample_prompt(5, 16, c0.vocab_size), 24)
    code = (
        "import paper_2407_11798_b200 as sp\n"
        "from paper_2407_11798_b200.engine import ExperimentConfig\n"
        f"base = {DEEP!r}\n"
        f"want = {want!r}\n"
        "for mode, nodes in [('iterative', 1), ('async-speculative', 4), ('sync-speculative', 3)]:\n"
        "    c = ExperimentConfig(**{**base, 'mode': mode, 'nodes': nodes, 'gen_len': 24,\n"
        "                            'prompt_len': 16, 'max_context': 512, 'prompt_seed': 5,\n"
        "                            'target_seed': 7, 'draft_seed': 11,\n"
        "                            'draft_backend': 'synthetic', 'alpha': 0.5})\n"
        "    res = sp.simulate(c)\n"
        "    assert res.tokens == want, (mode, res.tokens, want)\n"
        "assert sp.reference_decode(c.target_config(), sp.sample_prompt(5, 16, c.vocab_size), 24) == want\n"
        "print('ok')\n")
    env = dict(os.environ, SP_STAGE_MK="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("mode,nodes", [("sync-speculative", 4), ("async-speculative", 4),
                                        ("async-speculative", 2)])
@pytest.mark.parametrize("seed", [5, 21])
def test_tree_speculation_streams(sp, golden, mode, nodes, seed):
    """Tree speculation (tree_width 2: chain + the draft's runner-up as a
    sibling leaf per proposal, tree-masked through partition membership)
    emits the reference's serial greedy stream on the fp32 toy decoder."""
    res = sp.simulate(cfg(sp, mode=mode, nodes=nodes, prompt_seed=seed, tree_width=2,
                          draft_backend="synthetic", alpha=0.5, alpha_sibling=0.6,
                          partitions=16))
    assert res.tokens == _golden_stream(golden, seed)


def test_tree_speculation_llama_deep(sp):
    """Same on the bf16 llama path (tcgen05 GEMMs, tree-masked attention):
    equals the iterative stream of the same weights, and siblings land."""
    it = sp.simulate(deep(sp, mode="iterative", nodes=1, gen_len=48)).tokens
    for mode, nodes in (("sync-speculative", 3), ("async-speculative", 3),
                        ("async-speculative", 2)):
        res = sp.simulate(deep(sp, mode=mode, nodes=nodes, draft_backend="synthetic",
                               alpha=0.5, tree_width=2, alpha_sibling=0.6, partitions=16,
                               gen_len=48))
        assert res.tokens == it, mode


def test_report_contract_on_gpu(sp, tmp_path, golden):
    """run_experiment -> export -> load_report round trip, and the compare
    command's verdict across all four modes (reference bench.py / cli.py)."""
    from dataclasses import replace
    from paper_2407_11798_b200 import report as R
    base = cfg(sp, repetitions=2, draft_backend="synthetic", alpha=0.6)
    reps = [R.run_experiment(replace(base, mode=m, nodes=n))
            for m, n in (("iterative", 1), ("pipeline-iterative", 3),
                         ("sync-speculative", 4), ("async-speculative", 4))]
    assert reps[0].tokens[0] == _golden_stream(golden, 5)
    code, detail = R.compare_exit_code(reps)
    assert code == 0, detail
    p = tmp_path / "rep.json"
    R.export(reps[3], "json", str(p))
    back = R.load_report(str(p))
    assert back.checksum() == reps[3].checksum() and back.tokens == reps[3].tokens
    R.export(reps[3], "csv", str(tmp_path / "rep.csv"))
    assert all(R.consistency_gap(m) < 0.01 for m in reps[3].runs)
