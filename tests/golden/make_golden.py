"""Generate golden vectors by running the REFERENCE simulator itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box); the outputs are committed next to this script:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything the oracle (``oracle/``) and the GPU product are pinned against in
``tests/`` comes from here: weight checksums, prompts, greedy token streams,
logits rows, KV-cache operation traces (including the tie order of the
visibility plan), verification results, layer splits, allocator sequences,
synthetic-draft emissions and whole-engine token streams for all four modes.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from specpipe import engine as E  # noqa: E402
from specpipe import kvcache as KC  # noqa: E402
from specpipe import model as M  # noqa: E402
from specpipe import speculation as S  # noqa: E402
from specpipe import verify as V  # noqa: E402


def cfg_dict(c: M.ModelConfig) -> dict:
    return dict(vocab_size=c.vocab_size, embed_dim=c.embed_dim,
                n_layers=c.n_layers, n_heads=c.n_heads,
                max_context=c.max_context, seed=c.seed)


STREAM_CASES = [
    # (config, prompt seeds, prompt_len, gen_len)
    (M.ModelConfig(256, 64, 12, 1, 512, 1), [1000, 1001, 1002], 128, 256),
    (M.ModelConfig(256, 64, 8, 2, 512, 1), [5, 21], 32, 96),
    (M.ModelConfig(64, 32, 6, 4, 256, 7), [5, 21], 16, 40),
    (M.ModelConfig(16, 16, 2, 1, 128, 3), [3], 8, 24),
    (M.ModelConfig(32000, 256, 4, 4, 512, 1), [1], 32, 32),
]


def streams() -> list:
    out = []
    for cfg, seeds, pl, gl in STREAM_CASES:
        model = M.build_model(cfg)
        for s in seeds:
            prompt = M.sample_prompt(s, pl, cfg.vocab_size)
            dec = M.SerialDecoder(model)
            tip = dec.feed(prompt)
            toks, gaps = [], []
            for _ in range(gl):
                srt = np.sort(tip)
                gaps.append(float(srt[-1] - srt[-2]))
                t = M.greedy_sample(tip)
                toks.append(t)
                tip = dec.feed([t])
            out.append(dict(config=cfg_dict(cfg), checksum=model.checksum(),
                            prompt_seed=s, prompt=prompt, tokens=toks,
                            min_top2_gap=min(gaps)))
        print("streams", cfg, file=sys.stderr)
    return out


def logits_rows() -> dict:
    """Logits along a decode and for batched / tree / split evaluations."""
    arrs = {}
    cfg = M.ModelConfig(64, 32, 6, 4, 256, 7)
    model = M.build_model(cfg)
    prompt = M.sample_prompt(5, 12, 64)
    dec = M.SerialDecoder(model)
    rows = [dec.feed(prompt)]
    for _ in range(8):
        rows.append(dec.feed([M.greedy_sample(rows[-1])]))
    arrs["decode_prompt"] = np.array(prompt)
    arrs["decode_rows"] = np.stack(rows)
    # chain batch, all flagged
    cache = KC.KVCache(cfg.embed_dim, range(cfg.n_layers), cfg.max_context, 8)
    toks = [5, 9, 1, 33, 60]
    batch = M.Batch(tuple(M.BatchToken(t, i, frozenset([0]), True)
                          for i, t in enumerate(toks)), kind=M.PREFILL)
    acts = M.eval_layers(model, (0, 6), None, batch, cache)
    arrs["chain_tokens"] = np.array(toks)
    arrs["chain_acts"] = acts
    arrs["chain_rows"] = M.logits(model, acts, batch)
    # tree batch (tests/test_model.py:91-123 shape)
    tree = M.Batch(tokens=(
        M.BatchToken(3, 0, frozenset([1, 2]), True),
        M.BatchToken(7, 1, frozenset([1]), True),
        M.BatchToken(8, 1, frozenset([2]), True),
        M.BatchToken(9, 2, frozenset([1]), True),
        M.BatchToken(11, 2, frozenset([2]), True)), kind=M.SPECULATIVE, run_id=1)
    cache = KC.KVCache(cfg.embed_dim, range(cfg.n_layers), cfg.max_context, 8)
    arrs["tree_rows"] = M.logits(model, M.eval_layers(model, (0, 6), None, tree,
                                                      cache), tree)
    # speculative chain on top of a copied prefix (seq 3), positions 12..15
    cache = KC.KVCache(cfg.embed_dim, range(cfg.n_layers), cfg.max_context, 8)
    pre = M.Batch(tuple(M.BatchToken(t, i, frozenset([0]), False)
                        for i, t in enumerate(prompt)), kind=M.PREFILL)
    M.eval_layers(model, (0, 6), None, pre, cache)
    cache.copy(0, [3], len(prompt))
    spec_toks = [4, 44, 17, 2]
    spec = M.Batch(tuple(M.BatchToken(t, len(prompt) + i, frozenset([3]), True)
                         for i, t in enumerate(spec_toks)),
                   kind=M.SPECULATIVE, run_id=2)
    arrs["spec_tokens"] = np.array(spec_toks)
    arrs["spec_rows"] = M.logits(model, M.eval_layers(model, (0, 6), None, spec,
                                                      cache), spec)
    # mid-model input: layers [2, 4) from a fixed activation
    cache = KC.KVCache(cfg.embed_dim, range(2, 4), cfg.max_context, 8)
    x = np.random.Generator(np.random.PCG64(9)).standard_normal((3, 32))
    b3 = M.Batch(tuple(M.BatchToken(t, i, frozenset([0]), True)
                       for i, t in enumerate([1, 2, 3])), kind=M.PREFILL)
    arrs["mid_in"] = x
    arrs["mid_out"] = M.eval_layers(model, (2, 4), x, b3, cache)
    # ref arch numerics helpers
    r = np.random.Generator(np.random.PCG64(11))
    v = r.standard_normal((6, 40))
    arrs["vec_in"] = v
    arrs["vec_argmax"] = np.array([M.greedy_sample(a) for a in v])
    arrs["vec_second"] = np.array([M.second_best(a) for a in v])
    arrs["vec_maxsoft"] = np.array([M.max_softmax(a) for a in v])
    arrs["pos_table_64x32"] = M._position_table(64, 32)
    return arrs


def cache_traces() -> list:
    """Random insert/copy/remove/free schedules; snapshot after every op."""
    traces = []
    for seed in range(6):
        r = np.random.Generator(np.random.PCG64(seed))
        n_seq, maxc = 6, 48
        cache = KC.KVCache(2, range(1), maxc, n_seq)
        ops, snaps = [], []
        for _ in range(60):
            op = int(r.integers(0, 5))
            if op <= 1:
                pos = int(r.integers(0, maxc))
                seqs = sorted({int(s) for s in r.integers(0, n_seq, size=2)})
                cache.insert(0, pos, seqs, np.zeros(2), np.zeros(2))
                ops.append(["insert", pos, seqs])
            elif op == 2:
                src = int(r.integers(0, n_seq))
                dsts = sorted({int(s) for s in r.integers(0, n_seq, size=3)})
                end = int(r.integers(0, maxc + 1))
                cache.copy(src, dsts, end)
                ops.append(["copy", src, dsts, end])
            elif op == 3:
                seq = int(r.integers(0, n_seq))
                frm = int(r.integers(0, maxc))
                cache.remove(seq, frm)
                ops.append(["remove", seq, frm])
            else:
                seq = int(r.integers(1, n_seq))
                cache.free_sequence(seq)
                ops.append(["free", seq])
            snap = [[int(p), sorted(s)] for p, s in cache.snapshot()]
            vis = {str(s): [int(p) for p in cache.visible_positions(s, maxc, 0)]
                   for s in range(n_seq)}
            snaps.append(dict(snapshot=snap, visible=vis,
                              rows=[int(x) for x in cache.snapshot().rows]))
        # gather plans for a 3-token chain and a 2-seq query against the end state
        plans = []
        for q in ([(1, 40, [int(r.integers(0, n_seq))])],
                  [(2, 30, [0, 1]), (3, 31, [1])]):
            b = M.Batch(tuple(M.BatchToken(t, p, frozenset(s), True)
                              for t, p, s in q), kind=M.SPECULATIVE, run_id=1)
            m = M.build_mask_from_cache(b, cache)
            plans.append(dict(batch=[[t, p, s] for t, p, s in q],
                              plans=[[sel.astype(int).tolist(), cr.tolist(),
                                      br.tolist()] for sel, cr, br in m.gather_plans()]))
        traces.append(dict(seed=seed, n_seq=n_seq, max_context=maxc, ops=ops,
                           snaps=snaps, plans=plans))
    return traces


def verify_cases() -> dict:
    r = np.random.Generator(np.random.PCG64(77))
    cases = []
    for _ in range(300):
        vocab = 8
        n_acc = int(r.integers(1, 8))
        accepted = [int(t) for t in r.integers(0, vocab, n_acc)]
        mn = int(r.integers(max(0, n_acc - 3), n_acc + 1))
        ln = int(r.integers(1, 5))
        toks = [int(t) for t in r.integers(0, vocab, ln)]
        # make decided positions agree most of the time
        for i in range(ln):
            if mn + i < n_acc and r.random() < 0.85:
                toks[i] = accepted[mn + i]
        preds = [int(t) for t in r.integers(0, vocab, ln)]
        rows = np.zeros((ln, vocab))
        for i, t in enumerate(preds):
            rows[i, t] = 1.0
        base = int(r.integers(0, vocab))
        base_row = np.zeros(vocab)
        base_row[base] = 1.0
        eos = int(r.integers(0, vocab)) if r.random() < 0.3 else None
        rec = E.RunRecord(run_id=1, kind="speculative", tokens=tuple(toks),
                          min_pos=mn, max_pos=mn + ln - 1, seq_id=3,
                          logit_slots={mn + i: i for i in range(ln)})
        try:
            res = V.verify_run(rec, rows, accepted, base_logits=base_row,
                               eos_token=eos)
            out = dict(accepted=list(res.accepted), n_accepted=res.n_accepted,
                       next_token=res.next_token, terminal=res.terminal,
                       examined=res.examined, mismatch=res.mismatch,
                       matched_end=res.matched_end)
        except V.VerifyError:
            out = "VerifyError"
        live = sorted({int(s) for s in r.integers(1, 8, size=3)})
        cmds = []
        if out != "VerifyError":
            V.apply_acceptance(res, rec, lambda op, a: cmds.append([op, a]), live)
        cases.append(dict(accepted=accepted, min_pos=mn, tokens=toks,
                          preds=preds, base=base, eos=eos, result=out,
                          live=live,
                          commands=[[op, list(a[0:1]) + [list(a[1])] + [a[2]]
                                     if op == "copy" else list(a)]
                                    for op, a in cmds]))
    stale = []
    for _ in range(100):
        accepted = [int(t) for t in r.integers(0, 4, int(r.integers(2, 10)))]
        fifo = []
        for k in range(int(r.integers(1, 5))):
            kind = "speculative" if r.random() < 0.7 else "non-speculative"
            mn = int(r.integers(0, len(accepted) + 2))
            ln = 1 if kind == "non-speculative" else int(r.integers(1, 4))
            toks = tuple(int(t) for t in r.integers(0, 4, ln))
            basis = tuple((p, int(r.integers(0, 4)))
                          for p in range(max(0, mn - 2), mn))
            st = "in-flight" if r.random() < 0.85 else "completed"
            fifo.append(E.RunRecord(run_id=k, kind=kind, tokens=toks, min_pos=mn,
                                    max_pos=mn + ln - 1, seq_id=k + 1,
                                    logit_slots={}, basis=basis, status=st))
        got = V.detect_stale_runs(fifo, accepted)
        stale.append(dict(accepted=accepted,
                          fifo=[dict(run_id=f.run_id, kind=f.kind,
                                     tokens=list(f.tokens), min_pos=f.min_pos,
                                     basis=[list(b) for b in f.basis],
                                     status=f.status) for f in fifo],
                          result=[[rec.run_id, why] for rec, why in got]))
    return dict(verify=cases, stale=stale)


def misc() -> dict:
    splits = []
    for n_layers, n_nodes, w in [(12, 4, None), (12, 4, [2, 1, 1, 2]),
                                 (13, 4, None), (32, 4, None), (40, 8, None),
                                 (80, 8, None), (32, 3, [1, 2, 2]),
                                 (22, 5, [0.5, 1, 1, 1, 1]), (7, 7, None)]:
        splits.append(dict(n_layers=n_layers, n_nodes=n_nodes, weights=w,
                           ranges=[list(x) for x in
                                   E.plan_layer_split(n_layers, n_nodes, w)]))
    alloc = KC.SequenceAllocator(8)
    seq_log = []
    r = np.random.Generator(np.random.PCG64(4))
    for _ in range(40):
        if alloc.available() and (not alloc.live() or r.random() < 0.6):
            seq_log.append(["alloc", alloc.alloc()])
        else:
            s = alloc.live()[int(r.integers(0, len(alloc.live())))]
            alloc.free(s)
            seq_log.append(["free", s])
    # synthetic draft emissions along the TRUE path: the draft context is
    # always the accepted prefix, so each emission is best/second-best by a
    # PCG64 draw (speculation.py:127-132)
    cfg = M.ModelConfig(64, 32, 6, 4, 256, 7)
    model = M.build_model(cfg)
    prompt = M.sample_prompt(5, 16, 64)
    truth = M.reference_decode(cfg, prompt, 24)
    synth = []
    for alpha, seed in [(0.8, 11 * 1000003 + 5), (0.35, 3), (1.0, 4), (0.0, 5)]:
        d = S.SyntheticDraft(model, alpha, seed)
        d.feed(prompt)
        emitted = []
        for i in range(24):
            t = d.emit()
            emitted.append(t)
            d.truncate(len(prompt) + i)
            d.feed([truth[i]])
        synth.append(dict(alpha=alpha, seed=seed, emitted=emitted))
    return dict(splits=splits, allocator=seq_log, synth_prompt=prompt,
                synth_truth=truth, synthetic=synth,
                synth_config=cfg_dict(cfg))


def engine_streams() -> list:
    base = dict(vocab_size=64, embed_dim=32, target_layers=6, draft_layers=2,
                max_context=512, prompt_len=16, gen_len=20, target_seed=7,
                draft_seed=11, cutoff=0.0, cutoff_decay=0.0,
                per_layer_delay=1e-4, link_latency=1e-6, draft_token_delay=5e-5)
    out = []
    for seed in (5, 21):
        for mode, nodes, extra in [("iterative", 1, {}),
                                   ("pipeline-iterative", 3, {}),
                                   ("sync-speculative", 4, {}),
                                   ("async-speculative", 4, {}),
                                   ("async-speculative", 4,
                                    dict(draft_backend="synthetic", alpha=0.6))]:
            cfg = E.ExperimentConfig(mode=mode, nodes=nodes, prompt_seed=seed,
                                     **{**base, **extra})
            res = E.simulate(cfg)
            out.append(dict(mode=mode, nodes=nodes, prompt_seed=seed,
                            extra=extra, tokens=res.tokens,
                            checksum=res.metrics.token_checksum))
    return out


def main():
    golden = dict(streams=streams(), caches=cache_traces(), **verify_cases(),
                  misc=misc(), engine=engine_streams())
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(golden, f, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "reference_logits.npz"),
                        **logits_rows())
    print("wrote golden vectors", file=sys.stderr)


if __name__ == "__main__":
    main()
