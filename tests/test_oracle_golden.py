"""Pin the CPU oracle against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``).  CPU only."""

import numpy as np
import pytest

from oracle import kvcache as OK
from oracle import model as OM
from oracle import verify as OV


def _cfg(d):
    return OM.OracleConfig(vocab_size=d["vocab_size"], embed_dim=d["embed_dim"],
                           n_layers=d["n_layers"], n_heads=d["n_heads"],
                           max_context=d["max_context"], seed=d["seed"])


def _chain(toks, start=0, seq=0, flag_all=True):
    return [(t, start + i, frozenset([seq]), flag_all or i == len(toks) - 1)
            for i, t in enumerate(toks)]


def test_weight_checksums_and_prompts(golden):
    seen = set()
    for s in golden["streams"]:
        key = tuple(sorted(s["config"].items()))
        if key not in seen:
            seen.add(key)
            assert OM.build_ref_model(_cfg(s["config"])).checksum() == s["checksum"]
        c = s["config"]
        assert OM.sample_prompt(s["prompt_seed"], len(s["prompt"]),
                                c["vocab_size"]) == s["prompt"]


@pytest.mark.parametrize("idx", [3, 5, 7])
def test_streams_small(golden, idx):
    s = golden["streams"][idx]
    m = OM.build_ref_model(_cfg(s["config"]))
    got = OM.OracleDecoder(m).greedy_decode(s["prompt"], len(s["tokens"]))
    assert got == s["tokens"]


@pytest.mark.slow
def test_stream_cfg1_full(golden):
    s = golden["streams"][0]
    m = OM.build_ref_model(_cfg(s["config"]))
    got = OM.OracleDecoder(m).greedy_decode(s["prompt"], 64)
    assert got == s["tokens"][:64]


def test_logits_rows_bitwise(golden_arrays):
    a = golden_arrays
    cfg = OM.OracleConfig(64, 32, 6, 4, 256, 7)
    m = OM.build_ref_model(cfg)
    dec = OM.OracleDecoder(m)
    rows = [dec.feed([int(t) for t in a["decode_prompt"]])]
    for _ in range(8):
        rows.append(dec.feed([OM.greedy_sample(rows[-1])]))
    # the restatement keeps the reference's per-token op order: bit-exact
    assert np.array_equal(np.stack(rows), a["decode_rows"])

    cache = OK.OracleCache(32, range(6), 256, 8)
    b = _chain([int(t) for t in a["chain_tokens"]])
    x = OM.eval_layers(m, 0, 6, None, b, cache)
    assert np.array_equal(x, a["chain_acts"])
    assert np.array_equal(OM.logits(m, x, b), a["chain_rows"])

    tree = [(3, 0, frozenset([1, 2]), True), (7, 1, frozenset([1]), True),
            (8, 1, frozenset([2]), True), (9, 2, frozenset([1]), True),
            (11, 2, frozenset([2]), True)]
    cache = OK.OracleCache(32, range(6), 256, 8)
    assert np.array_equal(
        OM.logits(m, OM.eval_layers(m, 0, 6, None, tree, cache), tree),
        a["tree_rows"])

    prompt = [int(t) for t in a["decode_prompt"]]
    cache = OK.OracleCache(32, range(6), 256, 8)
    OM.eval_layers(m, 0, 6, None, _chain(prompt, flag_all=False), cache)
    cache.copy(0, [3], len(prompt))
    spec = _chain([int(t) for t in a["spec_tokens"]], start=len(prompt), seq=3)
    assert np.array_equal(
        OM.logits(m, OM.eval_layers(m, 0, 6, None, spec, cache), spec),
        a["spec_rows"])

    cache = OK.OracleCache(32, range(2, 4), 256, 8)
    b3 = _chain([1, 2, 3])
    assert np.array_equal(OM.eval_layers(m, 2, 4, a["mid_in"], b3, cache),
                          a["mid_out"])


def test_sampling_helpers(golden_arrays):
    a = golden_arrays
    for v, am, sb, ms in zip(a["vec_in"], a["vec_argmax"], a["vec_second"],
                             a["vec_maxsoft"]):
        assert OM.greedy_sample(v) == am
        assert OM.second_best(v) == sb
        assert OM.max_softmax(v) == ms
    assert np.array_equal(OM.position_table(64, 32), a["pos_table_64x32"])


def test_cache_traces(golden):
    for tr in golden["caches"]:
        c = OK.OracleCache(2, range(1), tr["max_context"], tr["n_seq"])
        for op, snap in zip(tr["ops"], tr["snaps"]):
            if op[0] == "insert":
                c.insert(0, op[1], op[2], np.zeros(2), np.zeros(2))
            elif op[0] == "copy":
                c.copy(op[1], op[2], op[3])
            elif op[0] == "remove":
                c.remove(op[1], op[2])
            else:
                c.free_sequence(op[1])
            got = [[p, sorted(s)] for p, s in c.snapshot()]
            assert got == snap["snapshot"]
            for s, want in snap["visible"].items():
                assert c.visible_positions(int(s), tr["max_context"], 0) == want
        # gather plans: cache rows first, ties by row, batch rows after
        for pl in tr["plans"]:
            batch = [(t, p, frozenset(s), True) for t, p, s in pl["batch"]]
            plans = OM._plans(batch, c, 0)
            for mine, (sel, crows, brows) in zip(plans, pl["plans"]):
                assert [int(src == 0) for src, _ in mine] == sel
                assert [j for src, j in mine if src == 0] == crows
                assert [j for src, j in mine if src == 1] == brows


class _Rec:
    def __init__(self, tokens, min_pos, kind="speculative", seq=3, run_id=1,
                 basis=(), status="in-flight"):
        self.tokens = tuple(tokens)
        self.min_pos = min_pos
        self.max_pos = min_pos + len(tokens) - 1
        self.kind, self.seq_id, self.run_id = kind, seq, run_id
        self.basis, self.status = tuple(basis), status
        self.logit_slots = {min_pos + i: i for i in range(len(tokens))}

    def chain(self):
        yield from self.basis
        for i, t in enumerate(self.tokens):
            yield self.min_pos + i, t


def test_verify_cases(golden):
    for c in golden["verify"]:
        rows = np.zeros((len(c["preds"]), 8))
        for i, t in enumerate(c["preds"]):
            rows[i, t] = 1.0
        base = np.zeros(8)
        base[c["base"]] = 1.0
        rec = _Rec(c["tokens"], c["min_pos"])
        try:
            res = OV.verify_run(rec, rows, c["accepted"], base, c["eos"])
        except OV.OracleVerifyError:
            assert c["result"] == "VerifyError"
            continue
        want = dict(c["result"])
        want["accepted"] = tuple(want["accepted"])
        assert res == want
        cmds = OV.apply_acceptance(res["matched_end"], rec, c["live"])
        assert [[op, [a[0], list(a[1]), a[2]] if op == "copy" else list(a)]
                for op, a in cmds] == c["commands"]


def test_stale_cases(golden):
    for c in golden["stale"]:
        fifo = [_Rec(f["tokens"], f["min_pos"], kind=f["kind"], run_id=f["run_id"],
                     basis=[tuple(b) for b in f["basis"]], status=f["status"])
                for f in c["fifo"]]
        got = [[r.run_id, why] for r, why in OV.detect_stale_runs(fifo, c["accepted"])]
        assert got == c["result"]


def test_allocator_sequence(golden):
    a = OK.OracleAllocator(8)
    for op, s in golden["misc"]["allocator"]:
        if op == "alloc":
            assert a.alloc() == s
        else:
            a.free(s)


def test_oracle_caller_mask_matches_reference():
    """eval_layers(..., mask=) -- a caller-built mask that hides cache cells
    (reference model.py:369-373, golden from make_mask_golden.py)."""
    import os
    from oracle import model as OM
    from oracle.kvcache import OracleCache
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_mask.npz"))
    m = OM.build_ref_model(OM.OracleConfig(64, 32, 6, 4, 256, 7))
    prompt = [int(t) for t in g["prompt"]]
    toks = [(int(t), int(p), frozenset(s for s in range(8) if (int(mk) >> s) & 1), True)
            for t, p, mk in g["tree"]]
    plans = [[] for _ in toks]
    for i, src, j in g["order"]:
        plans[int(i)].append((int(src), int(j)))
    for use_mask, want in ((False, g["plain"]), (True, g["custom"])):
        c = OracleCache(32, range(6), 256, 8)
        OM.eval_layers(m, 0, 6, None, [(t, i, frozenset([0]), False)
                                       for i, t in enumerate(prompt)], c)
        c.copy(0, [2, 3], len(prompt))
        x = OM.eval_layers(m, 0, 6, None, toks, c, plans=plans if use_mask else None)
        assert np.array_equal(OM.logits(m, x, toks), want)
