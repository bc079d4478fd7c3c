"""CPU-only tests: the C ABI library loads and exports every declared symbol,
and the host logic (allocator, layer split, verification, speculation state,
weight draws) matches the reference's golden vectors."""

import ast
import os
import re

import numpy as np
import pytest

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200 import _lib
from paper_2407_11798_b200.model import _ref_host_weights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "specpipe_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.exported_symbols())
    assert lib.sp_version().startswith(b"specpipe_b200")


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2407_11798_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom) and node.module:
                    assert not node.module.startswith("oracle"), f


def test_ref_weight_draws_match_reference_checksum(golden):
    import hashlib
    s = golden["streams"][0]
    c = s["config"]
    cfg = sp.ModelConfig(c["vocab_size"], c["embed_dim"], c["n_layers"], c["n_heads"],
                         c["max_context"], c["seed"])
    host = _ref_host_weights(cfg)
    h = hashlib.sha256()
    h.update(host["embedding"].tobytes())
    h.update(host["pos_table"].tobytes())
    for lw in host["layers"]:
        for k in ("wq", "wk", "wv", "wo", "w1", "w2"):
            h.update(lw[k].tobytes())
    h.update(host["w_out"].tobytes())
    assert h.hexdigest() == s["checksum"]


def test_sample_prompt(golden):
    for s in golden["streams"]:
        assert sp.sample_prompt(s["prompt_seed"], len(s["prompt"]),
                                s["config"]["vocab_size"]) == s["prompt"]


def test_plan_layer_split(golden):
    for c in golden["misc"]["splits"]:
        got = sp.plan_layer_split(c["n_layers"], c["n_nodes"], c["weights"])
        assert [list(r) for r in got] == c["ranges"]
    with pytest.raises(sp.EngineError):
        sp.plan_layer_split(3, 4)
    with pytest.raises(sp.EngineError):
        sp.plan_layer_split(12, 4, [1, 1])
    with pytest.raises(sp.EngineError):
        sp.plan_layer_split(12, 2, [1, 0])


def test_allocator(golden):
    a = sp.SequenceAllocator(8)
    for op, s in golden["misc"]["allocator"]:
        if op == "alloc":
            assert a.alloc() == s
        else:
            a.free(s)
    b = sp.SequenceAllocator(8)
    for _ in range(7):
        b.alloc()
    with pytest.raises(sp.AllocationExhausted):
        b.alloc()
    with pytest.raises(sp.CacheError):
        b.free(0)
    with pytest.raises(sp.CacheError):
        sp.SequenceAllocator(1)


class _Rec:
    def __init__(self, tokens, min_pos, kind="speculative", seq=3, run_id=1,
                 basis=(), status="in-flight"):
        self.tokens, self.min_pos = tuple(tokens), min_pos
        self.max_pos = min_pos + len(tokens) - 1
        self.kind, self.seq_id, self.run_id = kind, seq, run_id
        self.basis, self.status = tuple(basis), status
        self.logit_slots = {min_pos + i: i for i in range(len(tokens))}

    def chain(self):
        yield from self.basis
        for i, t in enumerate(self.tokens):
            yield self.min_pos + i, t


@pytest.mark.parametrize("as_rows", [False, True])
def test_verify_matches_reference(golden, as_rows):
    """The same walk over float rows and over fused-head RowResults."""
    for c in golden["verify"]:
        if as_rows:
            rows = [sp.RowResult(t, -1, 1.0) for t in c["preds"]]
            base = sp.RowResult(c["base"], -1, 1.0)
        else:
            rows = np.zeros((len(c["preds"]), 8))
            for i, t in enumerate(c["preds"]):
                rows[i, t] = 1.0
            base = np.zeros(8)
            base[c["base"]] = 1.0
        rec = _Rec(c["tokens"], c["min_pos"])
        try:
            res = sp.verify_run(rec, rows, c["accepted"], base, c["eos"])
        except sp.VerifyError:
            assert c["result"] == "VerifyError"
            continue
        want = c["result"]
        assert list(res.accepted) == want["accepted"]
        assert (res.n_accepted, res.next_token, res.terminal, res.examined,
                res.mismatch, res.matched_end) == (
            want["n_accepted"], want["next_token"], want["terminal"],
            want["examined"], want["mismatch"], want["matched_end"])
        cmds = []
        sp.apply_acceptance(res, rec, lambda op, a: cmds.append([op, a]), c["live"])
        assert [[op, [a[0], list(a[1]), a[2]] if op == "copy" else list(a)]
                for op, a in cmds] == c["commands"]


def test_detect_stale(golden):
    for c in golden["stale"]:
        fifo = [_Rec(f["tokens"], f["min_pos"], kind=f["kind"], run_id=f["run_id"],
                     basis=[tuple(b) for b in f["basis"]], status=f["status"])
                for f in c["fifo"]]
        got = [[r.run_id, why] for r, why in sp.detect_stale_runs(fifo, c["accepted"])]
        assert got == c["result"]


def test_cutoff_controller():
    c = sp.CutoffController(base=0.4, recovery=0.05, decay=0.05)
    c.note_success()
    assert c.current == pytest.approx(0.45)
    c.on_speculation_idle()
    c.on_speculation_idle()
    assert c.current == pytest.approx(0.35)
    c.on_run_accepted()
    assert c.current == 0.4
    hi = sp.CutoffController(base=0.99, recovery=0.5)
    hi.note_success()
    assert hi.current == 1.0
    lo = sp.CutoffController(base=0.01, decay=0.5)
    lo.on_speculation_idle()
    assert lo.current == 0.0
    with pytest.raises(sp.SpeculationError):
        sp.CutoffController(base=1.5)
    with pytest.raises(sp.SpeculationError):
        sp.CutoffController(recovery=-1)


def test_token_checksum(golden):
    for e in golden["engine"]:
        assert sp.token_checksum(e["tokens"]) == e["checksum"]


def test_greedy_helpers_host():
    v = np.zeros(64)
    v[42] = 1.0
    assert sp.greedy_sample(v) == 42
    assert sp.greedy_sample(np.ones(16)) == 0
    with pytest.raises(sp.ModelError):
        sp.greedy_sample(np.array([1.0, np.nan]))
    r = sp.RowResult(7, 3, 0.25)
    assert (sp.greedy_sample(r), sp.second_best(r), sp.max_softmax(r)) == (7, 3, 0.25)


def test_config_validation():
    with pytest.raises(sp.ModelError):
        sp.ModelConfig(embed_dim=63, n_heads=2).validate()
    with pytest.raises(sp.ModelError):
        sp.ModelConfig(vocab_size=1).validate()
    with pytest.raises(sp.ModelError):
        sp.ModelConfig(arch="gpt").validate()
    c = sp.llama_config("llama2-7b")
    # per-token streamed bytes: layers + LM head (the embedding contributes M rows only)
    assert c.weight_bytes() == pytest.approx(13.48e9 - 0.262e9, rel=0.002)
    assert sp.llama_config("llama2-70b").weight_bytes() == pytest.approx(137.95e9 - 0.524e9, rel=0.002)
