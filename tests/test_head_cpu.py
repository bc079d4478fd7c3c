"""The head's decision logic on CPU under randomized timing.

``FakePipeline`` executes the head's transactions on the float64 oracle
(test infrastructure) with the reference worker's stage semantics
(engine.py:563-623): in-order transactions per stage, placeholder
propagation, skip of cancelled speculative runs with partition purge, the
coverage check.  Completion latency and cancel visibility are randomized —
cancels become visible monotonically in issue order, as the device-visible
cancel words do — so runs overlap, get cancelled before or after each stage,
and the F4(a)/(b) situations arise.  Every output must equal the oracle's
serial greedy stream (criterion 2 of the reference's acceptance suite)."""

from collections import deque

import numpy as np
import pytest

from oracle import model as OM
from oracle.kvcache import OracleCache
from paper_2407_11798_b200 import errors
from paper_2407_11798_b200.engine import ExperimentConfig, Head, plan_layer_split
from paper_2407_11798_b200.model import RowResult
from paper_2407_11798_b200.pipeline import RunResult


class FakePipeline:
    def __init__(self, om, ranges, partitions, rng):
        self.om, self.ranges, self.P, self.rng = om, ranges, partitions, rng
        self.n_stages = len(ranges)
        self.reset()

    def reset(self):
        c = self.om.cfg
        self.caches = [OracleCache(c.kv_dim, range(lo, hi), c.max_context, self.P)
                       for lo, hi in self.ranges]
        self.ops, self.fifo, self.done = deque(), deque(), {}
        self.clock, self.vis_from, self.last_vis = 0, {}, 0
        self.skips = 0

    def launch(self, run_id, kind, toks, flags, rows):
        self.ops.append(("run", run_id, kind, toks.copy(), list(rows)))
        self.fifo.append(run_id)

    def copy(self, src, dsts, end):
        self.ops.append(("copy", src, tuple(dsts), end))

    def remove(self, seq, frm):
        self.ops.append(("remove", seq, frm))

    def cancel_run(self, run_id):
        self.last_vis = max(self.last_vis, self.clock + int(self.rng.integers(0, 4)))
        self.vis_from[run_id] = self.last_vis

    def _cancelled(self, run_id):
        v = self.vis_from.get(run_id)
        return v is not None and self.clock >= v

    def _step(self):
        op = self.ops.popleft()
        if op[0] == "copy":
            for c in self.caches:
                c.copy(op[1], op[2], op[3])
            return
        if op[0] == "remove":
            for c in self.caches:
                c.remove(op[1], op[2])
            return
        _, run_id, kind, toks, rows = op
        batch = [(int(t["token"]), int(t["pos"]),
                  frozenset(i for i in range(32) if (int(t["seq_mask"]) >> i) & 1),
                  bool(t["want_logits"])) for t in toks]
        x, placeholder = None, False
        for (lo, hi), cache in zip(self.ranges, self.caches):
            self.clock += 1
            if placeholder:
                continue
            if kind == 2 and self._cancelled(run_id):
                for _, _, seqs, _ in batch:
                    for s in seqs:
                        if s:
                            cache.remove(s, 0)
                placeholder = True
                self.skips += 1
                continue
            counts = OM.visible_counts(batch, cache, lo)
            for (_, p, _, _), n in zip(batch, counts):
                if n != p:
                    raise errors.ProtocolError(f"run {run_id}: pos {p} sees {n} cells")
            x = OM.eval_layers(self.om, lo, hi, x, batch, cache)
        out = []
        if not placeholder:
            for r in OM.logits(self.om, x, batch):
                out.append(RowResult(OM.greedy_sample(r), OM.second_best(r), OM.max_softmax(r)))
        self.done[run_id] = RunResult(run_id, placeholder, out, 0,
                                      [1 if placeholder else 0] * self.n_stages)

    def _run_until(self, run_id):
        while run_id not in self.done:
            self._step()

    def ready(self):
        if not self.fifo:
            return False
        if self.fifo[0] not in self.done and self.rng.random() < 0.35:
            self._run_until(self.fifo[0])
        return self.fifo[0] in self.done

    def poll(self):
        return self.done.pop(self.fifo.popleft()) if self.ready() else None

    def wait(self):
        self._run_until(self.fifo[0])
        return self.done.pop(self.fifo.popleft())

    def in_flight(self):
        return len(self.fifo)


class FakeDraft:
    """SyntheticDraft semantics over the oracle's greedy table, random latency."""

    def __init__(self, truth, runner, alpha, seed, max_context, rng, alpha_sibling=0.0):
        self.truth, self.runner, self.alpha = truth, runner, alpha
        self.g = np.random.Generator(np.random.PCG64(seed))
        self.g2 = np.random.Generator(np.random.PCG64(seed + 99))
        self.alpha_sibling = alpha_sibling
        self.seconds = ()
        self.max_context, self.rng = max_context, rng
        self.tokens, self.pending = [], None
        self.forwards = 0

    def __len__(self):
        return len(self.tokens)

    def request(self, truncate_to, feed, max_tokens, cutoff):
        assert self.pending is None
        del self.tokens[truncate_to:]
        self.tokens.extend(feed)
        if max_tokens and not self.tokens:
            raise errors.SpeculationError("draft has no context yet")
        budget = max(0, min(max_tokens, self.max_context - len(self.tokens), 4))
        props, secs = [], []
        if budget and self.alpha >= cutoff:
            for _ in range(budget):
                p = len(self.tokens)
                on = self.tokens == self.truth[:p]
                best = self.truth[p] if p < len(self.truth) else 0
                second = self.runner[p] if p < len(self.runner) else 1
                tok = best if self.g.random() < self.alpha else second
                if not on:
                    tok = second
                hit = self.g2.random() < self.alpha_sibling
                secs.append(second if tok == best else best if hit else (best + 1) % 16
                            if (best + 1) % 16 != tok else (best + 2) % 16)
                self.tokens.append(tok)
                props.append(tok)
        self.pending = tuple(props)
        self.seconds = tuple(secs)

    def ready(self):
        return self.pending is not None and self.rng.random() < 0.5

    def busy(self):
        return self.pending is not None

    def reply(self):
        p, self.pending = self.pending, None
        return p, tuple(self.alpha for _ in p)


@pytest.fixture(scope="module")
def world():
    cfg = OM.OracleConfig(16, 16, 4, 1, 96, 3)
    om = OM.build_ref_model(cfg)
    streams = {}
    for s in range(3):
        prompt = OM.sample_prompt(s, 8, 16)
        dec = OM.OracleDecoder(om)
        tip = dec.feed(prompt)
        truth, runner = list(prompt), [0] * len(prompt)
        for _ in range(48):
            truth.append(OM.greedy_sample(tip))
            runner.append(OM.second_best(tip))
            tip = dec.feed([truth[-1]])
        streams[s] = (prompt, truth, runner)
    return om, streams


def test_async_head_randomized_matches_serial(world):
    om, streams = world
    r = np.random.Generator(np.random.PCG64(7))
    skipped = cancelled = folded = sib_hits = 0
    for trial in range(60):
        seed = int(r.integers(0, 3))
        prompt, truth, runner = streams[seed]
        nodes = int(r.integers(2, 5))
        cfg = ExperimentConfig(
            mode="async-speculative", nodes=nodes, vocab_size=16, embed_dim=16,
            target_layers=4, max_context=96, prompt_len=8, gen_len=int(r.integers(6, 40)),
            partitions=int(r.integers(2, 9)), microbatch=int(r.integers(1, 5)),
            continuous=bool(r.integers(0, 2)), alpha=float(r.choice([0.0, 0.4, 0.8, 1.0])),
            cutoff=float(r.choice([0.0, 0.3])), cutoff_recovery=float(r.choice([0.0, 0.05])),
            cutoff_decay=float(r.choice([0.0, 0.05])), spec_ramp=trial % 4 != 3,
            fold_frontier=[None, True, False][trial % 3],
            max_inflight=[None, 0, 1, 2, 3][trial % 5], tree_width=1 + (trial % 2))
        pipe = FakePipeline(om, plan_layer_split(4, nodes - 1), cfg.partitions, r)
        draft = FakeDraft(truth, runner, cfg.alpha, trial, 96, r,
                          alpha_sibling=0.5 if cfg.tree_width == 2 else 0.0)
        head = Head(cfg, pipe, draft, prompt, 16)
        head.run_async_speculative()
        out = head.accepted[len(prompt):]
        assert out == truth[len(prompt):len(prompt) + cfg.gen_len], (trial, cfg)
        folded += head.folded_runs
        sib_hits += head.sibling_hits
        skipped += pipe.skips
        cancelled += head.cancelled_invalid + head.cancelled_superfluous
        for e in head.cancel_log:
            if e.reason == "superfluous":
                assert e.max_pos < e.accepted_len_at_cancel - 1
            else:
                assert any(p < e.accepted_len_at_cancel and t != truth[p] for p, t in e.chain)
    assert cancelled > 0 and skipped > 0 and folded > 0 and sib_hits > 0


@pytest.mark.parametrize("mode,nodes", [("iterative", 1), ("pipeline-iterative", 3),
                                        ("sync-speculative", 3)])
def test_other_modes_match_serial(world, mode, nodes):
    om, streams = world
    r = np.random.Generator(np.random.PCG64(1))
    prompt, truth, runner = streams[1]
    cfg = ExperimentConfig(mode=mode, nodes=nodes, vocab_size=16, embed_dim=16,
                           target_layers=4, max_context=96, prompt_len=8, gen_len=30,
                           alpha=0.6, cutoff=0.0)
    pipe = FakePipeline(om, plan_layer_split(4, cfg.n_stages()), cfg.partitions, r)
    draft = FakeDraft(truth, runner, 0.6, 3, 96, r) if cfg.uses_draft() else None
    head = Head(cfg, pipe, draft, prompt, 16)
    {"iterative": head.run_iterative, "pipeline-iterative": head.run_iterative,
     "sync-speculative": head.run_sync_speculative}[mode]()
    assert head.accepted[len(prompt):] == truth[len(prompt):len(prompt) + 30]


def test_f4b_backoff_refeeds_tip(world):
    """A context that is a strict prefix of the draft's state is served by
    truncating one token further and re-feeding it."""
    om, streams = world
    prompt, truth, runner = streams[0]
    cfg = ExperimentConfig(mode="async-speculative", nodes=2, vocab_size=16, embed_dim=16,
                           target_layers=4, max_context=96, prompt_len=8, gen_len=8)
    pipe = FakePipeline(om, [(0, 4)], 8, np.random.Generator(np.random.PCG64(0)))
    head = Head(cfg, pipe, None, prompt, 16)
    head.mirror = list(prompt) + [5, 6, 7]
    assert head._backoff(len(prompt), list(prompt)) == (len(prompt) - 1, [prompt[-1]])
    assert head._backoff(len(prompt) - 2, list(prompt)) == (len(prompt) - 2, prompt[-2:])


def test_spec_ramp_caps_requests(world):
    """The reference's continuous micro-batch ramp (engine.py:1027-1030): a
    fresh chain asks the draft for one token, deeper chains up to
    ``microbatch``; spec_ramp=False always asks for ``microbatch``."""
    om, streams = world
    prompt, truth, runner = streams[0]
    caps = {}
    for ramp in (True, False):
        cfg = ExperimentConfig(mode="async-speculative", nodes=2, vocab_size=16, embed_dim=16,
                               target_layers=4, max_context=96, prompt_len=8, gen_len=24,
                               microbatch=4, alpha=1.0, cutoff=0.0, spec_ramp=ramp,
                               fold_frontier=False, max_inflight=0)
        r = np.random.Generator(np.random.PCG64(1))
        pipe = FakePipeline(om, [(0, 4)], cfg.partitions, r)
        draft = FakeDraft(truth, runner, cfg.alpha, 0, 96, r)
        head = Head(cfg, pipe, draft, prompt, 16)
        seen = []
        orig = head._draft_request

        def spy(truncate_to, feed, max_tokens, cutoff, _orig=orig, _seen=seen):
            _seen.append(max_tokens)
            return _orig(truncate_to, feed, max_tokens, cutoff)

        head._draft_request = spy
        head.run_async_speculative()
        assert head.accepted[len(prompt):] == truth[len(prompt):len(prompt) + 24]
        caps[ramp] = seen
    ramp, flat = [c for c in caps[True] if c > 0], [c for c in caps[False] if c > 0]  # (0: prefill feed)
    assert ramp[0] == 1 and all(1 <= c <= 4 for c in ramp)
    assert set(flat) == {4}


def test_fold_frontier_one_stage(world):
    """B200 policy on a 1-stage pipeline (fold_frontier, max_inflight=1):
    every run after the prefill carries the frontier token followed by the
    draft's proposals (sync-speculative's run shape, engine.py:955-970), no
    run is cancelled, and the stream is the serial one."""
    om, streams = world
    prompt, truth, runner = streams[2]
    r = np.random.Generator(np.random.PCG64(5))
    cfg = ExperimentConfig(mode="async-speculative", nodes=2, vocab_size=16, embed_dim=16,
                           target_layers=4, max_context=96, prompt_len=8, gen_len=30,
                           alpha=0.7, cutoff=0.0)
    pipe = FakePipeline(om, [(0, 4)], cfg.partitions, r)
    head = Head(cfg, pipe, FakeDraft(truth, runner, 0.7, 1, 96, r), prompt, 16)
    assert head.fold_frontier and head.max_inflight == 1     # the 1-stage defaults
    head.run_async_speculative()
    assert head.accepted[len(prompt):] == truth[len(prompt):len(prompt) + 30]
    assert head.folded_runs == head.runs_started - 1 > 0
    assert head.cancelled_invalid + head.cancelled_superfluous == 0
    for rec in head.records[1:]:
        assert len(rec.tokens) >= 2 and rec.tokens[0] == truth[rec.min_pos]


@pytest.mark.parametrize("mode,nodes", [("sync-speculative", 3), ("async-speculative", 2),
                                        ("async-speculative", 4)])
def test_tree_speculation_matches_serial(world, mode, nodes):
    """tree_width 2: every proposal carries the draft's runner-up as a
    sibling leaf on its own partition (visibility per build_tree_mask,
    model.py:262-284); the head accepts a sibling that equals the target's
    greedy token and takes its row's prediction as the next token.  Streams
    equal the serial ones, siblings get accepted, and a tree round accepts
    more tokens per run than a chain round."""
    om, streams = world
    prompt, truth, runner = streams[0]
    per_run = {}
    for width in (1, 2):
        r = np.random.Generator(np.random.PCG64(11))
        cfg = ExperimentConfig(mode=mode, nodes=nodes, vocab_size=16, embed_dim=16,
                               target_layers=4, max_context=96, prompt_len=8, gen_len=36,
                               alpha=0.5, cutoff=0.0, tree_width=width, partitions=16)
        pipe = FakePipeline(om, plan_layer_split(4, cfg.n_stages()), cfg.partitions, r)
        draft = FakeDraft(truth, runner, 0.5, 4, 96, r, alpha_sibling=0.6 if width == 2 else 0.0)
        head = Head(cfg, pipe, draft, prompt, 16)
        {"sync-speculative": head.run_sync_speculative,
         "async-speculative": head.run_async_speculative}[mode]()
        assert head.accepted[len(prompt):] == truth[len(prompt):len(prompt) + 36], width
        completed = sum(1 for rec in head.records if rec.status == "completed")
        per_run[width] = 36 / completed
        if width == 2:
            assert head.tree_siblings > 0
            # (a 3-stage pipeline completes few speculative runs on 36 tokens)
            assert head.sibling_hits > 0 or nodes > 2
            assert not head.allocator.live()          # every partition released
    if mode == "sync-speculative":
        assert per_run[2] > per_run[1]


def test_common_prefix_matches_elementwise_scan():
    """Head._common_prefix (slice compares) == the element-wise scan it
    replaced, for lists and tuples, equal / prefix / diverging contexts."""
    import random
    from paper_2407_11798_b200.engine import Head

    def scan(a, b):
        n = 0
        for x, y in zip(a, b):
            if x != y:
                break
            n += 1
        return n

    rng = random.Random(7)
    for _ in range(3000):
        la, lb = rng.randint(0, 700), rng.randint(0, 700)
        base = [rng.randint(0, 5) for _ in range(max(la, lb))]
        a, b = base[:la], list(base[:lb])
        if b and rng.random() < 0.6:
            i = rng.randrange(len(b))
            b[i] += 1
        if rng.random() < 0.2:
            b = tuple(b)
        assert Head._common_prefix(a, b) == scan(a, b)
