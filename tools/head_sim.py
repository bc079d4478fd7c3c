"""Virtual-time model of the head's scheduling policies on B200 costs.

Drives the REAL ``engine.Head`` (verification, cancellation, speculation
decisions) against a modelled pipeline and draft with B200-measured costs,
so head policies can be compared on CPU before spending GPU time:

* a stage-run costs ``t_stage`` per stage regardless of its token count
  (weight streaming; measured flat for M <= 16), a cancelled run whose gate
  sees the cancel word costs ``t_skip``, a run cancelled mid-flight stops at
  the next observation point (every ``1/obs`` of the stage);
* runs are FIFO per stage; stage i+1 starts a run when stage i finished it
  (+ ``t_hop``) and is free;
* the draft serves one request at a time: ``t_req + t_tok * forwards``;
* each head action costs host time (``h_*``).

Usage: python tools/head_sim.py [--n 1] [--alpha 0.66] [policy knobs...]
Not product code: a design tool (DESIGN.md §5c cites its outputs).
"""

from __future__ import annotations

import argparse
import heapq
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_11798_b200 import engine as E  # noqa: E402
from paper_2407_11798_b200.model import RowResult  # noqa: E402
from paper_2407_11798_b200.pipeline import RunResult  # noqa: E402


class Clock:
    def __init__(self):
        self.t = 0.0


class SimPipeline:
    def __init__(self, clock, n_stages, t_stage, t_skip, obs, t_hop, t_launch, truth,
                 runner, t_head=0.0):
        self.c = clock
        self.n_stages = n_stages
        self.t_stage, self.t_skip, self.obs, self.t_hop = t_stage, t_skip, obs, t_hop
        self.t_launch, self.t_head = t_launch, t_head
        self.truth, self.runner = truth, runner
        self.fifo = []               # launched runs (dicts), FIFO
        self.cancel_t = {}           # run_id -> time the cancel word was set
        self.stage_free = [0.0] * n_stages
        self.busy = 0.0              # GPU-seconds of stage time spent
        self.cancelled_cost = 0.0

    # -- schedule a run through the stages at launch (cancels are consulted
    #    lazily: a run's stage segments are computed when first needed) -----
    def launch(self, run_id, kind, toks, flags, rows):
        r = dict(id=run_id, toks=[(int(t["token"]), int(t["pos"])) for t in toks],
                 skippable=bool(flags & 2), rows=list(rows), t0=self.c.t + self.t_launch,
                 done=None, placeholder=False, stage=0, ready=self.c.t + self.t_launch)
        self.fifo.append(r)

    def copy(self, *a):
        pass

    def remove(self, *a):
        pass

    def cancel_run(self, run_id):
        self.cancel_t.setdefault(run_id, self.c.t)

    def _cancelled_by(self, r, t):
        ct = self.cancel_t.get(r["id"])
        return r["skippable"] and ct is not None and ct <= t

    def _advance_run(self, r, upto, prev_stage):
        """Progress run r through the stages it may enter (FIFO per stage:
        stage s only after the previous run left it) while its decisions fall
        before ``upto``; returns the time of its next pending decision."""
        while r["done"] is None:
            s = r["stage"]
            if s >= prev_stage:
                return None                     # waits for the previous run
            start = max(r["ready"], self.stage_free[s])
            if start > upto:
                return start
            if r["placeholder"] or self._cancelled_by(r, start):
                end = start + self.t_skip
                r["placeholder"] = True
                self.cancelled_cost += self.t_skip
            else:
                T = self.t_stage + (self.t_head if s == self.n_stages - 1 else 0.0)
                end = start + T
                if r["skippable"]:
                    for k in range(1, self.obs):
                        tb = start + T * k / self.obs
                        if tb > upto:      # decide later (a cancel may still come)
                            return tb
                        if self._cancelled_by(r, tb):
                            end = tb + self.t_skip
                            r["placeholder"] = True
                            self.cancelled_cost += end - start
                            break
                self.busy += end - start
            self.stage_free[s] = end
            r["ready"] = end + self.t_hop
            r["stage"] += 1
            if r["stage"] == self.n_stages:
                r["done"] = end
        return r["done"]

    def _advance(self, upto):
        nxt = []
        prev = self.n_stages
        for r in self.fifo:
            t = self._advance_run(r, upto, prev)
            if t is not None:
                nxt.append(t)
            prev = r["stage"] if r["done"] is None else self.n_stages
        return nxt

    def next_event(self):
        """Earliest time the modelled GPU changes state (a completion or a
        pending stage/observation decision)."""
        if not self.fifo:
            return None
        nxt = [t for t in self._advance(self.c.t) if t is not None]
        later = [t for t in nxt if t > self.c.t]
        return min(later) if later else self.c.t + 1e-7

    def ready(self):
        if not self.fifo:
            return False
        self._advance(self.c.t)
        return self.fifo[0]["done"] is not None and self.fifo[0]["done"] <= self.c.t

    def _rows(self, r):
        out = []
        # predictions along the run's own tokens; the head only consumes rows
        # of runs whose chain is on the true path up to the row
        for i in r["rows"]:
            tok, pos = r["toks"][i]
            ok = all(self.truth[p] == t for t, p in r["toks"][:i + 1])
            a = self.truth[pos + 1] if ok and pos + 1 < len(self.truth) else 0
            b = self.runner[pos + 1] if ok and pos + 1 < len(self.runner) else 1
            if not ok:
                a, b = (self.truth[pos + 1] + 1) % 32000, a
            out.append(RowResult(a, b, 0.5))
        return out

    def poll(self):
        r = self.fifo.pop(0)
        return RunResult(r["id"], r["placeholder"], [] if r["placeholder"] else self._rows(r), 0,
                         [2 if r["placeholder"] else 0] * self.n_stages)

    def wait(self):
        while not self.ready():
            self.c.t = max(self.c.t, self.next_event())
        return self.poll()

    def in_flight(self):
        return len(self.fifo)

    def reset(self):
        pass


class SimDraft:
    def __init__(self, clock, truth, runner, alpha, seed, t_req, t_tok):
        self.c = clock
        self.truth, self.runner = truth, runner
        self.alpha = alpha
        self.rng = np.random.Generator(np.random.PCG64(seed))
        self.t_req, self.t_tok = t_req, t_tok
        self.tokens = []
        self.done = None
        self.props = None
        self.forwards = 0
        self.free_at = 0.0

    def request(self, truncate_to, feed, max_tokens, cutoff):
        del self.tokens[truncate_to:]
        self.tokens.extend(feed)
        budget = max(0, int(max_tokens))
        props = []
        if budget > 0 and not self.alpha < cutoff:
            for _ in range(budget):
                p = len(self.tokens)
                best = self.truth[p] if p < len(self.truth) else 0
                sec = self.runner[p] if p < len(self.runner) else 1
                t = best if self.rng.random() < self.alpha else sec
                self.tokens.append(t)
                props.append(t)
        n_fwd = (1 if feed else 0) + len(props)
        start = max(self.c.t, self.free_at)
        self.done = start + self.t_req + self.t_tok * n_fwd
        self.free_at = self.done
        self.props = tuple(props)
        self.forwards += n_fwd

    def ready(self):
        return self.done is not None and self.done <= self.c.t

    def reply(self):
        if self.done > self.c.t:
            self.c.t = self.done
        self.done = None
        return self.props, tuple(self.alpha for _ in self.props)


class SimHead(E.Head):
    """The engine's Head on a virtual clock with host costs per action."""

    H_COMPLETION, H_REPLY, H_REQUEST = 50e-6, 80e-6, 40e-6

    def __init__(self, clock, *a, **k):
        self.clock = clock
        super().__init__(*a, **k)

    def now(self):
        return self.clock.t

    def _handle_completion(self, res):
        super()._handle_completion(res)
        self.clock.t += self.H_COMPLETION

    def _handle_reply(self, toks, confs):
        super()._handle_reply(toks, confs)
        self.clock.t += self.H_REPLY

    def _send_draft_request(self):
        super()._send_draft_request()
        self.clock.t += self.H_REQUEST

    def _block_until_message(self):
        if self.pipe.in_flight() == 0 and not self.draft_busy:
            raise E.EngineError("deadlock")
        cands = []
        ne = self.pipe.next_event()
        if ne is not None:
            cands.append(ne)
        if self.draft_busy:
            cands.append(self.draft.done)
        self.clock.t = max(self.clock.t, min(cands))


def run(args, mode, seed=1234, **kw):
    V = 32000
    rng = np.random.Generator(np.random.PCG64(seed))
    n = 128 + args.gen + 64
    truth = [int(x) for x in rng.integers(0, V, n)]
    runner = [int((t + 1 + rng.integers(0, V - 1)) % V) for t in truth]
    prompt = truth[:128]
    cfg = E.ExperimentConfig(mode=mode, nodes=args.n + 1, alpha=args.alpha, prompt_len=128,
                             gen_len=args.gen, max_context=1024, vocab_size=V,
                             draft_backend="synthetic", capacity=8192, **kw)
    clock = Clock()
    stages = args.n if mode != "iterative" else 1
    t_stage = args.t_run / stages
    pipe = SimPipeline(clock, stages, t_stage, args.t_skip, max(1, args.obs // stages), args.t_hop,
                       args.t_launch, truth, runner, t_head=args.t_head)
    draft = SimDraft(clock, truth, runner, args.alpha, 7 + seed, args.t_req, args.t_tok) \
        if cfg.uses_draft() else None
    head = SimHead(clock, cfg, pipe, draft, prompt, 4096)
    {"iterative": head.run_iterative, "pipeline-iterative": head.run_iterative,
     "sync-speculative": head.run_sync_speculative,
     "async-speculative": head.run_async_speculative}[mode]()
    assert head.accepted[128:] == truth[128:128 + len(head.accepted) - 128], "stream diverged"
    m = head.build_metrics(0.0)
    return m, pipe


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1, help="pipeline stages")
    ap.add_argument("--alpha", type=float, default=0.66)
    ap.add_argument("--gen", type=int, default=256)
    ap.add_argument("--t-run", type=float, default=2.60e-3, help="whole-model stage-run")
    ap.add_argument("--t-head", type=float, default=0.07e-3)
    ap.add_argument("--t-skip", type=float, default=0.06e-3)
    ap.add_argument("--t-hop", type=float, default=0.02e-3)
    ap.add_argument("--t-launch", type=float, default=0.03e-3)
    ap.add_argument("--obs", type=int, default=4, help="observation points per run")
    ap.add_argument("--t-req", type=float, default=0.05e-3)
    ap.add_argument("--t-tok", type=float, default=0.25e-3)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--kw", action="append", default=[],
                    help="ExperimentConfig override k=v (python literal)")
    args = ap.parse_args()
    import ast
    kw = {}
    for s in args.kw:
        k, v = s.split("=", 1)
        kw[k] = ast.literal_eval(v)
    for mode in ("pipeline-iterative", "sync-speculative", "async-speculative"):
        sp, runs, canc, busy, cc = [], [], [], [], []
        for s in range(args.seeds):
            m, pipe = run(args, mode, seed=1234 + s, **(kw if mode == "async-speculative" else
                                                        {k: v for k, v in kw.items()
                                                         if k in ("tree_cap", "partitions")}))
            sp.append(m.generation_speed)
            runs.append(m.runs_started)
            canc.append(m.cancelled_runs)
            busy.append(pipe.busy / max(1e-9, m.duration))
            cc.append(pipe.cancelled_cost)
        print(f"{mode:20s} {np.mean(sp):8.1f} tok/s  runs {np.mean(runs):6.0f}  "
              f"cancelled {np.mean(canc):6.0f}  stage-busy {np.mean(busy):.2f}  "
              f"cancel-cost {np.mean(cc)*1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
