"""Where a 1-GPU generation's device time goes, per run (SP_RUN_TIMING=1).

Runs the bench workload (7B-shape target + 160M-shape draft, synthetic
draft, alpha 0.66) in the given modes and, from timing events recorded on
the stage stream around every run and on the draft stream around every
request, prints: stage busy time split by what the run turned out to be
(completed / cancelled mid-flight / skipped before start), stage idle time,
mean run cost by token count, and draft busy time.  Not product code: a
design tool for the head's scheduling policy.

    python tools/async_timeline.py [--gen-len 256] [--modes async-speculative,...]
           [--kw spec_ramp=False ...]
"""
import argparse
import ast
import collections
import os
import sys

os.environ["SP_RUN_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2407_11798_b200 import engine as E  # noqa: E402


def analyse(eng, res, label):
    pipe = eng.pipe
    recs = {r.run_id: r for r in res.records}
    tl = pipe.timeline
    ref = tl[0][3]
    rows = []
    for run_id, kind, n, e0, e1 in tl:
        rows.append((run_id, n, ref.elapsed_time(e0), ref.elapsed_time(e1)))
    busy = collections.defaultdict(float)
    count = collections.Counter()
    by_n = collections.defaultdict(list)
    idle, prev_end = 0.0, rows[0][2]
    for run_id, n, t0, t1 in rows:
        start = max(t0, prev_end)
        idle += max(0.0, t0 - prev_end)
        dur = t1 - start
        rec = recs.get(run_id)
        st = rec.status if rec is not None else "?"
        if st == E.COMPLETED:
            cls = "completed"
            by_n[n].append(dur)
        elif dur > 0.3:
            cls = "cancelled-midflight"
        else:
            cls = "skipped"
        busy[cls] += dur
        count[cls] += 1
        prev_end = t1
    span = rows[-1][3] - rows[0][2]
    m = res.metrics
    print(f"== {label}: {m.tokens_generated} tokens, {m.generation_speed:.1f} tok/s, "
          f"span {span:.1f} ms, runs {len(rows)}")
    for cls in ("completed", "cancelled-midflight", "skipped"):
        if count[cls]:
            print(f"   {cls:20s} n={count[cls]:5d} busy {busy[cls]:8.1f} ms "
                  f"({busy[cls] / span:5.1%})  mean {busy[cls] / count[cls]:.3f} ms")
    print(f"   {'stage idle':20s}        {idle:8.1f} ms ({idle / span:5.1%})")
    print("   completed run cost by tokens: " + ", ".join(
        f"M={n}: {sum(v) / len(v):.3f} ms x{len(v)}" for n, v in sorted(by_n.items())))
    tokens_per_completed = m.tokens_generated / max(1, count["completed"])
    print(f"   tokens per completed run {tokens_per_completed:.2f}")
    d = getattr(eng, "_table_draft", None) or eng.draft
    if d is not None and d.timeline:
        dd = [(nf, npr, ref.elapsed_time(a), ref.elapsed_time(b)) for nf, npr, a, b in d.timeline]
        dd = [x for x in dd if x[2] >= -1.0]
        tot = sum(b - a for _, _, a, b in dd)
        fw = collections.defaultdict(list)
        for nf, npr, a, b in dd:
            fw[(min(nf, 1), npr)].append(b - a)
        print(f"   draft: {len(dd)} requests, busy {tot:.1f} ms ({tot / span:5.1%}); "
              + ", ".join(f"feed{k[0]}+{k[1]}: {sum(v) / len(v):.3f} ms x{len(v)}"
                          for k, v in sorted(fw.items())))
        d.timeline.clear()
    pipe.timeline.clear()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gen-len", type=int, default=256)
    ap.add_argument("--modes", default="async-speculative,sync-speculative,pipeline-iterative")
    ap.add_argument("--kw", action="append", default=[])
    a = ap.parse_args()
    kw = {}
    for s in a.kw:
        k, v = s.split("=", 1)
        kw[k] = ast.literal_eval(v)
    cfg = E.ExperimentConfig(mode="async-speculative", nodes=2, target_shape=B.TARGET,
                             draft_shape=B.DRAFT, draft_backend="synthetic", alpha=B.ALPHA,
                             prompt_len=B.PROMPT_LEN, gen_len=a.gen_len, max_context=B.MAX_CTX,
                             target_seed=1, draft_seed=2, **kw)
    eng = E.Engine(cfg)
    for mode in a.modes.split(","):
        eng.run(prompt_seed=1234, mode=mode)     # warm (graphs, truth table)
        eng.pipe.timeline.clear()
        d = getattr(eng, "_table_draft", None)
        if d is not None:
            d.timeline.clear()
        torch.cuda.synchronize()
        res = eng.run(prompt_seed=1234, mode=mode)
        torch.cuda.synchronize()
        analyse(eng, res, mode)


if __name__ == "__main__":
    main()
