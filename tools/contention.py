"""How much a concurrently running draft slows the target's stage-runs on a
shared GPU (the N=1/2 layout), and which target kernels pay for it.

Back-to-back 1-token 7B stage-runs (32 layers + LM head, graph-replayed) on
the stage stream, with and without the 160M draft's persistent kernel
looping (feed 1 + propose 4) on its own high-priority stream; per-kernel
device time from torch.profiler (CUPTI).  Design tool, not product code.

    python tools/contention.py [--runs 60] [--budget 264]
"""
import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SP_RUN_TIMING"] = "1"

import torch  # noqa: E402

import paper_2407_11798_b200 as sp  # noqa: E402
from paper_2407_11798_b200.drafting import TableDraftServer  # noqa: E402
from paper_2407_11798_b200.model import BatchToken, encode_tokens  # noqa: E402
from paper_2407_11798_b200.pipeline import LocalPipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=60)
    ap.add_argument("--budget", type=int, default=264)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    tm = sp.build_model(sp.llama_config("llama2-7b"), dev)
    pipe = LocalPipeline(tm, [(0, 32)], partitions=8, capacity=4096, max_tokens=256)
    for st in pipe.stages:
        st.set_cta_budget(a.budget)
    dm = sp.build_model(sp.llama_config("llama-160m"), dev, tiled=False)
    hi = torch.cuda.Stream.priority_range()[1]
    srv = TableDraftServer(dm, list(range(8000)), list(range(8000)), 0.66, 1,
                           stream=torch.cuda.Stream(dev, priority=hi))
    srv.request(0, list(range(128)), 0, 1.0)
    srv.reply()
    ctx = 128
    pre = [BatchToken(5 + i, i, frozenset([0]), i == ctx - 1) for i in range(ctx)]
    pipe.launch(1, 0, encode_tokens(pre), 0, [ctx - 1])
    pipe.wait()
    state = {"rid": 2, "pos": ctx}

    def one_pass(with_draft, n):
        pipe.timeline.clear()
        srv.timeline.clear()
        inflight = 0
        done = 0
        while done < n:
            while inflight < 2 and state["rid"] - 2 < 10 ** 6:
                b = [BatchToken(7, state["pos"], frozenset([0]), True)]
                pipe.launch(state["rid"], 1, encode_tokens(b), 0, [0])
                state["rid"] += 1
                state["pos"] += 1
                inflight += 1
            if with_draft and not srv.busy():
                srv.request(len(srv), [7], 4, 0.0)
            if with_draft and srv.ready():
                srv.reply()
            if pipe.ready():
                pipe.poll()
                inflight -= 1
                done += 1
            if state["pos"] > 900:        # stay inside max_context
                while inflight:
                    pipe.wait()
                    inflight -= 1
                pipe.reset()
                pipe.launch(1, 0, encode_tokens(pre), 0, [ctx - 1])
                pipe.wait()
                state["pos"] = ctx
        while inflight:
            pipe.wait()
            inflight -= 1
        if srv.busy():
            srv.reply()
        torch.cuda.synchronize()
        tl = pipe.timeline
        ends = [e1 for *_, e1 in tl]
        gaps = [tl[0][3].elapsed_time(e) for e in ends]
        per = [(gaps[i] - gaps[i - 1]) for i in range(1, len(gaps))]
        per.sort()
        dr = [a0.elapsed_time(a1) for _, _, a0, a1 in srv.timeline]
        return per[len(per) // 2], (sum(dr) / len(dr) if dr else 0.0), len(dr)

    for with_draft in (False, True, False, True):
        t_run, t_req, nreq = one_pass(with_draft, a.runs)
        print(f"draft={'on ' if with_draft else 'off'}  target run median {t_run:.3f} ms   "
              f"draft request mean {t_req:.3f} ms x{nreq}", flush=True)
    # per-kernel attribution
    for with_draft in (False, True):
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            one_pass(with_draft, 20)
        path = f"/tmp/cont_{int(with_draft)}.json"
        prof.export_chrome_trace(path)
        ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
        agg = collections.defaultdict(lambda: [0, 0.0])
        for e in ev:
            k = e["name"].split("(")[0].replace("void ", "").replace("sp::", "")[:40]
            agg[k][0] += 1
            agg[k][1] += e["dur"]
        print(f"-- kernels, draft={'on' if with_draft else 'off'} (20 runs): total us / count / mean")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
            print(f"   {k:42s} {t:10.1f} {n:6d} {t / n:8.2f}")


if __name__ == "__main__":
    main()
