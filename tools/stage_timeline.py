"""Kernel timeline of ONE graph-replayed 7B decode stage-run (32 layers + LM
head, 1 token): per kernel kind, the increment it adds to the run's critical
path (end-to-end of consecutive kernel ends, robust to PDL overlap)."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.model import BatchToken, encode_tokens
from paper_2407_11798_b200 import _lib
from paper_2407_11798_b200.pipeline import LocalPipeline

ctx_arg = int(sys.argv[1]) if len(sys.argv) > 1 else 384
cfg = sp.llama_config("llama2-7b", max_context=max(1024, ctx_arg + 64))
m = sp.build_model(cfg, torch.device("cuda", 0))
pipe = LocalPipeline(m, [(0, 32)], partitions=8, capacity=max(4096, ctx_arg + 256), max_tokens=256)
ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 384
pre = [BatchToken(5 + (i % 100), i, frozenset([0]), i == ctx - 1) for i in range(ctx)]
for c0 in range(0, ctx, 128):
    chunk = pre[c0:c0 + 128]
    pipe.launch(c0, 0, encode_tokens(chunk), 0, [len(chunk) - 1])
    pipe.wait()
M = int(os.environ.get("M", "1"))   # tokens per run (a verification run when > 1)
rid = 1000


def run_batch(p0):
    toks = [BatchToken(7 + i, p0 + i, frozenset([0]), True) for i in range(M)]
    # (coverage-checked, as every engine run is)
    pipe.launch(rid, 1 if M == 1 else 2, encode_tokens(toks), _lib.SP_FWD_CHECK_COVERAGE,
                list(range(M)))
    pipe.wait()
    pipe.remove(0, p0 + 1)       # keep one cell per run: contexts grow by one


for rep in range(4):   # warm + capture the graph
    run_batch(ctx + rep)
    rid += 1
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    run_batch(ctx + 4)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/st.json")
ev = [e for e in json.load(open("/tmp/st.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"] + e["dur"])
t_start = min(e["ts"] for e in ev)
prev_end = t_start
inc = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    end = e["ts"] + e["dur"]
    k = e["name"].split("(")[0].replace("void ", "").replace("sp::", "")[:36]
    g = e.get("args", {}).get("grid")
    if g and "gemm" in k:
        k += " g" + "x".join(str(v) for v in g)
    inc[k][0] += 1
    inc[k][1] += max(0.0, end - prev_end)
    prev_end = max(prev_end, end)
total = prev_end - t_start
print(f"ctx {ctx}: {len(ev)} kernels, run span {total:.1f} us")
for k, (n, t) in sorted(inc.items(), key=lambda x: -x[1][1]):
    print(f"  {k:44s} n={n:3d}  critical-path {t:8.1f} us  ({t / n:6.2f}/launch)")
