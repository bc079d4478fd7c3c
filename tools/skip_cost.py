"""GPU time of one 7B stage-run (32 layers, 1 token, graph-replayed) when it
runs vs when it is cancelled before it starts (gate skip) -- the cost an
abandoned speculative run still pays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200 import _lib
from paper_2407_11798_b200.model import BatchToken, encode_tokens
from paper_2407_11798_b200.pipeline import LocalPipeline

cfg = sp.llama_config("llama2-7b")
m = sp.build_model(cfg, torch.device("cuda", 0))
pipe = LocalPipeline(m, [(0, 32)], partitions=8, capacity=4096, max_tokens=256)
CTX = int(os.environ.get("CTX", "128"))
pre = [BatchToken(5 + (i % 100), i, frozenset([0]), i == CTX - 1) for i in range(CTX)]
for c0 in range(0, CTX, 128):
    chunk = pre[c0:c0 + 128]
    pipe.launch(1 + c0, 0, encode_tokens(chunk), 0, [len(chunk) - 1])
    pipe.wait()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
SPEC = _lib.SP_KIND_SPEC
flags = _lib.SP_FWD_SKIPPABLE
import time
times = {"run": [], "skipped": [], "cancelled_at_1ms": []}
rid = 10000
for rep in range(12):
    for kind in ("run", "skipped", "cancelled_at_1ms"):
        toks = encode_tokens([BatchToken(7, CTX + rep, frozenset([1]), True)])
        if kind == "skipped":
            pipe.cancel_run(rid)
        torch.cuda.synchronize()
        ev[0].record(pipe.stream)
        pipe.launch(rid, SPEC, toks, flags, [0])
        ev[1].record(pipe.stream)
        if kind == "cancelled_at_1ms":   # mid-flight: the head cancels ~1 ms in
            time.sleep(0.001)
            pipe.cancel_run(rid)
        pipe.wait()
        ev[1].synchronize()
        if rep >= 2:
            times[kind].append(ev[0].elapsed_time(ev[1]))
        pipe.remove(1, 0)
        rid += 1
for k, v in times.items():
    print(f"{k:8s} median {np.median(v)*1e3:8.1f} us")
