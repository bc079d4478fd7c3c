"""Iterative (one token per run) decode of the bench workload: wall time per
token vs GPU-busy time per token (CUPTI via torch.profiler) -> host overhead."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench as B
from paper_2407_11798_b200.engine import Engine, ExperimentConfig

mode = sys.argv[1] if len(sys.argv) > 1 else "iterative"
cfg = ExperimentConfig(mode=mode, nodes=2, target_shape=B.TARGET, draft_shape=B.DRAFT,
                       draft_backend="synthetic", alpha=B.ALPHA, prompt_len=B.PROMPT_LEN,
                       gen_len=64, max_context=B.MAX_CTX, target_seed=1, draft_seed=2)
eng = Engine(cfg)
eng.run(prompt_seed=1234)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    r = eng.run(prompt_seed=1234)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
prof.export_chrome_trace("/tmp/it.json")
ev = json.load(open("/tmp/it.json"))["traceEvents"]
k = [e for e in ev if e.get("cat") == "kernel"]
busy = sum(e["dur"] for e in k)
k.sort(key=lambda e: e["ts"])
span = (k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]) if k else 0
n = len(r.tokens)
print(f"{mode}: {n} tokens, wall {wall*1e3:.1f} ms, speed metric {r.metrics.generation_speed:.1f} tok/s")
print(f"  kernels {len(k)}, busy {busy/1e3:.1f} ms ({busy/1e3/n:.3f} ms/token), span {span/1e3:.1f} ms")
print("  host profile", {kk: round(v, 4) for kk, v in r.host_profile.items()})
