"""One async-speculative generation of the bench workload (7B + 160M, bf16)
inside a cudaProfilerStart/Stop range, for ncu (--profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench as B
from paper_2407_11798_b200.engine import Engine, ExperimentConfig

ap = argparse.ArgumentParser()
ap.add_argument("--gen-len", type=int, default=16)
ap.add_argument("--mode", default="async-speculative")
ap.add_argument("--depth", type=int, default=3, help="speculation depth (bench N=1 default 3)")
a = ap.parse_args()
cfg = ExperimentConfig(mode="async-speculative", nodes=2, target_shape=B.TARGET,
                       draft_shape=B.DRAFT, draft_backend="synthetic", alpha=B.ALPHA,
                       prompt_len=B.PROMPT_LEN, gen_len=a.gen_len, max_context=B.MAX_CTX,
                       target_seed=1, draft_seed=2, microbatch=a.depth, tree_cap=a.depth)
eng = Engine(cfg)
for _ in range(2):
    eng.run(prompt_seed=1234, mode=a.mode)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = eng.run(prompt_seed=1234, mode=a.mode)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("tokens", len(r.tokens), "speed", round(r.metrics.generation_speed, 1))
