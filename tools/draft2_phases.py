"""Cluster-form K15: per-edge timeline of CTA 0 (work = edge-to-edge minus
the barrier wait) and the total time spent waiting for ring chunks."""
import ctypes as C
import os
import sys

os.environ["SP_DRAFT_PROF"] = "1"
os.environ.setdefault("SP_DRAFT_FUSED", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.drafting import TableDraftServer

dev = torch.device("cuda", 0)
cfg = sp.llama_config(sys.argv[1] if len(sys.argv) > 1 else "llama-160m")
dm = sp.build_model(cfg, dev, tiled=False)
srv = TableDraftServer(dm, list(range(2000)), list(range(2000)), 0.66, 1)
srv.request(0, list(range(128)), 0, 1.0); srv.reply()
for _ in range(3):
    srv.request(len(srv), [7], 4, 0.0); srv.reply()
buf = (C.c_longlong * 4096)()
n = srv.stage.lib.sp_stage_draft_profile(srv.stage.h, buf, 4096)
raw = np.array(buf[:n], dtype=np.int64)
site = raw >> 56
val = raw & ((1 << 56) - 1)
MHZ = 1965.0
wait = val[-1] / MHZ
clk = val[:-1]
st = site[:-1]
work, edge = [], []
sub = {}
for i in range(1, len(clk)):
    dt = (clk[i] - clk[i - 1]) / MHZ
    if st[i] in (20, 21, 22, 23):
        sub.setdefault(int(st[i]), []).append(dt)
        continue
    if st[i - 1] in (20, 21, 22, 23):
        sub.setdefault(99, []).append(dt)
        continue
    (edge if st[i] == 9 else work).append(dt)
for k, v in sorted(sub.items()):
    print(f"  D sub {k}: mean {np.mean(v):.2f} us")
work, edge = np.array(work), np.array(edge)
print(f"{len(clk)} stamps; total {(clk[-1] - clk[0]) / MHZ:.1f} us; ring-wait {wait:.1f} us")
print(f"work  n={len(work)} mean {work.mean():.2f} p50 {np.median(work):.2f} max {work.max():.2f} total {work.sum():.1f}")
print(f"edge  n={len(edge)} mean {edge.mean():.2f} p50 {np.median(edge):.2f} max {edge.max():.2f} total {edge.sum():.1f}")
per = 5
for i in range(min(3 * per, len(work))):
    print(f"  phase {i % per}: work {work[i]:.2f}  edge {edge[i] if i < len(edge) else -1:.2f}")
