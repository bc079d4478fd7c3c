"""Phase timeline of the K15 persistent draft kernel (CTA 0's clock64 at
every phase edge, tagged with the phase id): work vs barrier time."""
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
shape = sys.argv[1] if len(sys.argv) > 1 else "llama-160m"
cfg = sp.llama_config(shape)
dm = sp.build_model(cfg, dev, tiled=False)
srv = TableDraftServer(dm, list(range(2000)), list(range(2000)), 0.66, 1)
if os.environ.get("KIND", "grid") == "grid":   # the exclusive (whole-GPU) kernel, draft.cu
    srv.shared_gpu = True
    srv.set_exclusive(True)
srv.request(0, list(range(128)), 0, 1.0); srv.reply()
for _ in range(5):
    srv.request(len(srv), [7], 4, 0.0); srv.reply()
buf = (C.c_longlong * 4096)()
n = srv.stage.lib.sp_stage_draft_profile(srv.stage.h, buf, 4096)
raw = np.array(buf[:n], dtype=np.int64)
site = raw >> 56
clk = raw & ((1 << 56) - 1)
MHZ = float(os.environ.get("SM_MHZ", "1965"))
dt = np.diff(clk) / MHZ
NAMES = {1: "A", 2: "B", 3: "C", 4: "D", 5: "E", 6: "H"}
agg = {}
for i in range(len(dt)):
    s0, s1 = int(site[i]), int(site[i + 1])
    if 60 <= s1 <= 66:
        key = {60: "B.kvloads-issue", 61: "B.q+scores", 62: "B.max-sync", 63: "B.pv+sum",
               64: "B.merge", 65: "B.wo-issue", 66: "B.opart"}[s1]
    elif s1 == 2 and s0 == 66:
        key = "B.tail"
    elif 40 <= s1 <= 43:
        key = {40: "A.wload", 41: "A.prefetch", 42: "A.loads+stores", 43: "A.syncthreads"}[s1]
    elif s1 == 33 and s0 == 43:
        key = "A.scales"
    elif s1 >= 48:
        key = NAMES[s1 - 48] + ".wait"
    elif s1 >= 32:
        key = NAMES[s1 - 32] + ".stage"
    elif s1 in NAMES and s0 >= 48:
        key = NAMES[s1] + ".compute"
    elif s1 in NAMES:            # work interval ending at phase s1's barrier
        key = NAMES[s1] + (" (after merge)" if s0 == 14 else "")
    elif s1 >= 9 and s1 - 8 in NAMES:
        key = "sync" + NAMES[s1 - 8]
    else:
        key = f"other {s0}->{s1}"
    agg.setdefault(key, []).append(dt[i])
print(f"{shape}: {n} stamps, total {(clk[-1] - clk[0]) / MHZ:.1f} us (clock64 @ {MHZ} MHz)")
for k in sorted(agg, key=lambda k: -sum(agg[k])):
    v = np.array(agg[k])
    print(f"  {k:18s} n={len(v):4d} mean {v.mean():7.2f} us  p50 {np.median(v):7.2f}"
          f"  max {v.max():7.2f}  total {v.sum():8.1f}")
