"""Phase timeline of the persistent decode stage kernel (stagemk.cu): CTA 0's
clock64 at every phase start (barrier passed) and end (work done), for one
graph-replayed 7B stage-run (32 layers, 1 token)."""
import os
import sys

os.environ["SP_MK_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.model import BatchToken, encode_tokens
from paper_2407_11798_b200.pipeline import LocalPipeline

cfg = sp.llama_config("llama2-7b")
m = sp.build_model(cfg, torch.device("cuda", 0))
pipe = LocalPipeline(m, [(0, 32)], partitions=8, capacity=4096, max_tokens=256)
ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 384
pre = [BatchToken(5 + (i % 100), i, frozenset([0]), i == ctx - 1) for i in range(ctx)]
for c0 in range(0, ctx, 128):
    chunk = pre[c0:c0 + 128]
    pipe.launch(c0, 0, encode_tokens(chunk), 0, [len(chunk) - 1])
    pipe.wait()
for rep in range(4):
    pipe.launch(1000 + rep, 1, encode_tokens([BatchToken(7, ctx + rep, frozenset([0]), True)]), 0, [0])
    pipe.wait()
st = pipe.stages[0]
buf = (C.c_longlong * 16384)()
n_all = st.lib.sp_stage_draft_profile(st.h, buf, 16383)
allraw = np.array(buf[:n_all], dtype=np.int64)
n = int(allraw[16381])
raw = allraw[:n]
site = raw >> 56
clk = raw & ((1 << 56) - 1)
MHZ = float(os.environ.get("SM_MHZ", "1965"))
NAMES = ["QKV", "ATTN", "O", "UP", "DOWN"]
work = {k: [] for k in NAMES}
wait = {k: [] for k in NAMES}
att = {}
for i in range(1, n):
    dt = (clk[i] - clk[i - 1]) / MHZ
    s0, s1 = int(site[i - 1]), int(site[i])
    if s1 >= 30:
        att.setdefault(f"{s0}->{s1}", []).append(dt)
        continue
    if s1 >= 20:
        work[NAMES[s1 - 20]].append(dt)
    elif s1 >= 10:
        wait[NAMES[s1 - 10]].append(dt)
for k, v in sorted(att.items()):
    print(f"  attention {k}: n={len(v)} mean {np.mean(v):6.2f} us")
print(f"ctx {ctx}: {n} stamps, CTA-0 span {(clk[-1] - clk[0]) / MHZ:.1f} us")
for k in NAMES:
    w, b = np.array(work[k] or [0]), np.array(wait[k] or [0])
    print(f"  {k:5s} work mean {w.mean():6.2f} us (total {w.sum():7.1f})   "
          f"barrier-wait before it mean {b.mean():6.2f} us (total {b.sum():7.1f})")

G = int(os.environ.get("MK_G", "148"))
t0 = allraw[4095:4095 + G]
t1 = allraw[4095 + 512:4095 + 512 + G]
base = t0.min()
print("layer-5 attention per CTA (us from first start): start min/max %.2f/%.2f  end min/median/max %.2f/%.2f/%.2f"
      % (0, (t0.max() - base) / 1e3, (t1.min() - base) / 1e3, np.median(t1 - base) / 1e3, (t1.max() - base) / 1e3))
order = np.argsort(t1)[-8:]
print("slowest CTAs:", [(int(c), round((t1[c] - base) / 1e3, 2)) for c in order])

u = allraw[4095 + 1024:4095 + 1024 + G * 8].reshape(G, 8)
for c in list(order[-4:]) + [0, 1]:
    ends = [(round((u[c, 2 * k] - base) / 1e3, 2), int(u[c, 2 * k + 1])) for k in range(4) if u[c, 2 * k] > 0]
    print("CTA", int(c), "unit ends (us, merged?)", ends, "attn end", round((t1[c] - base) / 1e3, 2))

pe = allraw[10239:10239 + 5 * 512].reshape(5, 512)[:, :G]
for ph, name in enumerate(NAMES):
    v = (pe[ph] - pe[ph].min()) / 1e3
    print(f"layer-5 {name:5s} per-CTA end spread: median {np.median(v):5.2f} p90 {np.percentile(v, 90):5.2f} max {v.max():5.2f} us; latest CTAs {list(np.argsort(v)[-5:])}")

nm = allraw[12799:12799 + 5 * 512].reshape(5, 512)[:, :G]
for ph, name in enumerate(NAMES):
    v = (pe[ph] - pe[ph].min()) / 1e3
    late = v > np.percentile(v, 90)
    print(f"  {name:5s} merges per CTA: late (p90+) mean {nm[ph][late].mean():.2f}, others {nm[ph][~late].mean():.2f};"
          f" late CTAs b<148: {int((np.where(late)[0] < 148).sum())}/{int(late.sum())}")
