"""Kernel timeline (CUPTI via torch.profiler) of one 160M-draft forward+head:
per-kernel device time and the gaps between consecutive kernels."""
import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.drafting import TableDraftServer

dev = torch.device("cuda", 0)
shape = sys.argv[1] if len(sys.argv) > 1 else "llama-160m"
dm = sp.build_model(sp.llama_config(shape), dev, tiled=bool(int(os.environ.get("DRAFT_TC", "0"))))
srv = TableDraftServer(dm, list(range(2000)), list(range(2000)), 0.66, 1)
srv.request(0, list(range(128)), 0, 1.0); srv.reply()
for _ in range(3):
    srv.request(len(srv), [7], 4, 0.0); srv.reply()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    srv.request(len(srv), [7], 4, 0.0); srv.reply()
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"]
      if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], ev[-1]["ts"] + ev[-1]["dur"]
busy = sum(e["dur"] for e in ev)
by = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].split("(")[0].replace("void ", "")[:60]
    by[k][0] += 1; by[k][1] += e["dur"]
print(f"{shape}: {len(ev)} kernels, span {t1 - t0:.1f} us, kernel-busy {busy:.1f} us, "
      f"gaps {t1 - t0 - busy:.1f} us")
for k, (n, d) in sorted(by.items(), key=lambda x: -x[1][1]):
    print(f"  {k:60s} n={n:3d} total {d:8.1f} us  avg {d / n:6.2f} us")
cpu = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"]
       if e.get("cat") in ("cuda_runtime", "cuda_driver")]
print("cuda runtime calls:", len(cpu), "host us:", round(sum(e["dur"] for e in cpu), 1))
byc = collections.defaultdict(lambda: [0, 0.0])
for e in cpu:
    byc[e["name"]][0] += 1; byc[e["name"]][1] += e["dur"]
for k, (n, d) in sorted(byc.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {k:40s} n={n:3d} total {d:8.1f} us")
import time
for nprop in (1, 4):
    tq, tr = [], []
    for _ in range(20):
        torch.cuda.synchronize()
        a = time.perf_counter()
        srv.request(len(srv), [7], nprop, 0.0)
        b = time.perf_counter()
        srv.reply()
        c = time.perf_counter()
        tq.append(b - a); tr.append(c - b)
    tq.sort(); tr.sort()
    print(f"props={nprop}: request() host {tq[10]*1e6:.0f} us, reply() wait {tr[10]*1e6:.0f} us")
