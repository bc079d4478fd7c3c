"""Wall time of a draft server's 128-token prompt feed (160M / 1.1B shapes).  Design tool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.drafting import TableDraftServer
dev = torch.device("cuda", 0)
for shape in ("llama-160m", "tinyllama-1.1b"):
    dm = sp.build_model(sp.llama_config(shape), dev, tiled=False)
    srv = TableDraftServer(dm, list(range(4000)), list(range(4000)), 0.66, 1)
    ts = []
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        srv.request(0, list(range(128)), 0, 1.0)
        srv.reply()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(shape, "128-token feed ms", [round(t, 2) for t in ts])
