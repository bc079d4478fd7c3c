"""Latency of one draft request (feed 1 token + propose 4) of the 160M-shape
draft: alone on the GPU vs while target stage-runs (7B, 8 layers) stream on
another stream of the same GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.drafting import TableDraftServer
from paper_2407_11798_b200.runtime import Stage
from paper_2407_11798_b200.model import encode_tokens

dev = torch.device("cuda", 0)
dcfg = sp.llama_config("llama-160m")
dm = sp.build_model(dcfg, dev, tiled=bool(int(os.environ.get("DRAFT_TC", "0"))))
truth = list(range(2000)); runner = list(range(2000))
hi = torch.cuda.Stream.priority_range()[1]
srv = TableDraftServer(dm, truth, runner, 0.66, 1, stream=torch.cuda.Stream(dev, priority=hi))
srv.request(0, list(range(128)), 0, 1.0); srv.reply()

tcfg = sp.llama_config("llama2-7b")
tm = sp.build_model(tcfg, dev, layer_range=(0, 8), head=False)
tst = Stage(tm, 0, 8, capacity=4096, max_tokens=16, n_seq_ids=8, stream=torch.cuda.Stream(dev))
for budget in (0, 2 * 132):
    tst.set_cta_budget(budget)
    for busy in (False, True):
        lat = []
        for i in range(20):
            if busy:
                for j in range(3):
                    b = [sp.BatchToken(5, 200 + 3 * i + j, frozenset([0]), True)]
                    tst.forward(encode_tokens(b), 0, 1, 0)
            t0 = time.perf_counter()
            n = len(srv)
            srv.request(n, [7], 4, 0.0)
            srv.reply()
            lat.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
        lat.sort()
        print(f"budget={budget} busy={busy}: draft request (feed 1 + 4 proposals) "
              f"median {lat[len(lat)//2]*1e3:.3f} ms  min {lat[0]*1e3:.3f} ms", flush=True)
        tst.reset()
