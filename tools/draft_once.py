"""A few draft requests (feed 1 + propose 4) of the 160M-shape draft on an
otherwise idle GPU -- the ncu target for the draft kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.drafting import TableDraftServer

dev = torch.device("cuda", 0)
dm = sp.build_model(sp.llama_config(sys.argv[1] if len(sys.argv) > 1 else "llama-160m"), dev,
                    tiled=False)
srv = TableDraftServer(dm, list(range(4000)), list(range(4000)), 0.66, 1)
srv.request(0, list(range(128)), 0, 1.0)
srv.reply()
for _ in range(int(os.environ.get("REQS", "4"))):
    srv.request(len(srv), [7], 4, 0.0)
    srv.reply()
torch.cuda.synchronize()
print("ok")
