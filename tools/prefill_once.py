"""One 128-token prefill run through the 7B shape (the M=128 tensor-core
GEMMs and attention) -- an ncu target.  Design tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_11798_b200 as sp  # noqa: E402
from paper_2407_11798_b200.model import BatchToken, encode_tokens  # noqa: E402
from paper_2407_11798_b200.pipeline import LocalPipeline  # noqa: E402

cfg = sp.llama_config("llama2-7b", max_context=1024)
m = sp.build_model(cfg, torch.device("cuda", 0))
pipe = LocalPipeline(m, [(0, 32)], partitions=8, capacity=4096, max_tokens=256)
ts = []
for rep in range(int(os.environ.get("REPS", "2"))):
    toks = [BatchToken(5 + (i % 100), i, frozenset([0]), i == 127) for i in range(128)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(pipe.stream)
    pipe.launch(rep, 0, encode_tokens(toks), 0, [127])
    e1.record(pipe.stream)
    pipe.wait()
    ts.append(e0.elapsed_time(e1))
    pipe.reset()
torch.cuda.synchronize()
print("ok: 128-token prefill ms", [round(t, 2) for t in ts])
