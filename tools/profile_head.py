"""cProfile of the head's host work during one async generation of the bench
workload (N=1): where the Python time between GPU events goes.  Design tool."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2407_11798_b200.engine import Engine, ExperimentConfig  # noqa: E402

cfg = ExperimentConfig(mode="async-speculative", nodes=2, target_shape=B.TARGET,
                       draft_shape=B.DRAFT, draft_backend="synthetic", alpha=B.ALPHA,
                       prompt_len=B.PROMPT_LEN, gen_len=int(sys.argv[1]) if len(sys.argv) > 1 else 256,
                       max_context=B.MAX_CTX, target_seed=1, draft_seed=2,
                       microbatch=int(os.environ.get("DEPTH", "4")),
                       tree_cap=int(os.environ.get("DEPTH", "4")))
eng = Engine(cfg)
eng.run(prompt_seed=1234)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
r = eng.run(prompt_seed=1234)
pr.disable()
print("tok/s", round(r.metrics.generation_speed, 1), "host profile", r.host_profile)
st = pstats.Stats(pr)
st.sort_stats(os.environ.get("SORT", "tottime")).print_stats(int(os.environ.get("TOP", "25")))
