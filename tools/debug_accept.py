import torch
import paper_2407_11798_b200 as sp
from paper_2407_11798_b200.engine import Engine, ExperimentConfig, truth_table

cfg = ExperimentConfig(mode="async-speculative", nodes=2, target_shape="llama2-7b",
                       draft_shape="llama-160m", draft_backend="synthetic", alpha=0.66,
                       prompt_len=128, gen_len=64, max_context=1024, target_seed=1,
                       draft_seed=2)
eng = Engine(cfg)
prompt = sp.sample_prompt(1234, 128, 32000)
truth, runner = truth_table(eng.target, prompt, 80)
for mode in ("iterative", "async-speculative", "sync-speculative"):
    r = eng.run(prompt=prompt, mode=mode, prompt_seed=1234)
    m = r.metrics
    gen = r.tokens
    mism = [i for i, (a, b) in enumerate(zip(gen, truth[128:])) if a != b]
    print(mode, "speed", round(m.generation_speed, 1), "acc", round(m.acceptance_rate, 3),
          "ex", m.examined, "ma", m.matched, "spec", m.spec_runs, "runs", m.runs_started,
          "cinv", m.cancelled_invalid, "csup", m.cancelled_superfluous,
          "first mismatch vs truth", mism[:5])
    if mode == "async-speculative":
        for rec in r.records[:30]:
            print("  ", rec.run_id, rec.kind, rec.min_pos, rec.tokens, rec.status, rec.seq_id)
