"""torchrun entry for the multi-GPU parity test (tests/test_gpu_multi.py).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/dist_parity_main.py OUT.json

Runs the NCCL pipeline (dist.py) in both layouts -- shared (every rank a
stage, the draft on rank 0's GPU) and dedicated (rank 0 = head + draft,
stages on ranks 1..N-1, engine.py:171-176) -- and, in each, the async,
sync and pipeline-iterative modes on:

* the reference's toy decoder (``ref`` arch, fp32): streams must equal the
  float64 oracle's greedy stream (oracle/model.py, pinned to the reference);
* a small llama config (bf16, RoPE, SwiGLU, tiled tcgen05 weights):
  streams must equal the 1-GPU greedy stream of the same weights
  (SerialDecoder), since every kernel is batch- and split-invariant.

Rank 0 writes {case: {mode: tokens}} plus the references to OUT.json.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GEN = 40
PROMPT = 16


def _cases():
    from paper_2407_11798_b200.engine import ExperimentConfig
    ref = ExperimentConfig(mode="async-speculative", vocab_size=256, embed_dim=64,
                           target_layers=8, n_heads=2, draft_layers=1, max_context=256,
                           prompt_len=PROMPT, gen_len=GEN, target_seed=3, draft_seed=4,
                           draft_backend="synthetic", alpha=0.6, capacity=2048,
                           partitions=16)
    llama = ExperimentConfig(mode="async-speculative", arch="llama", vocab_size=512,
                             embed_dim=256, target_layers=8, n_heads=4, draft_layers=1,
                             draft_embed_dim=256, max_context=256, prompt_len=PROMPT,
                             gen_len=GEN, target_seed=5, draft_seed=6,
                             draft_backend="synthetic", alpha=0.6, capacity=2048,
                             partitions=16)
    return {"ref": ref, "llama": llama}


def main(out_path):
    from dataclasses import replace

    import torch
    import torch.distributed as dist

    from paper_2407_11798_b200 import dist as D
    from paper_2407_11798_b200.engine import Engine
    from paper_2407_11798_b200.model import SerialDecoder, build_model, sample_prompt

    rank, world, local, plane, gloo = D.init()
    dev = torch.device("cuda", local)
    results, refs = {}, {}
    for name, base in _cases().items():
        prompt = sample_prompt(11, PROMPT, base.vocab_size)
        if rank == 0:
            if name == "ref":
                from oracle import model as OM
                tc = base.target_config()
                om = OM.build_ref_model(OM.OracleConfig(tc.vocab_size, tc.embed_dim,
                                                        tc.n_layers, tc.n_heads,
                                                        tc.max_context, tc.seed))
                refs[name] = OM.OracleDecoder(om).greedy_decode(prompt, GEN)
            else:
                full = build_model(base.target_config(), dev)
                dec = SerialDecoder(full)
                tip = dec.feed(prompt)
                toks = []
                for _ in range(GEN):
                    toks.append(tip.argmax)
                    tip = dec.feed([tip.argmax])
                refs[name] = toks
                del dec, full
                torch.cuda.empty_cache()
        for layout in ("shared", "dedicated"):
            first = 1 if layout == "dedicated" else 0
            cfg = replace(base, nodes=world if first else world + 1)
            model, ranges = D.build_slice(cfg, rank, world, None, first)
            if rank != 0:
                lo, hi = ranges[rank - first]
                D.worker_loop(model, lo, hi, rank, world, plane, cfg.partitions,
                              cfg.capacity, cfg.max_run_tokens, first=first)
            else:
                draft = build_model(cfg.draft_config(), dev)
                pipe = D.DistPipeline(model, ranges, plane, world, cfg.partitions,
                                      cfg.capacity, cfg.max_run_tokens,
                                      local_stage=not first)
                eng = Engine(cfg, target_model=model, draft_model=draft, pipeline=pipe)
                got = {}
                for mode in ("async-speculative", "sync-speculative", "pipeline-iterative"):
                    r = eng.run(prompt=list(prompt), mode=mode)
                    got[mode] = r.tokens
                    got[mode + ":cancelled"] = r.metrics.cancelled_runs
                # tree speculation (runner-up siblings on their own partitions)
                eng.cfg = replace(cfg, tree_width=2, alpha_sibling=0.6)
                for mode in ("async-speculative", "sync-speculative"):
                    got[mode + ":tree"] = eng.run(prompt=list(prompt), mode=mode).tokens
                eng.cfg = cfg
                results[f"{name}/{layout}"] = got
                pipe.shutdown()
                del eng, pipe, draft
            del model
            torch.cuda.synchronize()
            dist.barrier(group=gloo)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"world": world, "results": results, "refs": refs}, f)
    dist.barrier(group=gloo)
    plane.close(unlink=(rank == 0))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
