"""Summarise tools/bench_sweep.sh output: one row per variant."""
import json
import sys


def _pol(e):
    h = e.get("head_policy")
    if h is None:
        return f"{e.get('fold_frontier')}/{e.get('max_inflight')}"
    return (f"{'A' if h.get('adaptive') else ''}{h.get('fold_frontier')}/{h.get('max_inflight')}"
            f" folded {h.get('folded_runs')}")

for line in open(sys.argv[1]):
    d = json.loads(line)
    if "error" in d:
        print(f"{d['variant']:45s} ERROR {d['error'][-200:]}")
        continue
    x = d["line"]
    print(f"{d['variant']:45s} stages {x['config']['pipeline_stages']} async {x['value']:7.1f} "
          f"sync {x['sync_speculative_tokens_per_s']:7.1f} iter {x['pipeline_iterative_tokens_per_s']:7.1f} "
          f"a/s {x['async_over_sync']:.3f} e2e {x['e2e']['value']:7.1f} runs {x['runs_per_step']:6.1f} "
          f"canc {x['cancelled_runs_per_step']:6.1f} pol {_pol(x['config']['engine'])} "
          f"w{x['config']['engine'].get('tree_width')}"
          f" d{x['config']['engine'].get('microbatch')}")
