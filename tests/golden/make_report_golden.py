"""Golden report from the reference itself (run in the build container):

    PYTHONPATH=oracle/_ref python tests/golden/make_report_golden.py

Writes tests/golden/reference_report.json (the reference's ``export(...,
"json")`` of a 2-repetition virtual-clock experiment), its ``checksum()``,
its CSV export, and a config file + the config dict the reference builds
from it -- the fixtures for tests/test_report_cpu.py (report schema,
checksum recipe, CSV columns, config-file parsing)."""
import json
import os

from specpipe import bench
from specpipe.engine import ExperimentConfig

HERE = os.path.dirname(os.path.abspath(__file__))
cfg = ExperimentConfig(mode="async-speculative", nodes=4, vocab_size=64, embed_dim=32,
                       target_layers=4, draft_layers=1, draft_embed_dim=32, max_context=128,
                       prompt_len=12, gen_len=16, clock="virtual", draft_backend="synthetic",
                       alpha=0.7, repetitions=2, node_weights=(1.0, 2.0, 1.0))
rep = bench.run_experiment(cfg)
path = os.path.join(HERE, "reference_report.json")
bench.export(rep, "json", path)
bench.export(rep, "csv", os.path.join(HERE, "reference_report.csv"))
conf_text = ("# a config file\nmode = sync-speculative\nnodes = 3   # trailing comment\n"
             "vocab-size = 64\nembed_dim=32\ntarget_layers = 4\ncontinuous = off\n"
             "alpha = 0.5\nnode_weights = 1,2\neos_token = none\nprompt_len = 8\n"
             "gen_len = 8\nmax_context = 64\n")
with open(os.path.join(HERE, "reference_config.txt"), "w") as f:
    f.write(conf_text)
fv = bench.parse_config_file(os.path.join(HERE, "reference_config.txt"))
built = bench.config_to_dict(bench.config_from_sources(fv, {"gen_len": 10}))
with open(os.path.join(HERE, "reference_report_meta.json"), "w") as f:
    json.dump({"checksum": rep.checksum(), "parsed_config_file": fv,
               "config_from_sources": built,
               "compare_self": bench.compare_outputs([rep, rep]).detail}, f, indent=1,
              sort_keys=True)
print("wrote", path, rep.checksum())
