"""The metrics / report contract (reference bench.py:27-300,
cli.py:128-145) against fixtures the reference itself wrote
(tests/golden/make_report_golden.py): a reference report loads here with
the same checksum, re-exports byte-compatible JSON and CSV, config files
parse to the same config, and compare's verdicts / exit codes match."""

import csv
import json
import os

import pytest

from paper_2407_11798_b200 import report as R
from paper_2407_11798_b200.engine import ExperimentConfig, RunMetrics

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "reference_report_meta.json")) as f:
        return json.load(f)


def test_reference_report_roundtrip(meta, tmp_path):
    rep = R.load_report(os.path.join(GOLD, "reference_report.json"))
    assert rep.checksum() == meta["checksum"]          # same schema, same recipe
    with open(os.path.join(GOLD, "reference_report.json")) as f:
        want = json.load(f)
    assert rep.to_dict() == want
    out = tmp_path / "r.json"
    R.export(rep, "json", str(out))
    assert json.loads(out.read_text()) == want
    assert R.load_report(str(out)).checksum() == meta["checksum"]


def test_csv_matches_reference(tmp_path):
    rep = R.load_report(os.path.join(GOLD, "reference_report.json"))
    out = tmp_path / "r.csv"
    R.export(rep, "csv", str(out))
    with open(os.path.join(GOLD, "reference_report.csv")) as f:
        want = list(csv.reader(f))
    got = list(csv.reader(open(out)))
    assert got[0] == want[0] == ["rep", "mode", *R.METRIC_FIELDS, "token_checksum"]
    assert got == want


def test_config_file_and_overrides(meta):
    fv = R.parse_config_file(os.path.join(GOLD, "reference_config.txt"))
    assert fv == meta["parsed_config_file"]
    cfg = R.config_from_sources(fv, {"gen_len": 10, "alpha": None})
    got = R.config_to_dict(cfg)
    want = dict(meta["config_from_sources"])
    # the one default that differs: the GPU has a wall clock only
    assert (got.pop("clock"), want.pop("clock")) == ("wall", "virtual")
    assert got == want
    assert cfg.node_weights == (1.0, 2.0) and cfg.continuous is False and cfg.eos_token is None
    # B200 fields ride along only when set
    cfg2 = R.config_from_sources(fv, {"tree_width": "2", "fold_frontier": "off",
                                      "max_inflight": "none"})
    d = R.config_to_dict(cfg2)
    assert d["tree_width"] == 2 and d["fold_frontier"] is False and "max_inflight" not in d
    with pytest.raises(R.BenchError):
        R.config_from_sources({"no_such_key": "1"})
    with pytest.raises(R.BenchError):
        R.config_from_sources({"continuous": "maybe"})


def test_compare_verdicts_and_exit_codes(meta):
    rep = R.load_report(os.path.join(GOLD, "reference_report.json"))
    ok = R.compare_outputs([rep, rep])
    assert ok.ok and ok.detail == meta["compare_self"]
    assert R.compare_exit_code([rep]) [0] == 2
    assert R.compare_exit_code([rep, rep])[0] == 0
    bad = R.Report(rep.config, rep.runs, [list(t) for t in rep.tokens], rep.mean)
    bad.tokens[1][5] ^= 1
    v = R.compare_outputs([rep, bad])
    assert not v.ok and v.first_diff == (1, 5)
    assert R.compare_exit_code([rep, bad])[0] == 1
    other = R.Report(R.config_from_sources(overrides={**R.config_to_dict(rep.config),
                                                      "gen_len": 15}),
                     rep.runs, rep.tokens, rep.mean)
    with pytest.raises(R.BenchError):
        R.compare_outputs([rep, other])


def test_consistency_gap():
    m = RunMetrics(mode="async-speculative", clock="wall", tokens_generated=11, duration=1.0,
                   generation_speed=10.0, ttft=0.1, itl=0.1, acceptance_rate=0.5, examined=4,
                   matched=2, runs_started=5, spec_runs=3, cancelled_invalid=0,
                   cancelled_superfluous=0, cancelled_runs=0, drained_runs=0, alloc_stalls=0,
                   inflight_mean=1.0, bytes_by_tag={}, msgs_by_tag={}, token_checksum="x",
                   virtual_end=0.0, wall_seconds=1.0)
    assert R.consistency_gap(m) < 1e-9
