"""Experiment reports: the reference's metrics / report contract
(``specpipe/bench.py:27-300``, ``cli.py:128-145``) over B200 runs.

* ``METRIC_FIELDS`` -- the per-repetition columns, in the reference's order
  (``bench.py:27-45``);
* ``parse_config_file`` / ``config_from_sources`` / ``config_to_dict`` --
  flat ``key = value`` files with CLI-style overrides (``bench.py:52-125``);
* ``Report`` (``to_dict``, ``checksum``) and ``run_experiment`` --
  repetitions shift the prompt seed by their index (``bench.py:128-172``);
* ``compare_outputs`` / ``compare_exit_code`` -- byte-exact token
  comparison across reports and the ``compare`` command's exit codes 0 / 1 /
  2 (``bench.py:175-208``, ``cli.py:128-145``);
* ``export`` / ``load_report`` / ``sweep`` / ``sweep_to_csv`` /
  ``consistency_gap`` (``bench.py:211-300``).

A report's ``config`` carries the reference's fields plus the B200 ones that
differ from their defaults, so a report of a reference-shaped experiment has
exactly the reference's schema (and checksum recipe: sha256 over the sorted
JSON without wall-clock fields).  Timing metrics are wall clock here, so the
token checksum -- not the report checksum -- is the cross-implementation
parity artifact.
"""

from __future__ import annotations

import csv
import dataclasses
import hashlib
import json
from dataclasses import dataclass, fields, replace
from typing import Dict, List, Optional, Sequence, Tuple

from .engine import ExperimentConfig, RunMetrics, simulate

METRIC_FIELDS = ("tokens_generated", "duration", "generation_speed", "ttft", "itl",
                 "acceptance_rate", "examined", "matched", "runs_started", "spec_runs",
                 "cancelled_invalid", "cancelled_superfluous", "cancelled_runs",
                 "drained_runs", "alloc_stalls", "inflight_mean")

# ExperimentConfig fields the reference does not have (engine.py:80-183)
B200_FIELDS = ("arch", "target_shape", "draft_shape", "capacity", "max_run_tokens",
               "draft_charge", "draft_tc", "draft_sm_reserve", "spec_ramp", "fold_frontier",
               "max_inflight", "tree_width", "alpha_sibling", "draft_exclusive")


class BenchError(RuntimeError):
    """Bad report input (reference bench.BenchError)."""


def parse_config_file(path: str) -> Dict[str, str]:
    """``key = value`` per line, ``#`` comments, dashes in keys as underscores."""
    values: Dict[str, str] = {}
    with open(path) as fh:
        for n, line in enumerate(fh, 1):
            body = line.partition("#")[0].strip()
            if not body:
                continue
            key, sep, val = body.partition("=")
            if not sep:
                raise BenchError(f"{path}:{n}: expected 'key = value'")
            values[key.strip().replace("-", "_")] = val.strip()
    return values


def _parse_bool(name: str, text: str) -> bool:
    t = text.strip().lower()
    if t in ("1", "true", "yes", "on"):
        return True
    if t in ("0", "false", "no", "off"):
        return False
    raise BenchError(f"{name}: cannot parse boolean from {text!r}")


def _convert(name: str, value, default):
    """String values take the type of the field's default (reference _coerce);
    optional fields keep None for '' / 'none'."""
    if not isinstance(value, str):
        return tuple(value) if isinstance(value, list) else value
    if name == "node_weights":
        v = value.strip()
        return tuple(float(x) for x in v.split(",")) if v else None
    if name in ("eos_token", "fold_frontier", "max_inflight", "target_shape", "draft_shape"):
        if value.strip().lower() in ("", "none"):
            return None
        if name == "fold_frontier":
            return _parse_bool(name, value)
        if name in ("eos_token", "max_inflight"):
            return int(value)
        return value
    if isinstance(default, bool):
        return _parse_bool(name, value)
    if isinstance(default, int):
        return int(value)
    if isinstance(default, float):
        return float(value)
    return value


def config_from_sources(file_values: Optional[Dict[str, str]] = None,
                        overrides: Optional[Dict[str, object]] = None) -> ExperimentConfig:
    """File values, then overrides on top (None = not given); validated."""
    known = {f.name: f for f in fields(ExperimentConfig)}
    base = ExperimentConfig()
    kw: Dict[str, object] = {}
    for src in (file_values or {}, overrides or {}):
        for raw_key, value in src.items():
            if value is None:
                continue
            key = raw_key.replace("-", "_")
            if key not in known:
                raise BenchError(f"unknown config key {key!r}")
            kw[key] = _convert(key, value, getattr(base, key))
    cfg = ExperimentConfig(**kw)
    cfg.validate()
    return cfg


def config_to_dict(cfg: ExperimentConfig) -> dict:
    """The reference's fields, plus B200 fields that differ from defaults."""
    base = ExperimentConfig()
    out = {}
    for f in fields(cfg):
        v = getattr(cfg, f.name)
        if f.name in B200_FIELDS and v == getattr(base, f.name):
            continue
        out[f.name] = list(v) if isinstance(v, tuple) else v
    return out


@dataclass
class Report:
    """One configuration, its repetitions' metrics and tokens, a mean row."""

    config: ExperimentConfig
    runs: List[RunMetrics]
    tokens: List[List[int]]
    mean: Dict[str, float]

    def to_dict(self, include_wall: bool = True) -> dict:
        return {"config": config_to_dict(self.config), "repetitions": len(self.runs),
                "runs": [r.to_dict(include_wall=include_wall) for r in self.runs],
                "mean": dict(self.mean), "tokens": [list(t) for t in self.tokens]}

    def checksum(self) -> str:
        text = json.dumps(self.to_dict(include_wall=False), sort_keys=True)
        return hashlib.sha256(text.encode()).hexdigest()


def _mean(runs: Sequence[RunMetrics]) -> Dict[str, float]:
    return {k: sum(getattr(r, k) for r in runs) / len(runs) for k in METRIC_FIELDS}


def run_experiment(cfg: ExperimentConfig) -> Report:
    """``cfg.repetitions`` runs on the GPU; repetition i uses prompt seed
    ``cfg.prompt_seed + i`` (models stay resident across repetitions)."""
    cfg.validate()
    metrics, toks = [], []
    for i in range(cfg.repetitions):
        res = simulate(replace(cfg, prompt_seed=cfg.prompt_seed + i))
        metrics.append(res.metrics)
        toks.append(list(res.tokens))
    return Report(cfg, metrics, toks, _mean(metrics))


@dataclass(frozen=True)
class CompareResult:
    ok: bool
    detail: str
    first_diff: Optional[Tuple[int, int]] = None   # (repetition, token index)


_SAME_EXPERIMENT = ("vocab_size", "embed_dim", "target_layers", "n_heads", "target_seed",
                    "prompt_seed", "prompt_len", "gen_len")


def compare_outputs(reports: Sequence[Report]) -> CompareResult:
    """Every report's tokens must equal the first's, repetition by
    repetition; the reports must describe the same experiment."""
    if len(reports) < 2:
        raise BenchError("need at least two reports to compare")
    first = reports[0]
    for rep in reports[1:]:
        for key in _SAME_EXPERIMENT:
            a, b = getattr(first.config, key), getattr(rep.config, key)
            if a != b:
                raise BenchError(f"mismatched configs: {key} differs ({a!r} vs {b!r})")
        if len(rep.tokens) != len(first.tokens):
            return CompareResult(False, "repetition counts differ")
        for i, (x, y) in enumerate(zip(first.tokens, rep.tokens)):
            if x != y:
                at = next((j for j, (u, v) in enumerate(zip(x, y)) if u != v),
                          min(len(x), len(y)))
                return CompareResult(False, f"outputs diverge: mode {rep.config.mode!r} "
                                            f"differs from {first.config.mode!r} at "
                                            f"repetition {i}, token {at}", (i, at))
    return CompareResult(True, f"{len(reports)} reports byte-identical")


def compare_exit_code(reports: Sequence[Report]) -> Tuple[int, str]:
    """The ``compare`` command's contract (cli.py:128-145): 2 when fewer
    than two reports are given, 1 when outputs diverge, 0 when identical."""
    if len(reports) < 2:
        return 2, "compare: need at least two reports (files and/or --modes)"
    verdict = compare_outputs(reports)
    return (0 if verdict.ok else 1), verdict.detail


def _csv_rows(report: Report, lead: tuple = ()):
    for i, r in enumerate(report.runs):
        yield list(lead) + [i, r.mode] + [getattr(r, k) for k in METRIC_FIELDS] + [r.token_checksum]
    yield list(lead) + ["mean", report.config.mode] + [report.mean[k] for k in METRIC_FIELDS] + [""]


def export(report: Report, fmt: str, path: str) -> None:
    """``json``: the whole report; ``csv``: one row per repetition + mean."""
    if fmt == "json":
        with open(path, "w") as fh:
            json.dump(report.to_dict(), fh, indent=2, sort_keys=True)
            fh.write("\n")
        return
    if fmt == "csv":
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(("rep", "mode") + METRIC_FIELDS + ("token_checksum",))
            w.writerows(_csv_rows(report))
        return
    raise BenchError(f"unknown export format {fmt!r}")


def load_report(path: str) -> Report:
    """A report written by ``export(..., "json")`` -- here or by the reference."""
    with open(path) as fh:
        data = json.load(fh)
    cfg = config_from_sources(overrides=dict(data["config"]))
    known = {f.name for f in fields(RunMetrics)}
    runs = []
    for r in data["runs"]:
        kw = {k: v for k, v in r.items() if k in known}
        kw.setdefault("wall_seconds", 0.0)
        kw["bytes_by_tag"] = dict(kw["bytes_by_tag"])
        kw["msgs_by_tag"] = dict(kw["msgs_by_tag"])
        runs.append(RunMetrics(**kw))
    return Report(cfg, runs, [list(t) for t in data["tokens"]], dict(data["mean"]))


def sweep(base: ExperimentConfig, param: str, values: Sequence) -> List[Report]:
    """One report per value of one config field."""
    if param not in {f.name for f in fields(ExperimentConfig)}:
        raise BenchError(f"unknown sweep parameter {param!r}")
    out = []
    for v in values:
        if param != "mode":
            v = _convert(param, v, getattr(base, param))
        out.append(run_experiment(replace(base, **{param: v})))
    return out


def sweep_to_csv(reports: Sequence[Report], param: str, path: str) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow((param, "rep", "mode") + METRIC_FIELDS + ("token_checksum",))
        for rep in reports:
            w.writerows(_csv_rows(rep, (getattr(rep.config, param),)))


def consistency_gap(m: RunMetrics) -> float:
    """|k / (ttft + itl*(k-1)) - speed| / speed with k = tokens_generated - 1:
    the speed and the TTFT/ITL bookkeeping must agree (reference: <= 1%)."""
    k = max(m.tokens_generated - 1, 0)
    if k == 0 or m.duration <= 0:
        return 0.0
    rebuilt = k / (m.ttft + m.itl * max(k - 1, 0))
    return abs(rebuilt - m.generation_speed) / m.generation_speed
