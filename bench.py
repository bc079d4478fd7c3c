#!/usr/bin/env python
"""Benchmark: single-request generated tokens/s + ITL of PipeInfer on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One *step* = one complete single-request generation (prefill of a 128-token
synthetic prompt, then ``gen_len`` accepted tokens) of the Llama-2-7B-shape
target (bf16, random init) with a 160M-shape draft, i.e. BASELINE.json
configs[1], in PipeInfer's async-speculative mode over an N-stage pipeline
(one stage per GPU; N=1 is the single-GPU pipeline).  ``value`` is the
reference's generation speed (engine.py:1234-1243: accepted tokens after
prefill / time from end of prefill to the last acceptance), aggregated over
the K timed steps; ``itl_ms`` the mean inter-token latency.

``--impl reference`` times the reference's CPU implementation on this host's
cores: the reference package itself when oracle/vendor_ref.sh has vendored
it into oracle/_ref (its decoder at the target's width, 2 layers
extrapolated to the target's depth + head; plus cfg1 reference_decode and
the four modes under simulate(clock="wall")), else the float64 oracle port.
"""

from __future__ import annotations

from typing import Optional
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TARGET, DRAFT = "llama2-7b", "llama-160m"
ALPHA = 0.66          # paper's observed acceptance for a 7B pair
# BASELINE.json configs by (target, draft) shape
WORKLOADS = {("llama2-7b", "llama-160m"): "configs[1]: Llama-2-7B-shape target + 160M-shape draft",
             ("llama2-13b", "tinyllama-1.1b"): "configs[2]: Llama-2-13B-shape target + "
                                               "TinyLlama-1.1B-shape draft",
             ("llama2-70b", "tinyllama-1.1b"): "configs[3]: Llama-2-70B-shape target + "
                                               "1.1B-shape draft"}
PROMPT_LEN, GEN_LEN, MAX_CTX = 128, 512, 1024


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.path = f"/tmp/clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (float64 oracle) on host cores
# ---------------------------------------------------------------------------

def cpu_baseline(n_decode: int = 3, layers: int = 2, prompt_len: int = 16,
                 shape: str = TARGET) -> dict:
    """The oracle's fp64 forward timed with every host thread BLAS can use
    (torchrun exports OMP_NUM_THREADS=1; the reference arm must not inherit it)."""
    import numpy  # noqa: F401  (load BLAS first: threadpoolctl only sees loaded libraries)
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=os.cpu_count() or 1):
            return _cpu_baseline(n_decode, layers, prompt_len, shape)
    except ImportError:
        return _cpu_baseline(n_decode, layers, prompt_len, shape)


def _cpu_baseline(n_decode: int, layers: int, prompt_len: int, shape: str = TARGET) -> dict:
    import numpy as np
    from oracle import model as OM
    from oracle.kvcache import OracleCache
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count() or 1
    from paper_2407_11798_b200.model import LLAMA_SHAPES
    sh = LLAMA_SHAPES[shape]
    d, f, V, H = sh["embed_dim"], sh["ffn_dim"], sh["vocab_size"], sh["n_heads"]
    KH, NL = sh["n_kv_heads"], sh["n_layers"]
    kvd = d // H * KH
    if d >= 8192:          # 70B width: one fp64 layer is ~6 GB of host memory
        layers = 1
    r = np.random.Generator(np.random.PCG64(0))
    cfg = OM.OracleConfig(vocab_size=V, embed_dim=d, n_layers=layers, n_heads=H,
                          max_context=1024, arch="llama", ffn_dim=f, n_kv_heads=KH)
    lw = []
    sd, sf = d ** -0.5, f ** -0.5
    for _ in range(layers):
        lw.append(dict(wq=r.standard_normal((d, d)) * sd, wk=r.standard_normal((d, kvd)) * sd,
                       wv=r.standard_normal((d, kvd)) * sd, wo=r.standard_normal((d, d)) * sd,
                       wg=r.standard_normal((d, f)) * sd, wu=r.standard_normal((d, f)) * sd,
                       wd=r.standard_normal((f, d)) * sf, attn_norm=np.ones(d),
                       mlp_norm=np.ones(d)))
    emb = r.standard_normal((V, d))
    w_out = r.standard_normal((d, V)) / 64
    m = OM.OracleModel(cfg, emb, None, lw, w_out, np.ones(d))
    cache = OracleCache(d, range(layers), 1024, 1)
    prompt = [int(t) for t in r.integers(0, V, prompt_len)]
    OM.eval_layers(m, 0, layers, None,
                   [(t, i, frozenset([0]), False) for i, t in enumerate(prompt)], cache)
    t_layers = []
    for i in range(n_decode):
        tok = [(int(r.integers(0, V)), prompt_len + i, frozenset([0]), True)]
        t0 = time.perf_counter()
        x = OM.eval_layers(m, 0, layers, None, tok, cache)
        t_layers.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    OM.logits(m, x, tok)
    t_head = time.perf_counter() - t0
    per_layer = statistics.median(t_layers) / layers
    per_token = per_layer * NL + t_head
    return {"value": 1.0 / per_token, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": (f"oracle fp64 llama forward, {layers} layers at {shape} width "
                       f"(d={d}, ffn={f}, kv heads {KH}/{H}), {n_decode} decode tokens after a "
                       f"{prompt_len}-token prompt, + LM head V={V}; per-token time "
                       f"extrapolated to {NL} layers ({per_layer*1e3:.1f} ms/layer, "
                       f"head {t_head*1e3:.1f} ms)"),
            "ms_per_token": per_token * 1e3}


# ---------------------------------------------------------------------------
# roofline: the dominant kernel (weight-streaming GEMV) timed with CUDA events
# ---------------------------------------------------------------------------

def gemv_roofline(engine, reps: int = 5) -> dict:
    """Roofline of the dominant kernel: the weight-streaming GEMM of every
    decoder layer of this rank's stage (QKV, O, gate/up, down; tcgen05 path
    for bf16 weights), one decode token (M=1), each launch timed with CUDA
    events on the stage stream after capture into a CUDA graph (so host
    launch gaps are excluded).  Algorithmic bytes per launch = the weight
    matrix + its activation row in and out; weights (>= 8 GB per stage) are
    far larger than the 126 MB L2."""
    import ctypes as C
    import torch
    from paper_2407_11798_b200 import _lib
    from paper_2407_11798_b200 import _lib as L_
    stages = getattr(engine.pipe, "stages", [])
    if stages:      # this rank's stage layers
        st = stages[0]
        cfg, lib, dev, layers = st.cfg, st.lib, st.device, range(st.lo, st.hi)
    else:           # head + dedicated draft rank: the one-layer target shell
        cfg, lib, dev = engine.target.config, L_.load(), engine.device
        layers = sorted(engine.target.layers)
    d, f = cfg.embed_dim, cfg.hidden
    q, kv = cfg.n_heads * cfg.head_dim, cfg.kv_dim
    X = torch.zeros((256, max(d, f)), device=dev, dtype=torch.bfloat16).normal_()
    out = torch.zeros((256, 2 * f + q + 2 * kv), device=dev, dtype=torch.float32)
    scratch = torch.zeros(8 << 20, device=dev)
    tick = torch.zeros(4096, dtype=torch.int32, device=dev)
    args, nbytes, kinds = [], 0, []
    for l in layers:
        L = engine.target.layers[l]
        for key, n, k in (("qkv", q + 2 * kv, d), ("o", d, q), ("up", 2 * f, d),
                          ("down", d, f)):
            a = _lib.sp_tc_args()
            a.w, a.n_rows, a.k, a.m, a.epi = L[key].data_ptr(), n, k, 1, _lib.SP_EPI_STORE
            a.out, a.ldo = out.data_ptr(), out.shape[1]
            a.scratch, a.tickets = scratch.data_ptr(), tick.data_ptr()
            args.append(a)
            kinds.append((key, n * k * 2 + 2 * k + 4 * n))
            nbytes += n * k * 2 + 2 * k + 4 * n
    s = torch.cuda.Stream(dev)
    graph = torch.cuda.CUDAGraph()
    for a in args:   # warm (first launches configure smem attributes)
        _lib.check(lib.sp_tc_gemm(C.byref(a), X.data_ptr(), 256, s.cuda_stream))
    s.synchronize()
    with torch.cuda.graph(graph, stream=s):
        for a in args:
            _lib.check(lib.sp_tc_gemm(C.byref(a), X.data_ptr(), 256, s.cuda_stream))
    times = []
    for rep in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):     # replay() launches on the current stream
            e0.record(s)
            graph.replay()
            e1.record(s)
        e1.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.median(times)
    peak, how = _peaks()
    achieved = nbytes / t / 1e9
    # per matrix kind: the same launches, one kind per graph
    per = {}
    for kind in ("qkv", "o", "up", "down"):
        sel = [a for a, (k_, _) in zip(args, kinds) if k_ == kind]
        byt = sum(b for k_, b in kinds if k_ == kind)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s):
            for a in sel:
                _lib.check(lib.sp_tc_gemm(C.byref(a), X.data_ptr(), 256, s.cuda_stream))
        ts = []
        for rep in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                g2.replay()
                e1.record(s)
            e1.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1) / 1e3)
        tk = statistics.median(ts)
        per[kind] = {"us_per_launch": round(tk / len(sel) * 1e6, 2),
                     "achieved": round(byt / tk / 1e9, 1), "frac": round(byt / tk / 1e9 / peak, 4)}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("bytes_per_launch")
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": "static: ncu --set full capture of the same GEMM replay, "
                              "profiles/ncu_gemm_traffic.json (dram read+write per launch)",
            "per_matrix": per,
            "kernel": "tc_gemm_kernel<NT=16> (tcgen05+TMEM, bulk-copied tiled bf16 "
                      "weights; QKV+O+gate/up+down of every layer of the stage, M=1)",
            "algorithmic_bytes_per_launch": round(nbytes / len(args)),
            "avg_launch_us": round(t / len(args) * 1e6, 2), "launches": len(args),
            "peak_source": how}


def stage_run_roofline(eng, peak: float, runs: int = 24) -> Optional[dict]:
    """In-context roofline of the product path: back-to-back 1-token decode
    stage-runs through the engine's own pipeline (graph-replayed
    sp_stage_step: fused QKV/RoPE, attention, residual and SwiGLU epilogues,
    fused LM head), timed with CUDA events on the stage stream after a
    128-token prefill.  Algorithmic bytes per run = every weight byte of the
    stage (+ LM head) + the K/V rows read; achieved = bytes / run time."""
    import torch
    import paper_2407_11798_b200 as sp
    from paper_2407_11798_b200.model import BatchToken, encode_tokens
    pipe = eng.pipe
    if not hasattr(pipe, "stream") or not getattr(pipe, "stages", None):
        return None            # (the distributed pipeline: workers hold the stages)
    cfg = eng.target.config
    pipe.reset()
    prompt = sp.sample_prompt(7, PROMPT_LEN, cfg.vocab_size)
    pre = [BatchToken(t, i, frozenset([0]), i == PROMPT_LEN - 1) for i, t in enumerate(prompt)]
    pipe.launch(1, sp.model.KIND_CODE[sp.PREFILL], encode_tokens(pre), 0, [PROMPT_LEN - 1])
    pipe.wait()

    def decode(rid, pos):
        b = [BatchToken(int(prompt[pos % PROMPT_LEN]), pos, frozenset([0]), True)]
        pipe.launch(rid, sp.model.KIND_CODE[sp.NON_SPECULATIVE], encode_tokens(b), 0, [0])
    for i in range(4):         # capture / warm the 1-token graph
        decode(2 + i, PROMPT_LEN + i)
        pipe.wait()
    st = pipe.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    base = PROMPT_LEN + 4
    for i in range(runs):
        decode(100 + i, base + i)
    e1.record(st)
    for _ in range(runs):
        pipe.wait()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / runs
    pipe.reset()
    layers = sum(st_.hi - st_.lo for st_ in pipe.stages)
    head = any(st_.hi == cfg.n_layers for st_ in pipe.stages)
    wb = cfg.weight_bytes(layers=layers, head=head)
    ctx = base + runs // 2
    kvb = layers * ctx * cfg.kv_dim * 2 * (4 if cfg.weight_dtype == "fp32" else 2)
    ach = (wb + kvb) / t / 1e9
    return {"ms_per_run": round(t * 1e3, 4), "layers": layers, "lm_head": head,
            "algorithmic_bytes_per_run": wb + kvb, "achieved": round(ach, 1),
            "frac": round(ach / peak, 4),
            "note": "1-token decode stage-runs back to back through the product path "
                    f"(graph replay, context {base}..{base + runs}), CUDA events on the "
                    "stage stream"}


# ---------------------------------------------------------------------------

def bench_knobs(args) -> dict:
    """Engine knobs the run overrides (the reference's defaults otherwise)."""
    kw = {}
    for k in ("microbatch", "partitions", "cutoff"):
        v = getattr(args, k, None)
        if v is not None:
            kw[k] = v
    if getattr(args, "no_continuous", False):   # reference knob (engine.py:102)
        kw["continuous"] = False
    if getattr(args, "no_ramp", False):
        kw["spec_ramp"] = False
    if getattr(args, "free_draft", False):   # experiment only: draft proposals cost nothing
        kw["draft_charge"] = False
    if getattr(args, "reference_policy", False):   # the reference head, unchanged
        kw.update(fold_frontier=False, max_inflight=0, draft_exclusive=False)
    if getattr(args, "tree_width", None) is not None:
        kw["tree_width"] = args.tree_width
    if getattr(args, "alpha_sibling", None) is not None:
        kw["alpha_sibling"] = args.alpha_sibling
    if getattr(args, "depth", None) is not None:     # speculation depth per run
        kw["microbatch"] = kw["tree_cap"] = args.depth
    if getattr(args, "max_inflight", None) is not None:
        kw["max_inflight"] = args.max_inflight
    if getattr(args, "fold", None) is not None:
        kw["fold_frontier"] = args.fold == "on"
    return kw


def run_ours(args) -> dict:
    import torch
    from paper_2407_11798_b200.engine import Engine, ExperimentConfig

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        from paper_2407_11798_b200 import dist
        return dist.bench_main(args)
    torch.cuda.set_device(0)
    cfg = ExperimentConfig(mode="async-speculative", nodes=2, target_shape=args.target,
                           draft_shape=args.draft, draft_backend="synthetic", alpha=args.alpha,
                           prompt_len=PROMPT_LEN, gen_len=args.gen_len, max_context=MAX_CTX,
                           target_seed=1, draft_seed=2, capacity=8192,
                           **bench_knobs(args))
    return measure(Engine(cfg), args, n_gpus=1)


def measure(eng, args, n_gpus: int, pipe=None) -> dict:
    """The timed protocol, shared by the 1-GPU and torchrun paths (rank 0)."""
    import torch
    import paper_2407_11798_b200 as sp

    seeds = [1234 + i for i in range(args.warmup + args.steps)]
    for s in seeds:   # synthetic-draft truth tables: setup, outside the timed region
        eng._make_draft(sp.sample_prompt(s, PROMPT_LEN, 32000), s)
    for i in range(args.warmup):
        eng.run(prompt_seed=seeds[i])
    torch.cuda.synchronize()
    res = []
    launches0 = eng.launch_count()
    with Clocks(torch.cuda.current_device()) as clk:
        if pipe is not None:
            pipe.mark(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            res.append(eng.run(prompt_seed=seeds[args.warmup + i]))
        torch.cuda.synchronize()
        total_s = time.perf_counter() - t0
        if pipe is not None:
            pipe.mark(2)
    launches = eng.launch_count() - launches0
    gen_tok = sum(r.metrics.tokens_generated - 1 for r in res)
    gen_time = sum(r.metrics.duration for r in res)
    value = gen_tok / gen_time
    itl = statistics.mean(r.metrics.itl for r in res)
    # baselines on the same kernels and pipeline: sync-speculative (the >=2x
    # target's denominator) and plain pipeline-iterative decoding
    nb = args.steps     # the same prompts as the timed async steps
    sync = [eng.run(prompt_seed=seeds[args.warmup + i], mode="sync-speculative")
            for i in range(nb)]
    itr = [eng.run(prompt_seed=seeds[args.warmup + i], mode="pipeline-iterative")
           for i in range(nb)]

    def speed(rs):
        return sum(r.metrics.tokens_generated - 1 for r in rs) / sum(r.metrics.duration for r in rs)

    sync_speed, it_speed = speed(sync), speed(itr)

    # every timed stream (and the baselines') must be the target's greedy
    # stream: the truth table is an iterative decode through the same stages
    def check(r, seed):
        prompt = sp.sample_prompt(seed, PROMPT_LEN, 32000)
        truth = eng._tables[tuple(prompt)][0]
        want = truth[PROMPT_LEN:PROMPT_LEN + len(r.tokens)]
        if len(r.tokens) != args.gen_len or r.tokens != want:
            raise SystemExit(f"bench: {r.metrics.mode} stream for prompt seed {seed} differs "
                             "from the greedy (iterative) stream")
    for i, r in enumerate(res):
        check(r, seeds[args.warmup + i])
    for i in range(nb):
        check(sync[i], seeds[args.warmup + i])
        check(itr[i], seeds[args.warmup + i])
    checksum = res[0].metrics.token_checksum
    # e2e: the public API on host token lists (prompt H2D, results D2H inside)
    prompt = sp.sample_prompt(seeds[-1], PROMPT_LEN, 32000)
    eng._make_draft(prompt, 1234)
    t0 = time.perf_counter()
    out = eng.generate(prompt)
    e2e_s = time.perf_counter() - t0
    if out != eng._tables[tuple(prompt)][0][PROMPT_LEN:PROMPT_LEN + len(out)]:
        raise SystemExit("bench: generate() stream differs from the greedy stream")
    rf = gemv_roofline(eng)
    rf["stage_run"] = stage_run_roofline(eng, rf["peak"])
    # the CPU baseline is timed on rank 0 at N=1 only (the bench contract)
    cpu = None
    if not args.no_cpu and n_gpus == 1:
        from oracle import reference_arm as R
        cpu = (_reference_baseline(args.target, n_decode=2) if R.available()
               else cpu_baseline(shape=args.target))
    wb = eng.target.config.weight_bytes()
    return {
        "metric": "single-request generated tokens/s + inter-token latency",
        "value": round(value, 2), "unit": "tokens/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_s / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, PCG64 prompts)",
        "config": {"workload": WORKLOADS.get((args.target, args.draft),
                                             f"{args.target} target + {args.draft} draft")
                               + f", bf16, async-speculative (PipeInfer), "
                               f"{eng.pipe.n_stages}-stage pipeline"
                               + (", dedicated draft GPU" if eng.pipe.n_stages < n_gpus
                                  else ", draft shares GPU 0"),
                   "target": args.target, "draft": args.draft, "alpha": args.alpha,
                   "prompt_len": PROMPT_LEN, "gen_len": args.gen_len,
                   "pipeline_stages": eng.pipe.n_stages,
                   "engine": {"microbatch": eng.cfg.microbatch, "partitions": eng.cfg.partitions,
                              "cutoff": eng.cfg.cutoff, "draft_kernel":
                              os.environ.get("SP_DRAFT_KERNEL", "cluster")
                              if os.environ.get("SP_DRAFT_FUSED", "1") != "0" else "per-forward",
                              "spec_ramp": eng.cfg.spec_ramp,
                              "continuous": eng.cfg.continuous,
                              "head_policy": dict(eng.last_head_policy),
                              "draft_exclusive": eng.cfg.draft_exclusive,
                              "tree_width": eng.cfg.tree_width,
                              **({"alpha_sibling": eng.cfg.alpha_sibling}
                                 if eng.cfg.tree_width > 1 else {}),
                              **({"free_draft": True} if not eng.cfg.draft_charge else {})},
                   "l2": f"weights {wb / 1e9:.1f} GB >> 126 MB L2 (no flush needed)"},
        "itl_ms": round(itl * 1e3, 3),
        "streams_checked": {"timed_steps": len(res), "sync": nb, "iterative": nb, "e2e": 1,
                            "equal_to_greedy": True,
                            "token_checksum_step0": checksum},
        "acceptance_rate": round(statistics.mean(r.metrics.acceptance_rate for r in res), 4),
        "cancelled_runs_per_step": round(statistics.mean(r.metrics.cancelled_runs for r in res), 1),
        "runs_per_step": round(statistics.mean(r.metrics.runs_started for r in res), 1),
        "inflight_mean": round(statistics.mean(r.metrics.inflight_mean for r in res), 2),
        "head_host_s_per_step": {k: round(statistics.mean(r.host_profile.get(k, 0.0) for r in res), 4)
                                 for k in ("completion", "reply+spec_launch", "draft_request", "wait")},
        "sync_speculative_tokens_per_s": round(sync_speed, 2),
        "pipeline_iterative_tokens_per_s": round(it_speed, 2),
        "async_over_sync": round(value / sync_speed, 3),
        "weight_stream_roofline_tokens_per_s": round(rf["peak"] * 1e9 / wb, 1),
        "e2e": {"value": round((len(out) - 1) / e2e_s, 2), "unit": "tokens/s",
                "h2d_bytes_per_step": PROMPT_LEN * 16, "d2h_bytes_per_step": len(out) * 16,
                "note": "generate() on a host token list, prefill included; the synthetic "
                        "draft's truth table (an iterative decode through the same "
                        "stages, SURVEY H6) is built before the timer"},
        "gpu_launches": launches,
        "roofline": rf,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }


def _reference_baseline(shape: str, n_decode: int) -> dict:
    """The reference itself (oracle/_ref, vendored by oracle/vendor_ref.sh)
    on this host's cores: its own decoder at the target's width, per-token
    time extrapolated to the target's depth."""
    import numpy  # noqa: F401  (BLAS loaded before threadpoolctl looks)
    from oracle import reference_arm as R
    from paper_2407_11798_b200.model import LLAMA_SHAPES
    sh = LLAMA_SHAPES[shape]
    sp = R.load()
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        with threadpool_limits(limits=os.cpu_count() or 1):
            cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
            w = R.width_extrapolated(sp, sh["embed_dim"], sh["n_heads"], sh["n_layers"],
                                     vocab=sh["vocab_size"], n_decode=n_decode,
                                     layers=1 if sh["embed_dim"] >= 8192 else 2)
    except ImportError:
        cores = os.cpu_count() or 1
        w = R.width_extrapolated(sp, sh["embed_dim"], sh["n_heads"], sh["n_layers"],
                                 vocab=sh["vocab_size"], n_decode=n_decode)
    return {"value": w["tokens_per_s"], "unit": "tokens/s", "cores": cores, "kind": "reference",
            "sample": w["sample"], "ms_per_token": w["ms_per_token"],
            "per_layer_ms": round(w["per_layer_ms"], 2), "head_ms": round(w["head_ms"], 2)}


def run_reference(args) -> dict:
    """The reference arm: the reference's CPU implementation of the path on
    this host's cores (rank 0 only).  With oracle/_ref present that is the
    reference package itself (kind "reference"): its decoder at the
    target's width (the reference cannot run Llama; extrapolated), plus the
    cfg1 figures BASELINE.md §3 asks for (reference_decode and the four
    modes under simulate(clock="wall")).  Without it, the float64 oracle
    port of the Llama forward (kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import reference_arm as R
    use_ref = R.available()
    vals = []
    t0 = time.perf_counter()
    if use_ref:
        c = _reference_baseline(args.target, n_decode=max(1, args.steps))
        vals = [c]
        sp = R.load()
        extra = {"reference_cfg1": {"setting": {**R.CFG1, "stages": 4, "alpha": 0.8,
                                                "clock": "wall", "delays": 0},
                                    "reference_decode": R.cfg1_decode(sp),
                                    "simulate_wall": R.cfg1_modes(sp)}}
    else:
        for _ in range(args.warmup):
            cpu_baseline(n_decode=1, shape=args.target)
        for _ in range(args.steps):
            vals.append(cpu_baseline(n_decode=2, shape=args.target))
        extra = {}
    el = time.perf_counter() - t0
    v = statistics.median(x["value"] for x in vals)
    c = vals[0]
    return {"metric": "single-request generated tokens/s + inter-token latency",
            "value": round(v, 4), "unit": "tokens/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(el / max(1, args.steps) * 1e3, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (random-init weights)", "impl": "reference",
            "config": {"workload": WORKLOADS.get((args.target, args.draft),
                                                 f"{args.target} target")
                                   + " (CPU reference, float64, one request)",
                       "target": args.target, "prompt_len": PROMPT_LEN},
            "itl_ms": round(1e3 / v, 1),
            "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "cores": c["cores"],
                             "kind": c["kind"], "sample": c["sample"]},
            "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}, **extra}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--gen-len", type=int, default=GEN_LEN)
    ap.add_argument("--target", default=TARGET, help="target shape (model.LLAMA_SHAPES)")
    ap.add_argument("--draft", default=DRAFT, help="draft shape (model.LLAMA_SHAPES)")
    ap.add_argument("--alpha", type=float, default=ALPHA,
                    help="synthetic draft acceptance (configs[3]: low alpha exercises "
                         "early cancellation)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--node-weights", type=lambda v: tuple(float(x) for x in v.split(",")),
                    default=None, help="pipeline stage speed weights (reference node_weights,"
                                       " engine.py:186-224), e.g. 0.8,1")
    ap.add_argument("--no-continuous", action="store_true",
                    help="engine knob (reference ExperimentConfig.continuous=False): one speculative"
                         " micro-batch per accepted round")
    ap.add_argument("--no-ramp", action="store_true",
                    help="engine knob: full micro-batches from a fresh chain (spec_ramp=False)")
    ap.add_argument("--free-draft", action="store_true",
                    help="experiment only (not a headline): the synthetic draft skips its forward")
    ap.add_argument("--reference-policy", action="store_true",
                    help="the reference head's scheduling (no frontier folding, unbounded "
                         "in-flight speculation, draft always on the 16-SM cluster kernel)")
    ap.add_argument("--max-inflight", type=int, default=None)
    ap.add_argument("--tree-width", type=int, default=None, choices=[1, 2],
                    help="1 = chain speculation; 2 = + the draft's runner-up as a sibling "
                         "leaf per proposal (configs[4] sweep)")
    ap.add_argument("--alpha-sibling", type=float, default=None,
                    help="synthetic draft: P(runner-up is the target's token | first choice "
                         "is not), tree width 2")
    ap.add_argument("--depth", type=int, default=None, choices=[1, 2, 3, 4],
                    help="speculation depth (microbatch = tree_cap)")
    ap.add_argument("--fold", choices=["on", "off"], default=None)
    ap.add_argument("--microbatch", type=int, default=None)
    ap.add_argument("--partitions", type=int, default=None)
    ap.add_argument("--cutoff", type=float, default=None)
    ap.add_argument("--draft-gpu", default="auto", choices=["auto", "on", "off"],
                    help="N>1: rank 0 = head + dedicated draft GPU, stages on ranks 1..N-1 "
                         "(the reference's nodes = stages + draft node); auto = on "
                         "(measured: the dedicated layout wins at N=2 and N=4)")
    args = ap.parse_args()
    if (args.depth is None and args.microbatch is None and not args.reference_policy
            and args.tree_width in (None, 1)):
        # speculation depth (proposals per run) by layout and acceptance, for
        # async and the sync baseline alike (profiles/r02_sweep_depth.txt):
        # alpha 0.66: N=1 3 > 4, N=2 4 > 3, N=4 2 > 3 > 4; alpha 0.9: 4 at
        # every N.  The engine's own default stays the reference's microbatch 4.
        if args.alpha >= 0.8:
            args.depth = 4
        else:
            args.depth = 3 if args.gpus == 1 else 4 if args.gpus == 2 else 2
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None and int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
