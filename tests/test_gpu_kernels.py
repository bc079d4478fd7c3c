"""Kernel-level GPU checks through the C ABI against numpy fp64 references:
GEMV epilogues (K2/K6/K7), LM head top-2/max-softmax (K9), embedding (K1)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2407_11798_b200 import _lib
    return torch, _lib, _lib.load()


def _gemv(env, W, x, epi, norm=False, gain=None, dtype="f32", **kw):
    torch, _lib, lib = env
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    Wd = torch.from_numpy(W).to("cuda", tdt).contiguous()
    xd = torch.from_numpy(x.astype(np.float32)).cuda().contiguous()
    n, k = W.shape
    m = x.shape[0]
    ldo = kw.pop("ldo", n)
    out = torch.from_numpy(kw.pop("out_init", np.zeros((m, ldo), np.float32))).cuda()
    a = _lib.sp_gemv_args()
    a.w, a.w_dtype, a.n_rows, a.k = Wd.data_ptr(), (0 if dtype == "f32" else 1), n, k
    a.x, a.m, a.ldx = xd.data_ptr(), m, k
    a.norm, a.norm_eps = int(norm), kw.pop("eps", 1e-8)
    g = None
    if gain is not None:
        g = torch.from_numpy(gain.astype(np.float32)).cuda()
        a.gain = g.data_ptr()
    a.epi, a.out, a.ldo = epi, out.data_ptr(), ldo
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    a.err = err.data_ptr()
    for key, v in kw.items():
        setattr(a, key, v)
    _lib.check(lib.sp_gemv(C.byref(a), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), Wd.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("k", [16, 32, 64, 128, 256, 1000, 4096])
@pytest.mark.parametrize("m", [1, 2, 3, 8, 13])
@pytest.mark.parametrize("norm", [False, True])
def test_gemv_store_f32(env, k, m, norm):
    r = np.random.default_rng(k * 31 + m)
    n = 37
    W = r.standard_normal((n, k))
    x = r.standard_normal((m, k))
    y, _ = _gemv(env, W, x, 0, norm=norm)
    ref = x @ W.T
    if norm:
        ref = ref / np.sqrt((x * x).mean(1, keepdims=True) + 1e-8)
    assert np.abs(y - ref).max() < 1e-4 * max(1, np.abs(ref).max())


@pytest.mark.parametrize("k", [64, 4096, 11008])
@pytest.mark.parametrize("m", [1, 4, 5])
def test_gemv_bf16_gain_norm(env, k, m):
    r = np.random.default_rng(k + m)
    n = 64
    W = r.standard_normal((n, k)) / np.sqrt(k)
    x = r.standard_normal((m, k))
    gain = 1 + 0.1 * r.standard_normal(k)
    y, Wq = _gemv(env, W, x, 0, norm=True, gain=gain, dtype="bf16", eps=1e-5)
    h = x / np.sqrt((x * x).mean(1, keepdims=True) + 1e-5) * gain
    assert np.abs(y - h @ Wq.T).max() < 1e-3


def test_gemv_resid_gelu_swiglu(env):
    r = np.random.default_rng(3)
    k, n, m = 128, 64, 3
    W = r.standard_normal((n, k)) / np.sqrt(k)
    x = r.standard_normal((m, k))
    base = r.standard_normal((m, n)).astype(np.float32)
    y, _ = _gemv(env, W, x, 1, out_init=base.copy())
    assert np.abs(y - (base + x @ W.T)).max() < 1e-4
    y, _ = _gemv(env, W, x, 3, norm=True)
    h = (x / np.sqrt((x * x).mean(1, keepdims=True) + 1e-8)) @ W.T
    g = 0.5 * h * (1 + np.tanh(0.7978845608028654 * (h + 0.044715 * h ** 3)))
    assert np.abs(y - g).max() < 1e-4
    y, _ = _gemv(env, W, x, 4, ldo=n // 2)
    z = x @ W.T
    sw = z[:, 0::2] / (1 + np.exp(-z[:, 0::2])) * z[:, 1::2]
    assert np.abs(y - sw).max() < 1e-4


def test_lmhead_top2_conf(env):
    torch, _lib, lib = env
    r = np.random.default_rng(5)
    for V, d, n in [(64, 32, 1), (32000, 256, 3), (17, 16, 2)]:
        W = r.standard_normal((V, d)) / np.sqrt(d)
        x = r.standard_normal((n, d))
        if V == 17:
            W[5] = W[3]      # exact tie: lowest id must win
        Wd = torch.from_numpy(W.astype(np.float32)).cuda()
        xd = torch.from_numpy(x.astype(np.float32)).cuda()
        out = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
        logit = torch.zeros((n, V), dtype=torch.float32, device="cuda")
        scratch = torch.zeros(n * ((V + 7) // 8) * 8, dtype=torch.float32, device="cuda")
        tick = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.sp_lmhead(Wd.data_ptr(), 0, V, d, xd.data_ptr(), None, n, 1, 1e-8,
                                 None, out.data_ptr(), logit.data_ptr(), scratch.data_ptr(),
                                 tick.data_ptr(), None, None,
                                 torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        lg = (x / np.sqrt((x * x).mean(1, keepdims=True) + 1e-8)) @ W.T
        o = out.cpu().numpy()
        L = logit.cpu().numpy()
        assert np.abs(L - lg).max() < 1e-4
        for i in range(n):
            v = L[i].astype(np.float64)
            assert o[i, 0] == int(np.argmax(v))
            v2 = v.copy()
            v2[o[i, 0]] = -np.inf
            assert o[i, 1] == int(np.argmax(v2))
            conf = o[i, 2:3].view(np.float32)[0]
            e = np.exp(v - v.max())
            assert abs(conf - e.max() / e.sum()) < 1e-5


# ---------------------------------------------------------------------------
# tcgen05 skinny GEMM (bf16 path)
# ---------------------------------------------------------------------------

def _tc(env, W, X, epi=0, m=None, norm=False, ss=None, ksplit=0, out=None, ldo=None,
        **kw):
    torch, _lib, lib = env
    n, k = W.shape
    m = X.shape[0] if m is None else m
    from paper_2407_11798_b200.model import tile_weight, untile_weight
    Wd = torch.from_numpy(W.astype(np.float32)).to("cuda", torch.bfloat16).contiguous()
    Wt = tile_weight(Wd)
    assert torch.equal(untile_weight(Wt), Wd)
    xr = max(128, X.shape[0])
    Xd = torch.zeros((xr, k), dtype=torch.bfloat16, device="cuda")
    Xd[:X.shape[0]] = torch.from_numpy(X.astype(np.float32)).to("cuda", torch.bfloat16)
    if out is None:
        out = torch.zeros((m, n if ldo is None else ldo), dtype=torch.float32, device="cuda")
    scratch = torch.zeros(8 << 20, dtype=torch.float32, device="cuda")
    tick = torch.zeros(4096, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = _lib.sp_tc_args()
    a.w = Wt.data_ptr()
    a.n_rows, a.k, a.m, a.epi, a.norm, a.norm_eps = n, k, m, epi, int(norm), 1e-5
    a.out, a.ldo = out.data_ptr(), out.shape[1]
    a.scratch, a.tickets, a.err, a.ksplit = scratch.data_ptr(), tick.data_ptr(), err.data_ptr(), ksplit
    keep = []
    if ss is not None:
        ssd = torch.from_numpy(ss.astype(np.float32)).cuda().contiguous()
        keep.append(ssd)
        a.ss_in, a.ss_nparts, a.ss_ld = ssd.data_ptr(), ss.shape[0], ss.shape[1]
    for key, v in kw.items():
        if hasattr(v, "data_ptr"):
            keep.append(v)
            v = v.data_ptr()
        setattr(a, key, v)
    _lib.check(lib.sp_tc_gemm(C.byref(a), Xd.data_ptr(), xr,
                              torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    Wq = Wd.float().cpu().numpy().astype(np.float64)
    Xq = Xd[:X.shape[0]].float().cpu().numpy().astype(np.float64)
    return out, Wq, Xq, tick


@pytest.mark.parametrize("m", [1, 3, 5, 16, 17, 128, 130])
@pytest.mark.parametrize("shape", [(128, 64), (256, 768), (4096, 4096), (384, 11008)])
def test_tc_gemm_store(env, m, shape):
    n, k = shape
    r = np.random.default_rng(n + k + m)
    W = r.standard_normal((n, k)) / np.sqrt(k)
    X = r.standard_normal((m, k))
    out, Wq, Xq, tick = _tc(env, W, X)
    ref = Xq @ Wq.T
    got = out.cpu().numpy()
    assert np.abs(got - ref).max() < 2e-3 * max(1.0, np.abs(ref).max()), np.abs(got - ref).max()
    assert int(tick.abs().sum()) == 0          # split-K tickets reset


def test_tc_gemm_norm_and_ksplit_invariance(env):
    r = np.random.default_rng(1)
    n, k, m = 512, 4096, 4
    W = r.standard_normal((n, k)) / np.sqrt(k)
    X = r.standard_normal((m, k))
    ss = np.stack([np.full(m, 0.0), (X * X).sum(1)])   # 2 partials summing to the stat
    outs = []
    for ks in (1, 3, 7):
        out, Wq, Xq, _ = _tc(env, W, X, norm=True, ss=ss, ksplit=ks)
        outs.append(out.cpu().numpy())
    inv = 1 / np.sqrt(ss.sum(0) / k + 1e-5)
    ref = (Xq @ Wq.T) * inv[:, None]
    for o in outs:
        assert np.abs(o - ref).max() < 2e-3
    # a token's result does not depend on the batch it shares the launch with
    o1, _, _, _ = _tc(env, W, X[:1], norm=True, ss=ss[:, :1], ksplit=3)
    assert np.array_equal(o1.cpu().numpy()[0], outs[1][0])


def test_tc_gemm_resid_swiglu(env):
    torch = env[0]
    r = np.random.default_rng(2)
    n, k, m = 256, 1024, 3
    W = r.standard_normal((n, k)) / np.sqrt(k)
    X = r.standard_normal((m, k))
    base = r.standard_normal((m, n)).astype(np.float32)
    g = (1 + 0.1 * r.standard_normal(n)).astype(np.float32)
    x = torch.from_numpy(base.copy()).cuda()
    xb = torch.zeros((m, n), dtype=torch.bfloat16, device="cuda")
    ssout = torch.zeros((n // 128, m), dtype=torch.float32, device="cuda")
    out, Wq, Xq, _ = _tc(env, W, X, epi=1, out=x, xb_next=xb,
                         gain_next=torch.from_numpy(g).cuda(), ss_out=ssout, ss_ld=m)
    new = base + Xq @ Wq.T
    assert np.abs(x.cpu().numpy() - new).max() < 2e-3
    assert np.abs(xb.float().cpu().numpy() - new * g).max() < 2e-2
    assert np.abs(ssout.cpu().numpy().sum(0) - (new * new).sum(1)).max() < 1e-2
    hb = torch.zeros((m, n // 2), dtype=torch.bfloat16, device="cuda")
    _tc(env, W, X, epi=4, out=hb)
    z = Xq @ Wq.T
    sw = z[:, 0::2] / (1 + np.exp(-z[:, 0::2])) * z[:, 1::2]
    assert np.abs(hb.float().cpu().numpy() - sw).max() < 2e-2



@pytest.mark.parametrize("shape", [(4096, 4096), (4096, 11008), (12288, 4096)])
def test_tc_gemm_tile_size_invariance(env, shape):
    """A token's GEMM result is the same whether its run takes the 16-token
    or the 128-token tile path (runs of <= 16 vs 17+ tokens): the split-K
    partition is a function of the shape only (7B O / down / QKV shapes)."""
    n, k = shape
    r = np.random.default_rng(n + k)
    W = r.standard_normal((n, k)) / np.sqrt(k)
    X = r.standard_normal((20, k))
    big, _, _, _ = _tc(env, W, X)                 # m = 20: the 128-token tile
    small, _, _, _ = _tc(env, W, X[:4])           # m = 4: the 16-token tile
    assert np.array_equal(big.cpu().numpy()[:4], small.cpu().numpy())


def test_attention_grid_and_merge_path_bitwise(tmp_path):
    """The attention's bits do not depend on its grid or merge path
    (attention.cu attn_kernel): one split per CTA equals CTAs looping over
    several splits, and merging the split partials from shared memory
    equals merging them from L2; the tensor-core kernel (40-query runs,
    attention_tc.cu) gives the same bits with its row tiles on one CTA or
    spread over row blocks -- on chains, tree siblings and arbitrary
    per-query plans, head dims 64 / 128, GQA; every output is also checked
    against fp32 (model.py:394-415)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for name, extra in (("base", {}), ("loops", {"SP_ATT_CTAS_PER_SM": "1"}),
                        ("l2merge", {"SP_ATT_MERGE_SMEM_KB": "0"}),
                        ("tc_one_block", {"SP_ATT_TC_RB": "1"})):
        path = str(tmp_path / f"{name}.npz")
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "attn_variant_main.py"),
                            path], env=env, cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        outs[name] = np.load(path)
    base = outs["base"]
    for name in ("loops", "l2merge", "tc_one_block"):
        for key in base.files:
            assert np.array_equal(base[key], outs[name][key]), (name, key)
