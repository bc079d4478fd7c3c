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
