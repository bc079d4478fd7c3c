"""Time the 7B per-token GEMV set (QKV, O, gate/up, down x 32 layers) vs the
number of tokens M, with CUDA events (weights 12.9 GB >> L2)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200 import _lib

cfg = sp.llama_config("llama2-7b")
m = sp.build_model(cfg, layer_range=(0, 32), embedding=False, head=False)
lib = _lib.load()
d, f = cfg.embed_dim, cfg.hidden
q = kv = d
x = torch.randn((128, f), device="cuda")
out = torch.zeros((128, 2 * f + 3 * d), device="cuda")
toks = torch.zeros(128 * 4, dtype=torch.int32, device="cuda")
kc = torch.zeros((256, kv), dtype=torch.bfloat16, device="cuda")
args = []
nbytes = 0
for l in range(32):
    L = m.layers[l]
    for w, n, k, epi, norm in ((L["qkv"], 3 * d, d, 2, 1), (L["o"], d, d, 1, 0),
                               (L["up"], 2 * f, d, 4, 1), (L["down"], d, f, 1, 0)):
        a = _lib.sp_gemv_args()
        a.w, a.w_dtype, a.n_rows, a.k = w.data_ptr(), 1, n, k
        a.x, a.ldx = x.data_ptr(), f
        a.norm, a.norm_eps = norm, 1e-5
        a.epi, a.out, a.ldo = epi, out.data_ptr(), out.shape[1]
        a.q_rows, a.kv_rows, a.k_cache, a.v_cache = q, kv, kc.data_ptr(), kc.data_ptr()
        a.rope, a.head_dim, a.rope_theta, a.toks = 1, 128, 10000.0, toks.data_ptr()
        args.append(a)
        nbytes += n * k * 2
s = torch.cuda.current_stream().cuda_stream
for M in (1, 2, 3, 4, 5, 8, 16, 32, 128):
    for a in args:
        a.m = M
    ts = []
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for a in args:
            _lib.check(lib.sp_gemv(C.byref(a), s))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[1:])
    print(f"M={M:4d}  {t:8.3f} ms  {nbytes / t / 1e6:8.1f} GB/s  ({t / min(ts[1:]) if M == 1 else 0})", flush=True)
