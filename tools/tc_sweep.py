"""Per-matrix timing of the 7B GEMM set (32 layers each) on the tcgen05 path
vs the CUDA-core GEMV, for several token counts M (CUDA events)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_11798_b200 as sp
from paper_2407_11798_b200 import _lib

cfg = sp.llama_config(os.environ.get("SHAPE", "llama2-7b"))
NL = cfg.n_layers
m = sp.build_model(cfg, layer_range=(0, NL), embedding=False, head=False)
lib = _lib.load()
d, f = cfg.embed_dim, cfg.hidden
X = torch.randn((256, f), device="cuda").to(torch.bfloat16)
Xf = torch.randn((256, f), device="cuda")
out = torch.zeros((256, 2 * f + 3 * d), device="cuda")
scratch = torch.zeros(8 << 20, device="cuda")
tick = torch.zeros(4096, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
kinds = {"qkv": (3 * d, d), "o": (d, d), "up": (2 * f, d), "down": (d, f)}


def timed(fn, reps=5):
    """GPU time of fn's launches: captured once into a CUDA graph, replayed."""
    global s
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s = st.cuda_stream
        with torch.cuda.graph(g, stream=st):
            fn()
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])


for M in [int(x) for x in (sys.argv[1:] or ["1", "4", "16"])]:
    for name, (n, k) in kinds.items():
        ws = [m.layers[l][{"qkv": "qkv", "o": "o", "up": "up", "down": "down"}[name]]
              for l in range(NL)]
        a = _lib.sp_tc_args()
        a.n_rows, a.k, a.m, a.epi, a.norm = n, k, M, 0, 0
        a.out, a.ldo = out.data_ptr(), out.shape[1]
        a.scratch, a.tickets = scratch.data_ptr(), tick.data_ptr()
        ks = int(os.environ.get("KSPLIT", "0"))
        a.ksplit = ks
        a.max_ctas = int(os.environ.get("MAXCTAS", "0"))   # a sharing budget (ticket merge)

        def tc():
            for w in ws:
                a.w = w.data_ptr()
                _lib.check(lib.sp_tc_gemm(C.byref(a), X.data_ptr(), 256, s))

        g = _lib.sp_gemv_args()
        g.w_dtype, g.n_rows, g.k, g.x, g.m, g.ldx = 1, n, k, Xf.data_ptr(), M, f
        g.epi, g.out, g.ldo = 0, out.data_ptr(), out.shape[1]

        def cc():
            for w in ws:
                g.w = w.data_ptr()
                _lib.check(lib.sp_gemv(C.byref(g), s))

        byt = NL * n * k * 2
        t1 = timed(tc)
        t2 = timed(cc) if not os.environ.get("NOGEMV") else t1
        print(f"M={M:3d} {name:5s} tc {t1*1e3/NL:7.2f} us/launch {byt/t1/1e6:7.0f} GB/s | "
              f"gemv {t2*1e3/NL:7.2f} us {byt/t2/1e6:7.0f} GB/s", flush=True)
