"""Attention kernel alone through the C ABI (sp_attention): one query per
run row over a synthetic plan of ``ctx`` cells, 7B (32/32 heads) or 70B
(64/8 heads, GQA) layout, bf16 K/V.  Prints us/launch (CUDA graph of 20
launches, events) and the K/V bytes per launch -> GB/s.  SP_ATT_LEGACY=1
selects the CUDA-core kernel.  Design tool.

    python tools/attn_bench.py [--heads 32 --kv-heads 32] [--n 1] [ctx ...]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_11798_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--hd", type=int, default=128)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("ctx", nargs="*", type=int, default=[384, 1024, 4096, 16384, 32768])
    a = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    H, KH, HD, n = a.heads, a.kv_heads, a.hd, a.n
    for ctx in a.ctx:
        cap = ctx + n
        k = torch.randn((cap, KH * HD), device=dev).to(torch.bfloat16)
        v = torch.randn((cap, KH * HD), device=dev).to(torch.bfloat16)
        q = torch.randn((n, H * HD), device=dev)
        ld = cap + 1
        vis = torch.zeros((n, ld), dtype=torch.int32, device=dev)
        vlen = torch.zeros(n, dtype=torch.int32, device=dev)
        for i in range(n):      # a chain: prefix rows 0..ctx-1, earlier run rows, own row
            vis[i, :ctx + i + 1] = torch.arange(ctx + i + 1, dtype=torch.int32, device=dev)
            vlen[i] = ctx + i + 1
        out = torch.zeros((n, H * HD), device=dev)
        nsplit = (ctx + n + 31) // 32
        scratch = torch.zeros(n * H * nsplit * (HD + 2) + 1024, device=dev)
        tick = torch.zeros(max(H * n, 4096), dtype=torch.int32, device=dev)
        rs = torch.zeros(1, dtype=torch.int32, device=dev)
        st = torch.cuda.Stream(dev)

        def launch():
            _lib.check(lib.sp_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), _lib.SP_DTYPE_BF16,
                                        vis.data_ptr(), vlen.data_ptr(), ld, n, H, KH, HD,
                                        ctx + n, out.data_ptr(), scratch.data_ptr(),
                                        tick.data_ptr(), rs.data_ptr(), C.c_void_p(st.cuda_stream)),
                       "sp_attention")
        launch()
        st.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20):
                launch()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                g.replay()
                e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        t = min(ts)
        assert torch.equal(out, ref), "attention output changed between launches"
        # fp32 check of head 0 of the last query against torch
        i = n - 1
        L = int(vlen[i])
        rows = vis[i, :L].long()
        errs = 0.0
        for h in (0, H - 1):
            kh = h // (H // KH)
            kk = k[rows, kh * HD:(kh + 1) * HD].float()
            vv = v[rows, kh * HD:(kh + 1) * HD].float()
            s = (kk @ q[i, h * HD:(h + 1) * HD]) / HD ** 0.5
            o = torch.softmax(s, 0) @ vv
            errs = max(errs, (o - out[i, h * HD:(h + 1) * HD]).abs().max().item())
        byt = ctx * KH * HD * 2 * 2
        print(f"ctx {ctx:6d} n {n} H {H}/{KH}: {t:8.2f} us/launch  K/V {byt / 1e6:7.2f} MB "
              f"-> {byt / t / 1e3:7.0f} GB/s   max|err| vs fp32 {errs:.2e}", flush=True)


if __name__ == "__main__":
    main()
