"""Attention through the C ABI (sp_attention) over a fixed set of plans:
verification chains, tree siblings whose plans leave the longest query's,
arbitrary per-query subsets, GQA and head dims 64 / 128, bf16 K/V.  Writes
every output to an .npz so tests/test_gpu_kernels.py can run it under
different grids / merge paths (SP_ATT_CTAS_PER_SM, SP_ATT_MERGE_SMEM_KB)
and compare the bits.  Usage: python tests/attn_variant_main.py OUT.npz"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_11798_b200 import _lib  # noqa: E402


def plans_for(kind, ctx, n, gen):
    """(list of row lists, cells) -- a query's own row is last."""
    if kind == "chain":     # prefix 0..ctx-1, run rows ctx.., query i sees run rows < i
        return [list(range(ctx)) + [ctx + j for j in range(i)] + [ctx + i] for i in range(n)], ctx + n
    if kind == "tree":      # odd queries are siblings of the chain token before them
        out = []
        for i in range(n):
            if i % 2 == 1:      # sibling of chain token i-1: sees the chain before i-1
                out.append(list(range(ctx)) + [ctx + j for j in range(0, i - 1, 2)] + [ctx + i])
            else:
                out.append(list(range(ctx)) + [ctx + j for j in range(0, i, 2)] + [ctx + i])
        return out, ctx + n
    # "subset": each query an arbitrary increasing subset of the cells
    cells = ctx + n
    out = []
    for i in range(n):
        keep = sorted(gen.choice(ctx, size=max(1, int(ctx * gen.uniform(0.3, 1.0))), replace=False))
        out.append([int(r) for r in keep] + [ctx + i])
    return out, cells


CASES = []
for (H, KH, HD) in ((32, 32, 128), (16, 4, 64)):
    for kind in ("chain", "tree", "subset"):
        for n in (1, 2, 5, 9, 16, 40):   # (40: the tensor-core kernel)
            for ctx in (3, 31, 32, 33, 100, 384, 1000):
                if kind != "chain" and n == 1:
                    continue
                CASES.append((H, KH, HD, kind, n, ctx))


def main():
    out_path = sys.argv[1]
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    res = {}
    for ci, (H, KH, HD, kind, n, ctx) in enumerate(CASES):
        gen = np.random.default_rng(ci)
        torch.manual_seed(ci)
        plans, cells = plans_for(kind, ctx, n, gen)
        k = torch.randn((cells, KH * HD), device=dev).to(torch.bfloat16)
        v = torch.randn((cells, KH * HD), device=dev).to(torch.bfloat16)
        q = torch.randn((n, H * HD), device=dev)
        ld = cells + 1
        vis = torch.zeros((n, ld), dtype=torch.int32, device=dev)
        vlen = torch.zeros(n, dtype=torch.int32, device=dev)
        for i, p in enumerate(plans):
            vis[i, :len(p)] = torch.tensor(p, dtype=torch.int32, device=dev)
            vlen[i] = len(p)
        max_vis = max(len(p) for p in plans) + 64     # a stage's bound exceeds the run's
        nsplit = (max_vis + 31) // 32
        out = torch.full((n, H * HD), float("nan"), device=dev)
        scratch = torch.zeros(n * H * nsplit * (HD + 2) + 1024, device=dev)
        tick = torch.zeros(max(H * n, 4096), dtype=torch.int32, device=dev)
        rs = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(lib.sp_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), _lib.SP_DTYPE_BF16,
                                    vis.data_ptr(), vlen.data_ptr(), ld, n, H, KH, HD, max_vis,
                                    out.data_ptr(), scratch.data_ptr(), tick.data_ptr(),
                                    rs.data_ptr(), C.c_void_p(st.cuda_stream)), "sp_attention")
        st.synchronize()
        # fp32 reference (loose: bf16 K/V are exact inputs, the kernel is fp32)
        for i, p in enumerate(plans):
            rows = torch.tensor(p, device=dev).long()
            for h in (0, H - 1):
                kh = h // (H // KH)
                s = (k[rows, kh * HD:(kh + 1) * HD].float() @ q[i, h * HD:(h + 1) * HD]) / HD ** 0.5
                o = torch.softmax(s, 0) @ v[rows, kh * HD:(kh + 1) * HD].float()
                err = (o - out[i, h * HD:(h + 1) * HD]).abs().max().item()
                assert err < 1e-4, (ci, H, KH, HD, kind, n, ctx, i, h, err)
        res[f"c{ci}"] = out.cpu().numpy()
    np.savez(out_path, **res)
    print(f"{len(CASES)} cases ok")


if __name__ == "__main__":
    main()
