"""Golden vectors for ``eval_layers(..., mask=...)`` by running the REFERENCE.

Build container only (``/root/reference`` is absent on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mask_golden.py

A prompt is evaluated into a cache, a speculative partition gets a copy of
its prefix, and a 4-token tree batch is evaluated twice through the
reference's ``eval_layers``: with the cache-derived mask and with a
caller-supplied ``build_tree_mask`` over a view that hides every third live
cell (model.py:262-284, 369-373).  Written: ``reference_mask.npz`` with the
tokens, the custom mask's per-query gather order and both logits blocks.
"""

from __future__ import annotations

import os

import numpy as np

from specpipe import kvcache as KC  # noqa: E402
from specpipe import model as M  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    cfg = M.ModelConfig(64, 32, 6, 4, 256, 7)
    model = M.build_model(cfg)
    prompt = M.sample_prompt(13, 12, 64)

    def fresh():
        cache = KC.KVCache(cfg.embed_dim, range(cfg.n_layers), cfg.max_context, 8)
        b = M.Batch(tokens=tuple(M.BatchToken(t, i, frozenset([0]), False)
                                 for i, t in enumerate(prompt)), kind="prefill")
        M.eval_layers(model, (0, cfg.n_layers), None, b, cache)
        cache.copy(0, [2, 3], len(prompt))
        return cache

    n = len(prompt)
    tree = M.Batch(tokens=(
        M.BatchToken(5, n, frozenset([2, 3]), True),
        M.BatchToken(9, n + 1, frozenset([2]), True),
        M.BatchToken(17, n + 1, frozenset([3]), True),
        M.BatchToken(33, n + 2, frozenset([2]), True)), kind="speculative", run_id=1)
    cache = fresh()
    plain = M.logits(model, M.eval_layers(model, (0, cfg.n_layers), None, tree, cache), tree)

    cache = fresh()
    view = cache.snapshot(0)
    keep = [i for i in range(len(view)) if i % 3 != 1]
    sub = KC.CacheView([view[i] for i in keep], np.asarray(view.rows)[keep])
    mask = M.build_tree_mask(tree, sub)
    custom = M.logits(model, M.eval_layers(model, (0, cfg.n_layers), None, tree, cache,
                                           mask=mask), tree)
    order = []
    rows = np.asarray(view.rows)[keep]
    for entries in mask.order:
        order.append([(src, int(rows[j]) if src == 0 else j) for src, j in entries])
    flat = np.array([(i, src, j) for i, e in enumerate(order) for src, j in e], dtype=np.int64)
    np.savez(os.path.join(HERE, "reference_mask.npz"), prompt=np.array(prompt),
             tree=np.array([(t.token, t.pos, sum(1 << s for s in t.seqs))
                            for t in tree.tokens]),
             plain=plain, custom=custom, order=flat)
    print("max |custom - plain| =", float(np.abs(custom - plain).max()))


if __name__ == "__main__":
    main()
