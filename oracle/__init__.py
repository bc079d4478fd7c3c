"""CPU oracle for the PipeInfer hot path — TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference simulator's
algorithms (``/root/reference/pkg/src/specpipe``).  Every function cites the
reference ``file:line`` it follows.  It exists to *check* the B200 product
path (``paper_2407_11798_b200``), never to *be* it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
  / ``--impl reference`` legs may import it;
* the product package never imports it
  (``tests/test_host_cpu.py::test_product_never_imports_oracle`` enforces
  this), and the product fails loudly when its CUDA library is missing.

Parity pinning: the restatement is pinned against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.json|npz``), see
``tests/test_oracle_golden.py``.  The ``llama`` architecture variant has no
counterpart in the reference (the reference can only run its ``ref``
architecture); for it the oracle is an independent restatement of
the standard Llama block and its parity is *internal* (GPU vs this oracle on
the same weights), i.e. "parity unpinned" against the reference.
"""

from .model import (  # noqa: F401
    OracleConfig,
    OracleModel,
    OracleDecoder,
    build_ref_model,
    eval_layers,
    greedy_sample,
    logits,
    max_softmax,
    position_table,
    sample_prompt,
    second_best,
)
from .kvcache import OracleAllocator, OracleCache  # noqa: F401
from .verify import apply_acceptance, detect_stale_runs, verify_run  # noqa: F401
