"""paper_2407_11798_b200: B200-native PipeInfer hot path.

Drop-in for the reference ``specpipe`` package's hot path (the public names
of ``specpipe/__init__.py:3-58``), re-built on hand-written sm_100a kernels
behind a C ABI (``include/specpipe_b200.h``).  No CPU fallback: compute
entry points raise ``LibraryMissing`` if ``libspecpipe_b200.so`` is absent.
"""

from .errors import (  # noqa: F401
    AllocationExhausted,
    CacheError,
    EngineError,
    LibraryMissing,
    ModelError,
    ProtocolError,
    SpeculationError,
    TransportError,
    VerifyError,
)
from .kvcache import KVCache, SequenceAllocator, free_sequence  # noqa: F401
from .model import (  # noqa: F401
    NON_SPECULATIVE,
    PREFILL,
    SPECULATIVE,
    Batch,
    BatchToken,
    DeviceModel,
    ModelConfig,
    RowResult,
    SerialDecoder,
    TreeAttentionMask,
    build_mask_from_cache,
    build_model,
    build_tree_mask,
    eval_layers,
    greedy_sample,
    llama_config,
    logits,
    max_softmax,
    reference_decode,
    sample_prompt,
    second_best,
)
from .verify import (  # noqa: F401
    VerifyResult,
    apply_acceptance,
    detect_stale_runs,
    verify_run,
)
from .speculation import (  # noqa: F401
    CutoffController,
    DraftBackend,
    SpeculationState,
    SyntheticDraft,
    ToyDraft,
    rollback_draft,
    speculate_microbatch,
    sync_backend,
)
from .engine import (  # noqa: F401
    ExperimentConfig,
    RunMetrics,
    RunRecord,
    SimResult,
    generate,
    plan_layer_split,
    simulate,
    token_checksum,
)

from . import report  # noqa: F401,E402  (reference bench.py's report contract)

LayeredModel = DeviceModel

__version__ = "0.1.0"

# the reference's public names (specpipe/__init__.py:3-58) plus the B200 extras
__all__ = [
    "AllocationExhausted", "Batch", "BatchToken", "CutoffController", "ExperimentConfig",
    "KVCache", "LayeredModel", "ModelConfig", "SequenceAllocator", "SimResult",
    "SpeculationState", "SyntheticDraft", "ToyDraft", "VerifyResult", "apply_acceptance",
    "build_model", "build_tree_mask", "detect_stale_runs", "eval_layers", "greedy_sample",
    "logits", "plan_layer_split", "reference_decode", "rollback_draft", "sample_prompt",
    "simulate", "speculate_microbatch", "verify_run",
    # B200 additions
    "TreeAttentionMask", "build_mask_from_cache", "generate", "RunMetrics", "RunRecord",
    "token_checksum", "DeviceModel", "SerialDecoder", "RowResult", "max_softmax",
    "second_best", "llama_config", "free_sequence", "CacheError", "ModelError",
    "EngineError", "ProtocolError", "SpeculationError", "TransportError", "VerifyError",
    "LibraryMissing", "DraftBackend", "sync_backend", "NON_SPECULATIVE", "PREFILL",
    "SPECULATIVE", "VerifyResult",
]
