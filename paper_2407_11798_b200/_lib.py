"""ctypes binding of ``libspecpipe_b200.so`` (the C ABI in include/specpipe_b200.h).

There is no fallback: if the library is missing or cannot be loaded, every
compute entry point raises ``LibraryMissing``.  The product path never routes
through a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import CacheError, LibraryMissing, ModelError, ProtocolError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SP_LIB_PATH") or os.path.join(HERE, "libspecpipe_b200.so")  # override: A/B tools only

# ---- status / flag constants (mirror the header) ---------------------------
SP_OK, SP_ERR_MODEL, SP_ERR_CACHE, SP_ERR_PROTOCOL, SP_ERR_CUDA, SP_ERR_ARG, \
    SP_ERR_CAPACITY = range(7)
SP_DEV_BAD_TOKEN, SP_DEV_BAD_POS, SP_DEV_NONFINITE, SP_DEV_NAN_LOGITS, \
    SP_DEV_COVERAGE, SP_DEV_BAD_SEQ, SP_DEV_PLAN_OVERFLOW = 1, 2, 4, 8, 16, 32, 64
SP_ARCH_REF, SP_ARCH_LLAMA = 0, 1
SP_DTYPE_F32, SP_DTYPE_BF16 = 0, 1
SP_KIND_PREFILL, SP_KIND_NONSPEC, SP_KIND_SPEC = 0, 1, 2
SP_STATUS_VALID, SP_STATUS_PLACEHOLDER = 0, 1
SP_FWD_CHECK_COVERAGE, SP_FWD_SKIPPABLE, SP_FWD_CONTINUE, SP_FWD_CHAIN = 1, 2, 4, 8
SP_EPI_STORE, SP_EPI_RESID, SP_EPI_QKV, SP_EPI_GELU, SP_EPI_SWIGLU, SP_EPI_LMHEAD = range(6)
SP_STEP_TIP, SP_STEP_CHAIN = 1, 2
SP_DRAFT_KIND_AUTO, SP_DRAFT_KIND_CLUSTER, SP_DRAFT_KIND_GRID = 0, 1, 2
SP_LAYOUT_NATURAL, SP_LAYOUT_TC_TILED, SP_LAYOUT_SWZ8 = 0, 1, 2


class sp_model_dims(C.Structure):
    _fields_ = [("arch", C.c_int32), ("vocab", C.c_int32), ("d_model", C.c_int32),
                ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("ffn_dim", C.c_int32), ("max_context", C.c_int32),
                ("w_dtype", C.c_int32), ("norm_eps", C.c_float),
                ("rope_theta", C.c_float), ("w_layout", C.c_int32)]


class sp_token(C.Structure):
    _fields_ = [("token", C.c_int32), ("pos", C.c_int32), ("seq_mask", C.c_uint32),
                ("want_logits", C.c_int32)]


class sp_row_result(C.Structure):
    _fields_ = [("argmax", C.c_int32), ("second", C.c_int32), ("conf", C.c_float),
                ("max_logit", C.c_float)]


class sp_gemv_args(C.Structure):
    _fields_ = [("w", C.c_void_p), ("w_dtype", C.c_int32), ("n_rows", C.c_int32),
                ("k", C.c_int32), ("x", C.c_void_p), ("m", C.c_int32),
                ("ldx", C.c_int32), ("norm", C.c_int32), ("norm_eps", C.c_float),
                ("gain", C.c_void_p), ("epi", C.c_int32), ("out", C.c_void_p),
                ("ldo", C.c_int32), ("q_rows", C.c_int32), ("kv_rows", C.c_int32),
                ("k_cache", C.c_void_p), ("v_cache", C.c_void_p),
                ("cache_row0", C.c_int32), ("rope", C.c_int32),
                ("head_dim", C.c_int32), ("rope_theta", C.c_float),
                ("toks", C.c_void_p), ("err", C.c_void_p), ("run_state", C.c_void_p),
                ("run_state_w", C.c_void_p), ("cancel_word", C.c_void_p),
                ("run_id", C.c_int32), ("cache_row0_dev", C.c_void_p), ("w_swz", C.c_int32)]


class sp_tc_args(C.Structure):
    _fields_ = [("w", C.c_void_p), ("n_rows", C.c_int32), ("k", C.c_int32), ("m", C.c_int32),
                ("tok0", C.c_int32), ("epi", C.c_int32), ("norm", C.c_int32),
                ("norm_eps", C.c_float), ("out", C.c_void_p), ("ldo", C.c_int32),
                ("q_rows", C.c_int32), ("kv_rows", C.c_int32), ("k_cache", C.c_void_p),
                ("v_cache", C.c_void_p), ("cache_row0", C.c_int32), ("head_dim", C.c_int32),
                ("rope_theta", C.c_float), ("toks", C.c_void_p), ("ss_in", C.c_void_p),
                ("ss_nparts", C.c_int32), ("ss_ld", C.c_int32), ("ss_out", C.c_void_p),
                ("xb_next", C.c_void_p), ("gain_next", C.c_void_p), ("scratch", C.c_void_p),
                ("tickets", C.c_void_p), ("ksplit", C.c_int32), ("max_ctas", C.c_int32),
                ("err", C.c_void_p),
                ("run_state", C.c_void_p), ("cache_row0_dev", C.c_void_p),
                ("lm_out", C.c_void_p), ("lm_part", C.c_void_p), ("lm_ticket", C.c_void_p),
                ("lm_err_out", C.c_void_p), ("lm_status_out", C.c_void_p),
                ("lm_tip", C.c_void_p), ("lm_gate", C.c_void_p), ("lm_chain_gate", C.c_int32),
                ("lm_cutoff", C.c_float), ("lm_hdr", C.c_void_p)]


P = C.c_void_p
I = C.c_int
U32 = C.c_uint32
F = C.c_float

# name -> (restype, argtypes)
PROTOTYPES = {
    "sp_embed": (I, [P, P, P, P, I, P, P, P]),
    "sp_gemv": (I, [P, P]),
    "sp_tc_gemm": (I, [P, P, I, P]),
    "sp_build_plan": (I, [P, P, I, I, P, I, I, P, P, I, I, P, P]),
    "sp_attention": (I, [P, P, P, I, P, P, I, I, I, I, I, I, P, P, P, P, P]),
    "sp_kv_meta_write": (I, [P, P, I, P, I, I, I, P, P]),
    "sp_kv_copy": (I, [P, P, I, I, U32, I, I, P]),
    "sp_kv_remove": (I, [P, P, I, U32, I, P]),
    "sp_kv_keep": (I, [P, I, I, P]),
    "sp_lmhead": (I, [P, I, I, I, P, P, I, I, F, P, P, P, P, P, P, P, P]),
    "sp_stage_create": (I, [P, I, I, I, I, I, P]),
    "sp_stage_destroy": (I, [P]),
    "sp_stage_set_embedding": (I, [P, P, P]),
    "sp_stage_set_layer": (I, [P, I, P, P, P, P, P, P]),
    "sp_stage_set_head": (I, [P, P, P]),
    "sp_stage_set_head_tiled": (I, [P, P]),
    "sp_stage_set_cancel_table": (I, [P, P, I]),
    "sp_stage_set_cta_budget": (I, [P, I]),
    "sp_stage_forward": (I, [P, P, I, I, I, I, P, P, P, P, I, P]),
    "sp_stage_forward_range": (I, [P, P, I, I, I, I, P, P, P, P, I, I, I, P]),
    "sp_stage_lmhead": (I, [P, P, P, I, P, P, P, I, I, F, P]),
    "sp_stage_step": (I, [P, P, I, I, I, I, P, I, I, F, P, P, P, P]),
    "sp_stage_io": (I, [P, P, P]),
    "sp_stage_decode_chain": (I, [P, P, I, I, P, I, F, P, P, P]),
    "sp_stage_truncate": (I, [P, I]),
    "sp_stage_decode_chain_ok": (I, [P]),
    "sp_stage_set_draft_kernel": (I, [P, I]),
    "sp_last_error": (C.c_char_p, []),
    "sp_stage_set_skip_graphs": (I, [P, I]),
    "sp_stage_compact": (I, [P, P]),
    "sp_stage_draft_profile": (I, [P, P, I]),
    "sp_stage_chain_begin": (I, [P, F, P, P]),
    "sp_stage_chain_state": (I, [P, P, P]),
    "sp_stage_invalidate_tip": (I, [P, P]),
    "sp_stage_cache_copy": (I, [P, I, U32, I, P]),
    "sp_stage_cache_remove": (I, [P, I, I, P]),
    "sp_stage_cache_keep": (I, [P, I, P]),
    "sp_stage_reset": (I, [P, P]),
    "sp_stage_cache_insert_meta": (I, [P, P, I, P]),
    "sp_stage_n_cells": (I, [P]),
    "sp_stage_meta_sync": (I, [P, P, P, I, P]),
    "sp_stage_read_kv_sync": (I, [P, I, I, P, P, P]),
    "sp_stage_error_sync": (I, [P, I, P]),
    "sp_stage_error_ptr": (I, [P, P]),
    "sp_stage_plan_sync": (I, [P, P, P, I, P]),
    "sp_stage_ld_vis": (I, [P]),
    "sp_stage_set_plan": (I, [P, P, P, I, P]),
    "sp_stage_plan_only": (I, [P, P, I, I, P]),
    "sp_host_register": (I, [P, C.c_size_t, P]),
    "sp_host_unregister": (I, [P]),
    "sp_signal": (I, [P, I, P]),
    "sp_copy_async": (I, [P, P, C.c_size_t, P]),
    "sp_version": (C.c_char_p, []),
    "sp_device_arch": (I, []),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the library; raise LibraryMissing otherwise."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryMissing(
                f"{path} not found: build it with `python -m paper_2407_11798_b200.build` "
                "(there is no CPU fallback)")
        try:
            lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
        except OSError as e:  # pragma: no cover - depends on the box
            raise LibraryMissing(f"cannot load {path}: {e}") from e
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list:
    return sorted(PROTOTYPES)


def check(rc: int, what: str = "") -> None:
    """Map a C status to the reference's exception types."""
    if rc == SP_OK:
        return
    msg = f"{what}: status {rc}"
    if rc == SP_ERR_MODEL:
        raise ModelError(msg)
    if rc in (SP_ERR_CACHE, SP_ERR_CAPACITY):
        raise CacheError(msg)
    if rc == SP_ERR_PROTOCOL:
        raise ProtocolError(msg)
    detail = ""
    try:
        detail = (load().sp_last_error() or b"").decode(errors="replace")
    except Exception:
        pass
    raise RuntimeError(f"specpipe_b200 CUDA failure ({msg}{': ' + detail if detail else ''})")


def raise_device_error(bits: int, where: str = "") -> None:
    """Translate sticky device error bits (checked at run completion)."""
    if not bits:
        return
    if bits & SP_DEV_COVERAGE:
        raise ProtocolError(f"{where}: token does not see exactly its position's "
                            "cells (coverage violation)")
    if bits & SP_DEV_PLAN_OVERFLOW:
        raise ProtocolError(f"{where}: visible list exceeded the launch bound")
    if bits & SP_DEV_BAD_SEQ:
        raise CacheError(f"{where}: sequence id out of range")
    if bits & SP_DEV_NONFINITE:
        raise ModelError(f"{where}: non-finite activations")
    if bits & SP_DEV_NAN_LOGITS:
        raise ModelError(f"{where}: NaN in logits")
    if bits & SP_DEV_BAD_TOKEN:
        raise ModelError(f"{where}: token id outside vocab")
    if bits & SP_DEV_BAD_POS:
        raise ModelError(f"{where}: position exceeds max_context")
    raise RuntimeError(f"{where}: device error bits {bits:#x}")
