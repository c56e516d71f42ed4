"""ctypes binding of libaccelgen_b200.so (declared in include/accelgen_b200.h).

There is deliberately no fallback: if the library is missing or CUDA is unavailable the
product path raises ``EngineFault`` instead of silently computing on the CPU.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import AllocationError, EngineFault, StateError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libaccelgen_b200.so"

AG_OK, AG_EINVAL, AG_ECUDA, AG_EALLOC, AG_EFAULT, AG_ENCCL, AG_ESTATE = range(7)

# kernel classes of ag_model_get_profile (include/accelgen_b200.h AG_K_*)
PROF_CLASSES = ("embed", "layernorm", "qkv_gemm", "attention", "out_gemm", "fc1_gemm", "fc2_gemm", "lmhead_gemm",
                "argmax", "allreduce")

i32 = C.c_int32
i64 = C.c_int64
f32 = C.c_float
f64 = C.c_double
vp = C.c_void_p
P_i32 = C.POINTER(C.c_int32)
P_f32 = C.POINTER(C.c_float)


# ag_host_collective_fn (include/accelgen_b200.h): (ctx, op, host_buf, count, dtype) -> 0 on success
HOST_COLLECTIVE_FN = C.CFUNCTYPE(i32, vp, i32, vp, i64, i32)
COLL_ALLREDUCE_SUM, COLL_ALLGATHER = 0, 1
DT_BF16, DT_F32, DT_I32 = 0, 1, 2


class ModelConfig(C.Structure):
    _fields_ = [("hidden", i32), ("num_layers", i32), ("num_heads", i32), ("ffn", i32), ("vocab", i32),
                ("pos_rows", i32), ("tp_rank", i32), ("tp_size", i32), ("num_blocks", i32),
                ("block_size", i32), ("max_tokens", i32), ("max_seqs", i32), ("max_blocks_per_seq", i32),
                ("ln_eps", f32)]


class LayerWeights(C.Structure):
    _fields_ = [(n, vp) for n in ("ln1_g", "ln1_b", "qkv_w", "qkv_b", "out_w", "out_b", "ln2_g", "ln2_b",
                                  "fc1_w", "fc1_b", "fc2_w", "fc2_b")]


class Step(C.Structure):
    _fields_ = [("num_tokens", i32), ("num_seqs", i32), ("num_logits", i32), ("block_table_stride", i32),
                ("token_ids", vp), ("positions", vp), ("cu_q", vp), ("ctx_len", vp), ("block_table", vp),
                ("slot_mapping", vp), ("logit_rows", vp)]


_SIGS = {
    "ag_last_error": (C.c_char_p, []),
    "ag_version": (i32, []),
    "ag_device_sm_count": (i32, []),
    "ag_model_create": (i32, [C.POINTER(ModelConfig), C.POINTER(vp)]),
    "ag_model_destroy": (None, [vp]),
    "ag_model_set_embeddings": (i32, [vp, vp, vp, vp, vp]),
    "ag_model_set_layer": (i32, [vp, i32, C.POINTER(LayerWeights)]),
    "ag_model_set_kv_cache": (i32, [vp, i32, vp, vp]),
    "ag_nccl_get_unique_id": (i32, [vp]),
    "ag_model_init_tp": (i32, [vp, vp]),
    "ag_model_init_tp_host": (i32, [vp, vp, vp]),
    "ag_model_forward": (i32, [vp, C.POINTER(Step), vp, vp, P_f32, vp]),
    "ag_model_submit": (i32, [vp, C.POINTER(Step), vp, i32, vp, vp]),
    "ag_model_wait": (i32, [vp, vp, i32, P_f32, C.POINTER(C.c_double)]),
    "ag_model_clock_ref": (i32, [vp, vp]),
    "ag_model_inflight": (i32, [vp]),
    "ag_model_stage_step": (i32, [vp, C.POINTER(Step), vp]),
    "ag_model_forward_staged": (i32, [vp, vp, vp, vp]),
    "ag_model_set_profiling": (i32, [vp, i32]),
    "ag_model_get_profile": (i32, [vp, vp, vp, vp, vp, i32]),
    "ag_model_set_roofline_peaks": (i32, [vp, f64, f64]),
    "ag_model_get_roofline_ms": (i32, [vp, vp, i32]),
    "ag_model_last_launches": (i64, [vp]),
    "ag_model_autotune": (i32, [vp, vp]),
    "ag_model_get_gemm_plans": (i32, [vp, vp, i32]),
    "ag_model_set_gemm_plans": (i32, [vp, vp, i32]),
    "ag_model_last_h2d_bytes": (i64, [vp]),
    "ag_gemm_bf16": (i32, [vp, i32, vp, i32, vp, vp, i32, i32, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, i64,
                           vp]),
    "ag_kv_append": (i32, [vp, vp, i32, vp, i32, i32, i32, vp, vp, vp]),
    "ag_paged_attention": (i32, [vp, i32, vp, vp, i32, vp, i32, vp, vp, vp, vp, i32, i32, i32, vp, i32, vp, i64, vp]),
    "ag_layernorm": (i32, [vp, vp, vp, vp, vp, vp, f32, i32, i32, vp, vp]),
    "ag_rmsnorm": (i32, [vp, vp, vp, f32, i32, i32, vp, vp]),
    "ag_rope": (i32, [vp, i32, vp, i32, i32, i32, i32, f32, vp]),
    "ag_embed_pos": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, vp]),
    "ag_argmax": (i32, [vp, i32, i32, i32, i32, vp, vp, vp]),
    "ag_kv_swap_out": (i32, [vp, vp, i32, i64, vp, vp]),
    "ag_kv_swap_in": (i32, [vp, vp, i32, i64, vp, vp]),
    "ag_kv_swap_out_planes": (i32, [vp, i64, vp, i32, i64, vp, i64, i32, vp]),
    "ag_kv_swap_in_planes": (i32, [vp, i64, vp, i32, i64, vp, i64, i32, vp]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def exported_symbols() -> list[str]:
    """Names the header declares (used by the CPU-side ABI test)."""
    return sorted(_SIGS)


def load() -> C.CDLL:
    """Load (once) and type the shared library; raises EngineFault if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise EngineFault(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == AG_OK:
        return
    msg = (load().ag_last_error() or b"").decode(errors="replace")
    if rc == AG_EINVAL:
        raise ValidationError(msg)
    if rc == AG_EALLOC:
        raise AllocationError(msg)
    if rc == AG_ESTATE:
        raise StateError(msg)
    raise EngineFault(f"device step failed (code {rc}): {msg}")
