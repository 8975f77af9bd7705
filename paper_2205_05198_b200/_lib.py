"""ctypes binding of libspl.so (include/spl.h). Fails loudly when the library is missing —
there is no CPU fallback for the layer."""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspl.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "spl.h")

SPL_OK, SPL_EINVAL, SPL_EDOMAIN, SPL_ECUDA, SPL_ENCCL, SPL_ESTATE, SPL_EBUDGET = range(7)
RECOMPUTE = {"none": 0, "full": 1, "selective": 2}
DTYPE = {"f32": 0, "fp32": 0, "float32": 0, "bf16": 1, "bfloat16": 1}
DTYPE_F64 = 2  # collectives only
KCLASS = ["gemm", "attention", "elementwise", "collective", "other"]


class SplError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class SplStateError(SplError, ValueError):
    """Backward without a matching forward (the reference raises std::invalid_argument)."""


class LayerDesc(C.Structure):
    _fields_ = [("heads", C.c_int64), ("hidden", C.c_int64), ("seq", C.c_int64),
                ("batch", C.c_int64), ("dropout_p", C.c_double), ("causal", C.c_int32),
                ("seed", C.c_uint64), ("layer_index", C.c_uint32), ("microbatch", C.c_uint32),
                ("ln_eps", C.c_double), ("recompute", C.c_int32),
                ("sequence_parallel", C.c_int32), ("dtype", C.c_int32),
                ("check_finite", C.c_int32), ("act_bytes", C.c_int64), ("mask_bytes", C.c_int64)]


class ModelDesc(C.Structure):
    _fields_ = [("heads", C.c_int64), ("hidden", C.c_int64), ("layers", C.c_int64),
                ("seq", C.c_int64), ("vocab", C.c_int64), ("tensor", C.c_int64),
                ("pipeline", C.c_int64), ("interleave", C.c_int64), ("microbatch", C.c_int64),
                ("microbatches", C.c_int64), ("recompute", C.c_int32),
                ("sequence_parallel", C.c_int32), ("act_bytes", C.c_int64),
                ("mask_bytes", C.c_int64), ("logits_bytes", C.c_int64)]


class LedgerEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("elements", C.c_int64), ("bytes", C.c_int64),
                ("physical_bytes", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -j` (python -c "
                          "'import __graft_entry__; __graft_entry__.build()')")
    L = C.CDLL(LIB_PATH)
    H, P, VP, I64, I32, D = C.c_void_p, C.POINTER, C.c_void_p, C.c_int64, C.c_int, C.c_double
    sig = {
        "spl_desc_default": (None, [P(LayerDesc)]),
        "spl_create_local": (I32, [P(LayerDesc), I32, I32, P(H)]),
        "spl_create": (I32, [P(LayerDesc), P(I32), I32, P(H)]),
        "spl_nccl_unique_id": (I32, [C.c_char_p]),
        "spl_create_nccl": (I32, [P(LayerDesc), I32, I32, I32, C.c_char_p, P(H)]),
        "spl_ipc_open": (I32, [P(LayerDesc), I32, I32, I32, P(H), C.c_char_p]),
        "spl_create_ipc": (I32, [P(LayerDesc), H, C.c_char_p, P(H)]),
        "spl_ipc_close": (I32, [H]),
        "spl_destroy": (I32, [H]),
        "spl_local_ranks": (I32, [H]),
        "spl_last_error": (C.c_char_p, []),
        "spl_set_stream": (I32, [H, VP]),
        "spl_load_params": (I32, [H, P(D)]),
        "spl_init_params": (I32, [H, C.c_uint64]),
        "spl_forward": (I32, [H, P(VP), P(VP)]),
        "spl_backward": (I32, [H, P(VP), P(VP)]),
        "spl_step_host": (I32, [H, VP, VP, VP, VP]),
        "spl_step_host_async": (I32, [H, VP, VP, VP, VP]),
        "spl_step_host_wait": (I32, [H]),
        "spl_get_grads": (I32, [H, P(D)]),
        "spl_get_w1_grad_shard": (I32, [H, I32, P(D)]),
        "spl_get_saved": (I32, [H, I32, C.c_char_p, P(D), I64]),
        "spl_attention_interior": (I32, [H, I32, P(D)]),
        "spl_ledger": (I32, [H, I32, P(LedgerEntry), P(I32)]),
        "spl_saved_bytes": (I32, [H, I32, P(I64), P(I64), P(I64)]),
        "spl_comm_log": (I32, [H, P(I64)]),
        "spl_comm_log_reset": (I32, [H]),
        "spl_per_layer_bytes": (I32, [I64, I64, I64, I64, I64, I32, I32, I64, I64, P(I64)]),
        "spl_per_layer_bytes_exact": (I32, [I64, I64, I64, I64, I64, I32, I32, I64, I64, P(I64), P(I64)]),
        "spl_timer_start": (I32, [H]),
        "spl_timer_stop": (I32, [H, P(C.c_float)]),
        "spl_synchronize": (I32, [H]),
        "spl_profile_enable": (I32, [H, I32]),
        "spl_profile_read": (I32, [H, P(D), P(I64), P(D), P(D)]),
        "spl_launch_count": (I32, [H, P(I64), I32]),
        "spl_comm_paths": (I32, [H, P(I32)]),
        "spl_set_graphs": (I32, [H, I32]),
        "spl_layer_component_breakdown": (I32, [I64, I64, I64, I64, I64, I64, P(I64)]),
        "spl_percent_of_baseline": (I32, [I64, I64, I64, I64, I64, I32, I32, I64, I64, P(I64), P(I64)]),
        "spl_total_first_stage_bytes": (I32, [I64, I64, I64, I64, I64, I32, I32, I64, I64, I64,
                                              I64, I64, P(I64)]),
        "spl_layer_comm_bytes": (I32, [I64, I64, I64, I64, I64, I32, P(I64)]),
        "spl_stack_create_local": (I32, [P(LayerDesc), I32, I32, I32, P(H)]),
        "spl_stack_destroy": (I32, [H]),
        "spl_stack_layers": (I32, [H]),
        "spl_stack_layer": (I32, [H, I32, P(H)]),
        "spl_stack_set_stream": (I32, [H, VP]),
        "spl_stack_forward": (I32, [H, P(VP), P(VP)]),
        "spl_stack_backward": (I32, [H, P(VP), P(VP)]),
        "spl_stack_memory": (I32, [H, I32, P(I64)]),
        "spl_model_desc_default": (None, [P(ModelDesc)]),
        "spl_microbatch_bytes": (I32, [P(ModelDesc), I64, P(I64), P(I64)]),
        "spl_window_plan": (I32, [P(ModelDesc), I64, P(C.c_uint8), P(I64), P(I64), P(I64), P(I64)]),
        "spl_stage_timeline": (I32, [P(ModelDesc), I64, P(C.c_uint8), I32, P(I64), I64, P(I64),
                                     P(I64)]),
        "spl_window_create_local": (I32, [P(LayerDesc), I32, I32, I32, I64, I64, I64,
                                          P(C.c_uint8), P(H)]),
        "spl_window_destroy": (I32, [H]),
        "spl_window_layer": (I32, [H, I32, P(H)]),
        "spl_window_set_stream": (I32, [H, VP]),
        "spl_window_run": (I32, [H, P(VP), P(VP), P(VP), P(VP)]),
        "spl_window_memory": (I32, [H, P(I64)]),
        "spl_attention_interior_qk": (I32, [P(LayerDesc), I32, VP, VP, I64, I64, VP, VP, VP, VP]),
        "spl_all_gather": (I32, [P(VP), I32, P(I64), I32, I32, I32, VP, P(I64), I32, VP]),
        "spl_reduce_scatter": (I32, [P(VP), I32, P(I64), I32, I32, I32, P(VP), P(I64), I32, VP]),
        "spl_all_reduce": (I32, [P(VP), I32, P(I64), I32, I32, VP, P(I64), I32, VP]),
        "spl_gemm_bf16": (I32, [I64, I64, I64, VP, I64, I32, VP, I64, I32, VP, I64, I32, VP, VP,
                                VP, I64, VP, P(I32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def header_symbols() -> list[str]:
    """Every function the C ABI header declares."""
    text = re.sub(r"/\*.*?\*/|//[^\n]*", "", open(HEADER).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(spl_[a-z0-9_]+)\s*\(", text)))


def check(rc: int):
    if rc == SPL_OK:
        return
    msg = lib().spl_last_error().decode(errors="replace")
    if rc == SPL_EINVAL:
        raise ValueError(msg)
    if rc == SPL_EDOMAIN:
        raise ArithmeticError(msg)
    if rc == SPL_ESTATE:
        raise SplStateError(rc, msg)
    raise SplError(rc, msg)
