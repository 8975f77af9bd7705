"""ctypes front end of the reference's OWN seqpar harness (TEST INFRASTRUCTURE ONLY).

oracle/_ref/libref_seqpar.so is /root/reference/proj/core/src/seqpar/{tensor,block,collectives,
rng}.cpp compiled unmodified (oracle/Makefile `ref`, Eigen/Boost stand-ins in oracle/shim/) plus
the C entry layer oracle/ref_seqpar_shim.cpp. The library is built here, where /root/reference
exists, and travels to the GPU box with the snapshot (git-ignored, not gpurun-ignored). Callers
must treat it as optional: `available()` is False when it was not built.

Same calling conventions as the restatement in oracle/__init__.py, so the two can be compared
entry point by entry point.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import (BlockConfig, CCommLog, CLedger, LEDGER_NAMES, LayerResult, OracleError,
               param_layout)

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libref_seqpar.so")
_LIB = None


def available() -> bool:
    return os.path.exists(PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise OracleError(f"{PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(PATH)
        i64, u64, dbl, i32 = C.c_int64, C.c_uint64, C.c_double, C.c_int
        pd = C.POINTER(C.c_double)
        pi = C.POINTER(C.c_int64)
        L.ref_last_error.restype = C.c_char_p
        L.ref_params_random.restype = i32
        L.ref_params_random.argtypes = [i64, u64, pd]
        L.ref_random_uniform2.argtypes = [u64, i64, dbl, dbl, pd]
        L.ref_hash_counter2.restype = u64
        L.ref_hash_counter2.argtypes = [u64, u64]
        L.ref_seqpar_layer.restype = i32
        L.ref_seqpar_layer.argtypes = [C.c_void_p, i64, pd, pd, pd, pd, pd, pd, pd, pd,
                                       C.POINTER(CCommLog), C.POINTER(CCommLog), C.POINTER(CLedger)]
        L.ref_reference_layer.restype = i32
        L.ref_reference_layer.argtypes = [C.c_void_p, pd, pd, pd, pd, pd, pd, pd, pd, pd,
                                          C.POINTER(CLedger)]
        L.ref_attention_interior.restype = i32
        L.ref_attention_interior.argtypes = [C.c_void_p, pd, pd, i64, i64, pd, pd, pd]
        L.ref_all_gather.restype = i32
        L.ref_all_gather.argtypes = [pd, i64, pi, i64, i64, pd, C.POINTER(CCommLog), i32]
        L.ref_reduce_scatter.restype = i32
        L.ref_reduce_scatter.argtypes = [pd, i64, pi, i64, i64, pd, C.POINTER(CCommLog), i32]
        L.ref_all_reduce.restype = i32
        L.ref_all_reduce.argtypes = [pd, i64, pi, i64, pd, C.POINTER(CCommLog), i32]
        L.ref_layer_comm_bytes_tp.restype = i64
        L.ref_layer_comm_bytes_tp.argtypes = [i64] * 5
        L.ref_layer_comm_bytes_sp.restype = i64
        L.ref_layer_comm_bytes_sp.argtypes = [i64] * 5
        _LIB = L
    return _LIB


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc: int):
    if rc == 1:
        raise ValueError(lib().ref_last_error().decode())
    if rc == 2:
        raise ArithmeticError(lib().ref_last_error().decode())
    if rc:
        raise OracleError(f"reference rc={rc}: {lib().ref_last_error().decode()}")


def params_random(h: int, seed: int) -> np.ndarray:
    """LayerParams::random (block.cpp:234-265), packed in named_tensors() order."""
    _, _, total = param_layout(h)
    out = np.empty(total, np.float64)
    _check(lib().ref_params_random(h, seed, _p(out)))
    return out


def random_uniform(key: int, shape, lo: float, hi: float) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, np.float64)
    lib().ref_random_uniform2(key, n, lo, hi, _p(out))
    return out.reshape(shape)


def hash_counter(key: int, index: int) -> int:
    return lib().ref_hash_counter2(key, index)


def seqpar_layer(cfg: BlockConfig, t: int, params: np.ndarray, x: np.ndarray,
                 dy: np.ndarray | None = None, want_interior: bool = False) -> LayerResult:
    """seqpar_block_forward + seqpar_block_backward (block.cpp:512-749) of the reference."""
    s, b, h, a = cfg.seq, cfg.batch, cfg.hidden, cfg.heads
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty((s, b, h))
    dx = np.empty((s, b, h)) if dy is not None else None
    grads = np.empty_like(params) if dy is not None else None
    w1s = np.empty((t, h, 4 * h // t)) if dy is not None else None
    interior = np.empty((3, a, b, s, s)) if want_interior else None
    fl, bl = CCommLog(), CCommLog()
    led = (CLedger * max(t, 1))()
    dyc = np.ascontiguousarray(dy, np.float64) if dy is not None else None
    cc = cfg.c()
    rc = lib().ref_seqpar_layer(C.addressof(cc), t, _p(params), _p(x), _p(dyc), _p(y), _p(dx),
                                _p(grads), _p(w1s), _p(interior), C.byref(fl), C.byref(bl), led)
    _check(rc)
    ledgers = [{n: (led[r].elements[i], led[r].bytes[i]) for i, n in enumerate(LEDGER_NAMES)}
               for r in range(t)]
    return LayerResult(y, dx, grads, w1s, interior, fl, bl, ledgers)


def reference_layer(cfg: BlockConfig, params: np.ndarray, x: np.ndarray,
                    dy: np.ndarray | None = None, want_interior: bool = False):
    """reference_block_forward / reference_block_backward (block.cpp:419-510)."""
    s, b, h, a = cfg.seq, cfg.batch, cfg.hidden, cfg.heads
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty((s, b, h))
    dx = np.empty((s, b, h)) if dy is not None else None
    grads = np.empty_like(params) if dy is not None else None
    q = np.empty((s, b, h))
    k = np.empty((s, b, h))
    interior = np.empty((3, a, b, s, s)) if want_interior else None
    led = CLedger()
    dyc = np.ascontiguousarray(dy, np.float64) if dy is not None else None
    cc = cfg.c()
    rc = lib().ref_reference_layer(C.addressof(cc), _p(params), _p(x), _p(dyc), _p(y), _p(dx),
                                   _p(grads), _p(q), _p(k), _p(interior), C.byref(led))
    _check(rc)
    ledger = {n: (led.elements[i], led.bytes[i]) for i, n in enumerate(LEDGER_NAMES)}
    return dict(y=y, dx=dx, grads=grads, q=q, k=k, interior=interior, ledger=ledger)


def attention_interior(cfg: BlockConfig, q: np.ndarray, k: np.ndarray, head_offset: int,
                       local_heads: int) -> np.ndarray:
    """attention_interior (block.cpp:381-417) -> {3, local_heads, b, s, s}."""
    s, b = cfg.seq, cfg.batch
    out = np.empty((3, local_heads, b, s, s))
    qc = np.ascontiguousarray(q, np.float64)
    kc = np.ascontiguousarray(k, np.float64)
    cc = cfg.c()
    _check(lib().ref_attention_interior(C.addressof(cc), _p(qc), _p(kc), head_offset, local_heads,
                                        _p(out[0]), _p(out[1]), _p(out[2])))
    return out


def _shape_arr(shape):
    arr = (C.c_int64 * len(shape))(*shape)
    return arr


def all_gather(shards: np.ndarray, axis: int, tag: int = 0):
    """all_gather (collectives.cpp:40-46) over shards[t, *shape]."""
    shards = np.ascontiguousarray(shards, np.float64)
    t, shape = shards.shape[0], list(shards.shape[1:])
    out_shape = list(shape)
    out_shape[axis] *= t
    out = np.empty(out_shape)
    log = CCommLog()
    _check(lib().ref_all_gather(_p(shards), t, _shape_arr(shape), len(shape), axis, _p(out),
                                C.byref(log), tag))
    return out, log


def reduce_scatter(partials: np.ndarray, axis: int, tag: int = 0):
    """reduce_scatter (collectives.cpp:48-57) -> [t, *piece_shape]."""
    partials = np.ascontiguousarray(partials, np.float64)
    t, shape = partials.shape[0], list(partials.shape[1:])
    piece = list(shape)
    piece[axis] //= t
    out = np.empty([t] + piece)
    log = CCommLog()
    _check(lib().ref_reduce_scatter(_p(partials), t, _shape_arr(shape), len(shape), axis, _p(out),
                                    C.byref(log), tag))
    return out, log


def all_reduce(partials: np.ndarray, tag: int = 0):
    """all_reduce (collectives.cpp:59-65)."""
    partials = np.ascontiguousarray(partials, np.float64)
    t, shape = partials.shape[0], list(partials.shape[1:])
    out = np.empty(shape)
    log = CCommLog()
    _check(lib().ref_all_reduce(_p(partials), t, _shape_arr(shape), len(shape), _p(out),
                                C.byref(log), tag))
    return out, log


def layer_comm_bytes_tp(s, b, h, t, elem=2):
    return lib().ref_layer_comm_bytes_tp(s, b, h, t, elem)


def layer_comm_bytes_sp(s, b, h, t, elem=2):
    return lib().ref_layer_comm_bytes_sp(s, b, h, t, elem)
