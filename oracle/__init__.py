"""ctypes front end of the fp64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this package. It restates the reference `actplan` seqpar harness
(/root/reference/proj/core/src/seqpar/*.cpp, activation_memory.cpp) — see oracle/oracle.h for
the file:line map and for how it is pinned (RNG bit-exact vs the compiled reference rng.cpp,
accountant vs the reference tests' known answers, layer numerics by the reference's own
relational verify suites).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

NPARAM_NAMES = ["wq", "wk", "wv", "bq", "bk", "bv", "wo", "bo", "w1", "b1", "w2", "b2",
                "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"]
LEDGER_NAMES = ["ln1_input", "qkv_input", "query", "key", "value", "softmax_out",
                "softmax_dropout_mask", "softmax_dropout_out", "attn_proj_input",
                "attn_dropout_mask", "ln2_input", "mlp_fc1_input", "gelu_input",
                "mlp_fc2_input", "mlp_dropout_mask"]
KIND = {"none": 0, "full": 1, "selective": 2}


class OracleError(RuntimeError):
    pass


class CBlockCfg(C.Structure):
    _fields_ = [("heads", C.c_int64), ("hidden", C.c_int64), ("seq", C.c_int64),
                ("batch", C.c_int64), ("dropout_p", C.c_double), ("causal", C.c_int32),
                ("seed", C.c_uint64), ("layer_index", C.c_uint32), ("microbatch", C.c_uint32),
                ("ln_eps", C.c_double)]


class CCounters(C.Structure):
    _fields_ = [("all_gathers", C.c_int64), ("reduce_scatters", C.c_int64),
                ("all_reduces", C.c_int64), ("ring_elements", C.c_int64)]


class CCommLog(C.Structure):
    _fields_ = [("schedule", CCounters), ("regather", CCounters), ("grad_sync", CCounters)]


class CLedger(C.Structure):
    _fields_ = [("elements", C.c_int64 * 15), ("bytes", C.c_int64 * 15)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        u64, i64, dbl, i32, u32 = C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_uint32
        pd = C.POINTER(C.c_double)
        L.orc_mix64.restype = u64; L.orc_mix64.argtypes = [u64]
        L.orc_hash_counter.restype = u64; L.orc_hash_counter.argtypes = [u64, u64]
        L.orc_uniform01.restype = dbl; L.orc_uniform01.argtypes = [u64, u64]
        L.orc_mask_key_fold.restype = u64; L.orc_mask_key_fold.argtypes = [u64, u32, u32, u32]
        L.orc_random_uniform.argtypes = [u64, i64, dbl, dbl, pd]
        L.orc_dropout_mask.restype = i32; L.orc_dropout_mask.argtypes = [u64, i64, dbl, pd]
        L.orc_param_layout.restype = i64
        L.orc_param_layout.argtypes = [i64, C.POINTER(i64), C.POINTER(i64)]
        L.orc_params_random.argtypes = [i64, u64, pd]
        L.orc_params_zeros.argtypes = [i64, pd]
        L.orc_layer_norm.argtypes = [pd, i64, i64, pd, pd, dbl, pd, pd, pd]
        L.orc_attention_interior.restype = i32
        L.orc_attention_interior.argtypes = [C.POINTER(CBlockCfg), pd, pd, i64, i64, pd, pd, pd]
        L.orc_seqpar_layer.restype = i32
        L.orc_seqpar_layer.argtypes = [C.POINTER(CBlockCfg), i64, pd, pd, pd, pd, pd, pd, pd, pd,
                                       C.POINTER(CCommLog), C.POINTER(CCommLog), C.POINTER(CLedger)]
        L.orc_reference_layer.restype = i32
        L.orc_reference_layer.argtypes = [C.POINTER(CBlockCfg), pd, pd, pd, pd, pd, pd, pd, pd, pd,
                                          C.POINTER(CLedger)]
        L.orc_last_error.restype = C.c_char_p
        L.orc_set_threads.restype = i32; L.orc_set_threads.argtypes = [i32]
        L.orc_per_layer_bytes.restype = i32
        L.orc_per_layer_bytes.argtypes = [i64, i64, i64, i64, i64, i32, i32, i64, i64, C.POINTER(i64)]
        L.orc_per_layer_bytes_exact.restype = i32
        L.orc_per_layer_bytes_exact.argtypes = [i64, i64, i64, i64, i64, i32, i32, i64, i64,
                                                C.POINTER(i64), C.POINTER(i64)]
        L.orc_layer_component_breakdown.restype = i32
        L.orc_layer_component_breakdown.argtypes = [i64, i64, i64, i64, i64, i64, C.POINTER(i64)]
        L.orc_percent_of_baseline.restype = i32
        L.orc_percent_of_baseline.argtypes = [i64, i64, i64, i64, i64, i32, i32, i64, i64,
                                              C.POINTER(i64), C.POINTER(i64)]
        L.orc_total_first_stage_bytes.restype = i32
        L.orc_total_first_stage_bytes.argtypes = [i64, i64, i64, i64, i64, i32, i32, i64, i64,
                                                  i64, i64, i64, C.POINTER(i64)]
        L.orc_layer_comm_bytes_tp.restype = i64
        L.orc_layer_comm_bytes_tp.argtypes = [i64, i64, i64, i64, i64]
        L.orc_layer_comm_bytes_sp.restype = i64
        L.orc_layer_comm_bytes_sp.argtypes = [i64, i64, i64, i64, i64]
        _LIB = L
    return _LIB


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class BlockConfig:
    """Mirror of actplan::seqpar::BlockConfig (block.hpp:28-42)."""
    heads: int
    hidden: int
    seq: int
    batch: int
    dropout_p: float = 0.0
    causal: bool = False
    seed: int = 42
    layer_index: int = 0
    microbatch: int = 1
    layer_norm_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def c(self) -> CBlockCfg:
        return CBlockCfg(self.heads, self.hidden, self.seq, self.batch, self.dropout_p,
                         int(self.causal), self.seed, self.layer_index, self.microbatch,
                         self.layer_norm_eps)


# ---------------------------------------------------------------- rng (rng.cpp)
def mix64(x: int) -> int:
    return lib().orc_mix64(x)


def hash_counter(key: int, index: int) -> int:
    return lib().orc_hash_counter(key, index)


def uniform01(key: int, index: int) -> float:
    return lib().orc_uniform01(key, index)


def mask_key_fold(seed: int, layer: int, op: int, microbatch: int) -> int:
    return lib().orc_mask_key_fold(seed, layer, op, microbatch)


def random_uniform(key: int, shape, lo: float, hi: float) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, np.float64)
    lib().orc_random_uniform(key, n, lo, hi, _p(out))
    return out.reshape(shape)


def dropout_mask(folded_key: int, n: int, p: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    if lib().orc_dropout_mask(folded_key, n, p, _p(out)):
        raise ValueError("dropout probability must lie in [0, 1)")
    return out


# ---------------------------------------------------------------- params
def param_layout(h: int):
    off = (C.c_int64 * 16)()
    sz = (C.c_int64 * 16)()
    total = lib().orc_param_layout(h, off, sz)
    return list(off), list(sz), total


def param_shapes(h: int):
    return {"wq": (h, h), "wk": (h, h), "wv": (h, h), "bq": (h,), "bk": (h,), "bv": (h,),
            "wo": (h, h), "bo": (h,), "w1": (h, 4 * h), "b1": (4 * h,), "w2": (4 * h, h),
            "b2": (h,), "ln1_gain": (h,), "ln1_bias": (h,), "ln2_gain": (h,), "ln2_bias": (h,)}


def params_random(h: int, seed: int) -> np.ndarray:
    _, _, total = param_layout(h)
    out = np.empty(total, np.float64)
    lib().orc_params_random(h, seed, _p(out))
    return out


def params_zeros(h: int) -> np.ndarray:
    _, _, total = param_layout(h)
    out = np.empty(total, np.float64)
    lib().orc_params_zeros(h, _p(out))
    return out


def unpack(h: int, packed: np.ndarray) -> dict:
    off, sz, _ = param_layout(h)
    shapes = param_shapes(h)
    return {n: packed[off[i]:off[i] + sz[i]].reshape(shapes[n]) for i, n in enumerate(NPARAM_NAMES)}


def _check(rc: int):
    if rc == 1:
        raise ValueError(lib().orc_last_error().decode())
    if rc == 2:
        raise ArithmeticError(lib().orc_last_error().decode())
    if rc:
        raise OracleError(f"oracle rc={rc}")


# ---------------------------------------------------------------- layer
@dataclass
class LayerResult:
    y: np.ndarray
    dx: np.ndarray | None
    grads: np.ndarray | None
    w1_grad_shards: np.ndarray | None
    interior: np.ndarray | None
    fwd_comm: CCommLog
    bwd_comm: CCommLog
    ledgers: list


def seqpar_layer(cfg: BlockConfig, t: int, params: np.ndarray, x: np.ndarray,
                 dy: np.ndarray | None = None, want_interior: bool = False) -> LayerResult:
    s, b, h, a = cfg.seq, cfg.batch, cfg.hidden, cfg.heads
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty((s, b, h), np.float64)
    dx = np.empty((s, b, h), np.float64) if dy is not None else None
    grads = np.empty_like(params) if dy is not None else None
    w1s = np.empty((t, h, 4 * h // t), np.float64) if dy is not None else None
    interior = np.empty((3, a, b, s, s), np.float64) if want_interior else None
    fl, bl = CCommLog(), CCommLog()
    led = (CLedger * max(t, 1))()
    dyc = np.ascontiguousarray(dy, np.float64) if dy is not None else None
    rc = lib().orc_seqpar_layer(C.byref(cfg.c()), t, _p(params), _p(x), _p(dyc), _p(y), _p(dx),
                                _p(grads), _p(w1s), _p(interior), C.byref(fl), C.byref(bl), led)
    _check(rc)
    ledgers = [{n: (led[r].elements[i], led[r].bytes[i]) for i, n in enumerate(LEDGER_NAMES)}
               for r in range(t)]
    return LayerResult(y, dx, grads, w1s, interior, fl, bl, ledgers)


def reference_layer(cfg: BlockConfig, params: np.ndarray, x: np.ndarray,
                    dy: np.ndarray | None = None, want_interior: bool = False):
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
    rc = lib().orc_reference_layer(C.byref(cfg.c()), _p(params), _p(x), _p(dyc), _p(y), _p(dx),
                                   _p(grads), _p(q), _p(k), _p(interior), C.byref(led))
    _check(rc)
    ledger = {n: (led.elements[i], led.bytes[i]) for i, n in enumerate(LEDGER_NAMES)}
    return dict(y=y, dx=dx, grads=grads, q=q, k=k, interior=interior, ledger=ledger)


def attention_interior(cfg: BlockConfig, q: np.ndarray, k: np.ndarray, head_offset: int,
                       local_heads: int) -> np.ndarray:
    s, b = cfg.seq, cfg.batch
    out = np.empty((3, local_heads, b, s, s))
    qc = np.ascontiguousarray(q, np.float64)
    kc = np.ascontiguousarray(k, np.float64)
    rc = lib().orc_attention_interior(C.byref(cfg.c()), _p(qc), _p(kc), head_offset, local_heads,
                                      _p(out[0]), _p(out[1]), _p(out[2]))
    _check(rc)
    return out


def set_threads(n: int) -> int:
    return lib().orc_set_threads(n)


# ---------------------------------------------------------------- accountant
def per_layer_bytes(a, h, s, b, t, kind, sequence_parallel, act=2, mask=1) -> int:
    out = C.c_int64()
    rc = lib().orc_per_layer_bytes(a, h, s, b, t, KIND.get(kind, kind), int(sequence_parallel),
                                   act, mask, C.byref(out))
    if rc:
        raise ValueError("invalid configuration")
    return out.value


def per_layer_bytes_exact(a, h, s, b, t, kind, sequence_parallel, act=2, mask=1):
    n, d = C.c_int64(), C.c_int64()
    rc = lib().orc_per_layer_bytes_exact(a, h, s, b, t, KIND.get(kind, kind), int(sequence_parallel),
                                         act, mask, C.byref(n), C.byref(d))
    if rc:
        raise ValueError("invalid configuration")
    return n.value, d.value


def layer_component_breakdown(a, h, s, b, act=2, mask=1):
    out = (C.c_int64 * 4)()
    if lib().orc_layer_component_breakdown(a, h, s, b, act, mask, out):
        raise ValueError("invalid configuration")
    return dict(attention=out[0], mlp=out[1], layer_norms=out[2], total=out[3])


def percent_of_baseline(a, h, s, b, t, kind, sequence_parallel, act=2, mask=1):
    n, d = C.c_int64(), C.c_int64()
    rc = lib().orc_percent_of_baseline(a, h, s, b, t, KIND.get(kind, kind), int(sequence_parallel),
                                       act, mask, C.byref(n), C.byref(d))
    if rc:
        raise ValueError("invalid configuration")
    return n.value, d.value


def total_first_stage_bytes(a, h, s, b, t, kind, sequence_parallel, layers, pipeline=1,
                            interleave=1, act=2, mask=1):
    out = C.c_int64()
    rc = lib().orc_total_first_stage_bytes(a, h, s, b, t, KIND.get(kind, kind),
                                           int(sequence_parallel), layers, pipeline, interleave,
                                           act, mask, C.byref(out))
    if rc:
        raise ValueError("invalid configuration")
    return out.value


def layer_comm_bytes_tp(s, b, h, t, elem=2):
    return lib().orc_layer_comm_bytes_tp(s, b, h, t, elem)


def layer_comm_bytes_sp(s, b, h, t, elem=2):
    return lib().orc_layer_comm_bytes_sp(s, b, h, t, elem)
