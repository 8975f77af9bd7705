"""Python mirror of the reference's seqpar layer API over the C ABI (include/spl.h).

Reference interface (/root/reference/proj/core/include/actplan/seqpar/block.hpp):
  BlockConfig (28-42), seqpar_block_forward (158-162), seqpar_block_backward (173-174),
  SeqparForward (136-154), SeqparBackward (164-171), ActivationLedger (61-73),
  CommLog (collectives.hpp:28-52), per_layer_bytes (activation_memory.hpp:83-84).
Same names, argument meaning and error classes: std::invalid_argument -> ValueError,
std::domain_error -> ArithmeticError. Host tensors are fp64 numpy arrays in the reference
layouts ({s,b,h}; params packed in LayerParams::named_tensors() order); the layer itself runs
on the GPU in the chosen dtype, device memory held as torch tensors (plumbing only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

PARAM_NAMES = ["wq", "wk", "wv", "bq", "bk", "bv", "wo", "bo", "w1", "b1", "w2", "b2",
               "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"]


@dataclass
class BlockConfig:
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
    act_bytes: int = 2
    mask_bytes: int = 1

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def param_count(h: int) -> int:
    return 12 * h * h + 13 * h


def _torch():
    import torch
    return torch


def _tdtype(dtype: str):
    torch = _torch()
    return torch.float32 if _lib.DTYPE[dtype] == 0 else torch.bfloat16


def _desc(cfg: BlockConfig, recompute: str, sequence_parallel: bool, dtype: str,
          check_finite: bool) -> "_lib.LayerDesc":
    d = _lib.LayerDesc()
    lib().spl_desc_default(C.byref(d))
    d.heads, d.hidden, d.seq, d.batch = cfg.heads, cfg.hidden, cfg.seq, cfg.batch
    d.dropout_p, d.causal, d.seed = cfg.dropout_p, int(cfg.causal), cfg.seed
    d.layer_index, d.microbatch, d.ln_eps = cfg.layer_index, cfg.microbatch, cfg.layer_norm_eps
    d.recompute = _lib.RECOMPUTE[recompute]
    d.sequence_parallel = int(sequence_parallel)
    d.dtype = _lib.DTYPE[dtype]
    d.check_finite = int(check_finite)
    d.act_bytes, d.mask_bytes = cfg.act_bytes, cfg.mask_bytes
    return d


class SeqparLayer:
    """One layer handle: t simulated ranks on one GPU (nccl=None), or one rank of an NCCL
    group (nccl=(rank, unique_id_bytes))."""

    def __init__(self, cfg: BlockConfig, t: int, recompute: str = "none",
                 sequence_parallel: bool = True, dtype: str = "bf16", device: int = 0,
                 check_finite: bool = True, nccl: tuple[int, bytes] | None = None,
                 _borrow=None, ipc=None):
        self.cfg, self.t, self.recompute, self.sp, self.dtype = cfg, t, recompute, sequence_parallel, dtype
        self.device = device
        self._owned = True
        if _borrow is not None:  # a layer of a SeqparStack: the stack owns the handle
            self._h, self._owned = _borrow, False
            self.local = lib().spl_local_ranks(self._h)
            self.rank0 = 0
            return
        d = _desc(cfg, recompute, sequence_parallel, dtype, check_finite)
        self._h = C.c_void_p()
        if ipc is not None:
            # one rank of a CUDA-IPC group: ipc = (rank, exchange) where exchange(handle_bytes)
            # returns the t ranks' handles in rank order (any host transport, e.g. gloo)
            rank, exchange = ipc
            obj = C.c_void_p()
            hb = C.create_string_buffer(64)
            check(lib().spl_ipc_open(C.byref(d), device, t, rank, C.byref(obj), hb))
            handles = b"".join(exchange(hb.raw[:64]))
            check(lib().spl_create_ipc(C.byref(d), obj, handles, C.byref(self._h)))
        elif nccl is None:
            check(lib().spl_create_local(C.byref(d), device, t, C.byref(self._h)))
        else:
            rank, uid = nccl
            check(lib().spl_create_nccl(C.byref(d), device, t, rank, uid, C.byref(self._h)))
        self.local = lib().spl_local_ranks(self._h)
        self.rank0 = nccl[0] if nccl is not None else (ipc[0] if ipc is not None else 0)

    # ---- lifecycle
    def close(self):
        if self._h and self._owned:
            lib().spl_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().spl_nccl_unique_id(buf))
        return buf.raw

    # ---- shapes
    @property
    def shard_rows(self) -> int:
        c = self.cfg
        return (c.seq // self.t if self.sp else c.seq)

    def shard_shape(self):
        return (self.shard_rows, self.cfg.batch, self.cfg.hidden)

    # ---- params
    def load_params(self, packed: np.ndarray):
        p = np.ascontiguousarray(packed, np.float64)
        assert p.size == param_count(self.cfg.hidden)
        check(lib().spl_load_params(self._h, p.ctypes.data_as(C.POINTER(C.c_double))))

    def init_params(self, seed: int):
        check(lib().spl_init_params(self._h, seed))

    # ---- compute (device tensors)
    def _bind_stream(self):
        torch = _torch()
        check(lib().spl_set_stream(self._h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def forward(self, x: list, y: list | None = None) -> list:
        torch = _torch()
        self._bind_stream()
        if len(x) != self.local:
            raise ValueError("expected one input shard per rank")
        for xi in x:
            if tuple(xi.shape) != self.shard_shape() or xi.dtype != _tdtype(self.dtype):
                raise ValueError(f"input shard must be {self.shard_shape()} {self.dtype}")
        if y is None:
            y = [torch.empty_like(xi) for xi in x]
        xs = (C.c_void_p * self.local)(*[xi.data_ptr() for xi in x])
        ys = (C.c_void_p * self.local)(*[yi.data_ptr() for yi in y])
        check(lib().spl_forward(self._h, xs, ys))
        return y

    def backward(self, dy: list, dx: list | None = None) -> list:
        torch = _torch()
        self._bind_stream()
        if len(dy) != self.local:
            raise ValueError("expected one gradient shard per rank")
        for di in dy:
            if tuple(di.shape) != self.shard_shape() or di.dtype != _tdtype(self.dtype):
                raise ValueError("dy shard shape mismatch")
        if dx is None:
            dx = [torch.empty_like(di) for di in dy]
        ds = (C.c_void_p * self.local)(*[di.data_ptr() for di in dy])
        xs = (C.c_void_p * self.local)(*[xi.data_ptr() for xi in dx])
        check(lib().spl_backward(self._h, ds, xs))
        return dx

    def step_host(self, x_host, dy_host, y_host, dx_host):
        check(lib().spl_step_host(self._h, x_host.data_ptr(), dy_host.data_ptr(),
                                  y_host.data_ptr(), dx_host.data_ptr()))

    def step_host_async(self, x_host, dy_host, y_host, dx_host):
        """Issue one host-buffer step (spl_step_host_async); buffers stay in use until
        step_host_wait()."""
        check(lib().spl_step_host_async(self._h, x_host.data_ptr(), dy_host.data_ptr(),
                                        y_host.data_ptr(), dx_host.data_ptr()))

    def step_host_wait(self):
        check(lib().spl_step_host_wait(self._h))

    # ---- read-back
    def grads(self) -> np.ndarray:
        out = np.empty(param_count(self.cfg.hidden), np.float64)
        check(lib().spl_get_grads(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def w1_grad_shard(self, r: int) -> np.ndarray:
        h = self.cfg.hidden
        out = np.empty((h, 4 * h // self.t), np.float64)
        check(lib().spl_get_w1_grad_shard(self._h, r, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def saved(self, r: int, name: str, shape) -> np.ndarray:
        out = np.empty(shape, np.float64)
        check(lib().spl_get_saved(self._h, r, name.encode(), out.ctypes.data_as(C.POINTER(C.c_double)),
                                  out.size))
        return out

    def interior(self, r: int) -> np.ndarray:
        c = self.cfg
        out = np.empty((3, c.heads // self.t, c.batch, c.seq, c.seq), np.float64)
        check(lib().spl_attention_interior(self._h, r, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def ledger(self, r: int = 0) -> dict:
        n = C.c_int(32)
        arr = (_lib.LedgerEntry * 32)()
        check(lib().spl_ledger(self._h, r, arr, C.byref(n)))
        return {arr[i].name.decode(): (arr[i].elements, arr[i].bytes, arr[i].physical_bytes)
                for i in range(n.value)}

    def saved_bytes(self, r: int = 0) -> tuple[int, int, int]:
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().spl_saved_bytes(self._h, r, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def comm_log(self) -> dict:
        arr = (C.c_int64 * 16)()
        check(lib().spl_comm_log(self._h, arr))
        tags = ["schedule", "regather", "grad_sync", "recompute"]
        return {t: dict(all_gathers=arr[4 * i], reduce_scatters=arr[4 * i + 1],
                        all_reduces=arr[4 * i + 2], ring_elements=arr[4 * i + 3])
                for i, t in enumerate(tags)}

    def comm_log_reset(self):
        check(lib().spl_comm_log_reset(self._h))

    # ---- timing / profiling
    def timer_start(self):
        check(lib().spl_timer_start(self._h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        check(lib().spl_timer_stop(self._h, C.byref(ms)))
        return ms.value

    def synchronize(self):
        check(lib().spl_synchronize(self._h))

    def profile(self, on: bool):
        check(lib().spl_profile_enable(self._h, int(on)))

    def profile_read(self) -> dict:
        ms, n = (C.c_double * 5)(), (C.c_int64 * 5)()
        fl, by = (C.c_double * 5)(), (C.c_double * 5)()
        check(lib().spl_profile_read(self._h, ms, n, fl, by))
        return {k: dict(ms=ms[i], launches=n[i], flops=fl[i], bytes=by[i])
                for i, k in enumerate(_lib.KCLASS)}

    def launch_count(self, reset: bool = False) -> int:
        v = C.c_int64()
        check(lib().spl_launch_count(self._h, C.byref(v), int(reset)))
        return v.value

    def comm_paths(self) -> dict:
        """Collective paths in use: fused reduce-scatter, and the all-gather as "copy" (gathered
        copies), "local" (consumers read the simulated ranks' shards) or "pull" (consumers read
        the peer ranks' shards in their memory)."""
        v = (C.c_int32 * 2)()
        check(lib().spl_comm_paths(self._h, v))
        return {"fused_rs": bool(v[0]), "all_gather": ("copy", "local", "pull")[v[1]]}

    def set_graphs(self, on: bool):
        check(lib().spl_set_graphs(self._h, int(on)))


# ---------------------------------------------------------------- reference-shaped API
@dataclass
class SeqparForward:
    """Mirror of SeqparForward (block.hpp:136-154): output shards, per-rank ledgers, CommLog,
    and the device layer holding the saved state."""
    t: int
    cfg: BlockConfig
    y_shards: list
    ledgers: list
    comm: dict
    layer: SeqparLayer = field(repr=False)
    params_digest: bytes = field(default=b"", repr=False)


def _digest(params: np.ndarray) -> bytes:
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(params, np.float64).tobytes(), digest_size=16).digest()


@dataclass
class SeqparBackward:
    """Mirror of SeqparBackward (block.hpp:164-171)."""
    dx_shards: list
    param_grads: np.ndarray
    w1_grad_shards: list
    comm: dict


def _to_dev(a: np.ndarray, dtype: str, device: int):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=f"cuda:{device}", dtype=_tdtype(dtype))


def _to_host(t) -> np.ndarray:
    return t.detach().to("cpu", dtype=_torch().float64).numpy()


def seqpar_block_forward(x_shards: list, params: np.ndarray, t: int, cfg: BlockConfig,
                         recompute: str = "none", sequence_parallel: bool = True,
                         dtype: str = "f32", device: int = 0) -> SeqparForward:
    """seqpar_block_forward(x_shards, params, t, cfg) (block.cpp:512-602) on the GPU."""
    if t < 1:
        raise ValueError("t must be >= 1")
    if len(x_shards) != t:
        raise ValueError("expected one input shard per rank")
    layer = SeqparLayer(cfg, t, recompute, sequence_parallel, dtype, device)
    layer.load_params(params)
    for xs in x_shards:
        if tuple(xs.shape) != layer.shard_shape():
            raise ValueError("input shard must be {s/t, b, h}")
    y = layer.forward([_to_dev(xs, dtype, device) for xs in x_shards])
    ledgers = [layer.ledger(r) for r in range(t)]
    return SeqparForward(t, cfg, [_to_host(v) for v in y], ledgers, layer.comm_log(), layer,
                         _digest(params))


def seqpar_block_backward(dy_shards: list, fwd: SeqparForward, params: np.ndarray) -> SeqparBackward:
    """seqpar_block_backward(dy_shards, fwd, params) (block.cpp:622-749) on the GPU."""
    layer = fwd.layer
    if len(dy_shards) != fwd.t:
        raise ValueError("expected one gradient shard per rank")
    for d in dy_shards:
        if tuple(d.shape) != layer.shard_shape():
            raise ValueError("dy shard shape mismatch")
    # the backward GEMMs use `params` (block.cpp:639-640): reload them when they are not the
    # forward's; full recomputation would also re-run the forward with them, which the
    # reference never does, so that combination is rejected
    if fwd.params_digest and _digest(params) != fwd.params_digest:
        if layer.recompute == "full":
            raise ValueError("full recomputation re-runs the forward: backward params must be "
                             "the forward's")
        layer.load_params(params)
    layer.comm_log_reset()
    dx = layer.backward([_to_dev(d, layer.dtype, layer.device) for d in dy_shards])
    return SeqparBackward([_to_host(v) for v in dx], layer.grads(),
                          [layer.w1_grad_shard(r) for r in range(fwd.t)], layer.comm_log())


def seqpar_block_forward_sharded(x: "RankShardedTensor", params: np.ndarray, cfg: BlockConfig,
                                 **kw) -> SeqparForward:
    """The RankShardedTensor overload (block.hpp:158-162, block.cpp:604-613)."""
    if x.axis != "sequence":
        raise ValueError("layer input must be sharded along the sequence axis")
    x.check()
    return seqpar_block_forward(x.shards, params, len(x.shards), cfg, **kw)


@dataclass
class ReferenceForward:
    """Mirror of ReferenceForward (block.hpp:104-119): the single-rank layer. On the GPU it is
    the t = 1 layer (the reference's t = 1 seqpar path is bit-identical to it,
    test_seqpar.cpp:161-168)."""
    y: np.ndarray
    ledger: dict
    cfg: BlockConfig
    layer: SeqparLayer = field(repr=False)
    params_digest: bytes = field(default=b"", repr=False)

    def saved(self, name: str) -> np.ndarray:
        n = self.ledger[name][0]
        return self.layer.saved(0, name, (n,))


@dataclass
class BlockGrads:
    """Mirror of BlockGrads (block.hpp:123-126): packed param grads + dx."""
    params: np.ndarray
    dx: np.ndarray


def reference_block_forward(x: np.ndarray, params: np.ndarray, cfg: BlockConfig,
                            recompute: str = "none", dtype: str = "f32",
                            device: int = 0) -> ReferenceForward:
    """reference_block_forward(x, params, cfg) (block.cpp:419-456) on the GPU."""
    if tuple(x.shape) != (cfg.seq, cfg.batch, cfg.hidden):
        raise ValueError("reference_block_forward: input must be {s, b, h}")
    if cfg.heads <= 0 or cfg.hidden % cfg.heads:
        raise ValueError("hidden not divisible by heads")
    f = seqpar_block_forward([x], params, 1, cfg, recompute, True, dtype, device)
    return ReferenceForward(f.y_shards[0], f.ledgers[0], cfg, f.layer, f.params_digest)


def reference_block_backward(dy: np.ndarray, fwd: ReferenceForward, params: np.ndarray) -> BlockGrads:
    """reference_block_backward(dy, fwd, params) (block.cpp:458-510) on the GPU."""
    if tuple(dy.shape) != tuple(fwd.y.shape):
        raise ValueError("dy shape mismatch")
    f = SeqparForward(1, fwd.cfg, [fwd.y], [fwd.ledger], {}, fwd.layer, fwd.params_digest)
    b = seqpar_block_backward([dy], f, params)
    return BlockGrads(b.param_grads, b.dx_shards[0])


class RankShardedTensor:
    """Mirror of RankShardedTensor (tensor.hpp:80-89, tensor.cpp:227-259); axis is
    "sequence", "hidden" or "replicated"."""

    def __init__(self, shards: list, axis: str = "replicated", logical_shape=None):
        self.shards, self.axis = list(shards), axis
        self.logical_shape = tuple(logical_shape) if logical_shape is not None else None

    @classmethod
    def from_full(cls, full: np.ndarray, axis: str, axis_index: int, ranks: int):
        if axis == "replicated":
            return cls([full.copy() for _ in range(ranks)], axis, full.shape)
        if full.shape[axis_index] % ranks:
            raise ValueError("split axis not divisible by part count")
        return cls([np.ascontiguousarray(p) for p in np.split(full, ranks, axis_index)], axis, full.shape)

    def to_full(self, axis_index: int) -> np.ndarray:
        if self.axis == "replicated":
            return self.shards[0]
        return np.concatenate(self.shards, axis_index)

    def check(self):
        if not self.shards:
            raise ValueError("sharded tensor has no shards")
        if any(s.shape != self.shards[0].shape for s in self.shards):
            raise ValueError("shard shapes differ across ranks")
        if self.axis == "replicated" and any(not np.array_equal(s, self.shards[0]) for s in self.shards):
            raise ValueError("replicated tensor has diverging shards")


def attention_interior(q: np.ndarray, k: np.ndarray, cfg: BlockConfig, head_offset: int,
                       local_heads: int, dtype: str = "f32", device: int = 0) -> np.ndarray:
    """attention_interior(q, k, cfg, head_offset, local_heads) (block.cpp:381-417) on the GPU
    kernel (spl_attention_interior_qk). Returns {3, local_heads, b, s, s}: softmax_out,
    dropout_mask (0/1), dropout_out, as fp64."""
    torch = _torch()
    s, b = cfg.seq, cfg.batch
    if cfg.heads <= 0 or cfg.hidden % cfg.heads:
        raise ValueError("hidden not divisible by heads")
    lw = local_heads * (cfg.hidden // cfg.heads)
    if tuple(q.shape) != (s, b, lw) or tuple(k.shape) != (s, b, lw):
        raise ValueError("attention_interior: q and k must be {s, b, local_heads*hd}")
    td = _tdtype(dtype)
    dev = f"cuda:{device}"
    qd, kd = _to_dev(q, dtype, device), _to_dev(k, dtype, device)
    n = (local_heads, b, s, s)
    sm = torch.empty(n, dtype=td, device=dev)
    sd = torch.empty(n, dtype=td, device=dev)
    mk = torch.empty(n, dtype=torch.uint8, device=dev)
    d = _desc(cfg, "none", True, dtype, True)
    stream = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    check(lib().spl_attention_interior_qk(C.byref(d), device, C.c_void_p(qd.data_ptr()),
                                          C.c_void_p(kd.data_ptr()), head_offset, local_heads,
                                          C.c_void_p(sm.data_ptr()), C.c_void_p(mk.data_ptr()),
                                          C.c_void_p(sd.data_ptr()), stream))
    torch.cuda.synchronize(device)
    return np.stack([_to_host(sm), mk.cpu().numpy().astype(np.float64), _to_host(sd)])


# ---------------------------------------------------------------- collectives (collectives.hpp:57-62)
COMM_TAGS = {"schedule": 0, "regather": 1, "grad_sync": 2}


def _comm_dict(log) -> dict:
    return {t: dict(all_gathers=log[4 * i], reduce_scatters=log[4 * i + 1],
                    all_reduces=log[4 * i + 2], ring_elements=log[4 * i + 3])
            for i, t in enumerate(COMM_TAGS)}


def _group(tensors: list, op: str, device: int):
    torch = _torch()
    if not tensors:
        raise ValueError(f"{op}: empty rank group")
    shape = tuple(np.shape(tensors[0]))
    if any(tuple(np.shape(x)) != shape for x in tensors):
        raise ValueError(f"{op}: shard shapes differ across ranks")
    dev = [torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(f"cuda:{device}") for x in tensors]
    ptrs = (C.c_void_p * len(dev))(*[d.data_ptr() for d in dev])
    return dev, ptrs, shape, (C.c_int64 * max(len(shape), 1))(*shape)


def all_gather(shards: list, axis: int, tag: str = "schedule", device: int = 0):
    """all_gather(span<const Tensor>, axis, CommLog*, tag) (collectives.cpp:40-46) on device
    buffers in fp64. Returns (full, comm log)."""
    torch = _torch()
    dev, ptrs, shape, cs = _group(shards, "all_gather", device)
    if not 0 <= axis < len(shape):
        raise ValueError("axis out of range")
    out_shape = list(shape)
    out_shape[axis] *= len(shards)
    out = torch.empty(out_shape, dtype=torch.float64, device=f"cuda:{device}")
    log = (C.c_int64 * 12)()
    check(lib().spl_all_gather(ptrs, len(dev), cs, len(shape), axis, _lib.DTYPE_F64,
                               C.c_void_p(out.data_ptr()), log, COMM_TAGS[tag],
                               C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return out.cpu().numpy(), _comm_dict(log)


def reduce_scatter(partials: list, axis: int, tag: str = "schedule", device: int = 0):
    """reduce_scatter (collectives.cpp:48-57): rank-ordered fp64 sum, split along axis."""
    torch = _torch()
    dev, ptrs, shape, cs = _group(partials, "reduce_scatter", device)
    t = len(dev)
    if not 0 <= axis < len(shape):
        raise ValueError("axis out of range")
    if shape[axis] % t:
        raise ValueError("split axis not divisible by part count")
    piece = list(shape)
    piece[axis] //= t
    outs = [torch.empty(piece, dtype=torch.float64, device=f"cuda:{device}") for _ in range(t)]
    optr = (C.c_void_p * t)(*[o.data_ptr() for o in outs])
    log = (C.c_int64 * 12)()
    check(lib().spl_reduce_scatter(ptrs, t, cs, len(shape), axis, _lib.DTYPE_F64, optr, log,
                                   COMM_TAGS[tag],
                                   C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return [o.cpu().numpy() for o in outs], _comm_dict(log)


def all_reduce(partials: list, tag: str = "schedule", device: int = 0):
    """all_reduce (collectives.cpp:59-65): rank-ordered fp64 sum."""
    torch = _torch()
    dev, ptrs, shape, cs = _group(partials, "all_reduce", device)
    out = torch.empty(shape, dtype=torch.float64, device=f"cuda:{device}")
    log = (C.c_int64 * 12)()
    check(lib().spl_all_reduce(ptrs, len(dev), cs, len(shape), _lib.DTYPE_F64,
                               C.c_void_p(out.data_ptr()), log, COMM_TAGS[tag],
                               C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
    return out.cpu().numpy(), _comm_dict(log)


@dataclass
class RecomputeStrategy:
    """RecomputeStrategy (config.hpp:53-67); parse/name restate config.cpp:36-84."""
    kind: str = "none"
    sequence_parallel: bool = False
    microbatch_level: bool = False

    @classmethod
    def parse(cls, spec: str) -> "RecomputeStrategy":
        out, have = cls(), False
        for tok in spec.split("+") if spec else []:
            if tok in ("none", "full", "selective"):
                if have:
                    raise ValueError(f"strategy '{spec}' names more than one recompute kind")
                have, out.kind = True, tok
            elif tok == "seq":
                out.sequence_parallel = True
            elif tok == "mblevel":
                out.microbatch_level = True
            else:
                raise ValueError(f"unknown strategy token '{tok}' (expected none|full|selective "
                                 "with optional +seq, +mblevel)")
        if not have:
            raise ValueError(f"strategy '{spec}' must name one of none|full|selective")
        if out.microbatch_level and out.kind == "none":
            raise ValueError("'none+mblevel' is not a strategy: the microbatch window needs a "
                             "full or selective base to checkpoint with")
        return out

    def name(self) -> str:
        return self.kind + ("+seq" if self.sequence_parallel else "") + \
            ("+mblevel" if self.microbatch_level else "")


def per_layer_bytes(a: int, h: int, s: int, b: int, t: int, kind: str, sequence_parallel: bool,
                    act: int = 2, mask: int = 1) -> int:
    """per_layer_bytes (activation_memory.cpp:79-82) through the C ABI."""
    out = C.c_int64()
    check(lib().spl_per_layer_bytes(a, h, s, b, t, _lib.RECOMPUTE[kind], int(sequence_parallel),
                                    act, mask, C.byref(out)))
    return out.value


def per_layer_bytes_exact(a, h, s, b, t, kind, sequence_parallel, act=2, mask=1):
    n, d = C.c_int64(), C.c_int64()
    check(lib().spl_per_layer_bytes_exact(a, h, s, b, t, _lib.RECOMPUTE[kind], int(sequence_parallel),
                                          act, mask, C.byref(n), C.byref(d)))
    return n.value, d.value


def layer_component_breakdown(a: int, h: int, s: int, b: int, act: int = 2, mask: int = 1) -> dict:
    """layer_component_breakdown (activation_memory.cpp:84-104) through the C ABI."""
    out = (C.c_int64 * 4)()
    check(lib().spl_layer_component_breakdown(a, h, s, b, act, mask, out))
    return dict(attention=out[0], mlp=out[1], layer_norms=out[2], total=out[3])


def percent_of_baseline(a, h, s, b, t, kind, sequence_parallel, act=2, mask=1):
    """percent_of_baseline (activation_memory.cpp:195-200): exact (num, den)."""
    n, d = C.c_int64(), C.c_int64()
    check(lib().spl_percent_of_baseline(a, h, s, b, t, _lib.RECOMPUTE[kind], int(sequence_parallel),
                                        act, mask, C.byref(n), C.byref(d)))
    return n.value, d.value


def total_first_stage_bytes(a, h, s, b, t, kind, sequence_parallel, layers, pipeline=1,
                            interleave=1, act=2, mask=1) -> int:
    """total_first_stage_bytes (activation_memory.cpp:112-123) through the C ABI."""
    out = C.c_int64()
    check(lib().spl_total_first_stage_bytes(a, h, s, b, t, _lib.RECOMPUTE[kind],
                                            int(sequence_parallel), layers, pipeline, interleave,
                                            act, mask, C.byref(out)))
    return out.value


def layer_comm_bytes(s: int, b: int, h: int, t: int, elem: int = 2,
                     sequence_parallel: bool = True) -> int:
    """layer_comm_bytes_tensor_sequence / _tensor_parallel (collectives.cpp:75-87)."""
    out = C.c_int64()
    check(lib().spl_layer_comm_bytes(s, b, h, t, elem, int(sequence_parallel), C.byref(out)))
    return out.value


class SeqparStack:
    """L layers (layer_index = cfg.layer_index + l) on t simulated ranks sharing one workspace
    (spl_stack_*): the p = 1 stage of total_first_stage_bytes / simulate_memory."""

    def __init__(self, cfg: BlockConfig, t: int, layers: int, recompute: str = "selective",
                 sequence_parallel: bool = True, dtype: str = "bf16", device: int = 0,
                 check_finite: bool = True):
        self.cfg, self.t, self.recompute, self.sp, self.dtype = cfg, t, recompute, sequence_parallel, dtype
        self.device = device
        d = _desc(cfg, recompute, sequence_parallel, dtype, check_finite)
        self._s = C.c_void_p()
        check(lib().spl_stack_create_local(C.byref(d), device, t, layers, C.byref(self._s)))
        self.layers = []
        for l in range(layers):
            h = C.c_void_p()
            check(lib().spl_stack_layer(self._s, l, C.byref(h)))
            cl = BlockConfig(**{**cfg.__dict__, "layer_index": cfg.layer_index + l})
            self.layers.append(SeqparLayer(cl, t, recompute, sequence_parallel, dtype, device,
                                           check_finite, _borrow=h))
        self.local = self.layers[0].local

    def close(self):
        for L in getattr(self, "layers", []):
            L.close()
        if getattr(self, "_s", None):
            lib().spl_stack_destroy(self._s)
            self._s = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_shape(self):
        return self.layers[0].shard_shape()

    def _bind_stream(self):
        torch = _torch()
        check(lib().spl_stack_set_stream(self._s, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def _run(self, fn, a: list, out: list | None) -> list:
        torch = _torch()
        self._bind_stream()
        if len(a) != self.local:
            raise ValueError("expected one shard per rank")
        for ai in a:
            if tuple(ai.shape) != self.shard_shape() or ai.dtype != _tdtype(self.dtype):
                raise ValueError(f"shard must be {self.shard_shape()} {self.dtype}")
        if out is None:
            out = [torch.empty_like(ai) for ai in a]
        ap = (C.c_void_p * self.local)(*[ai.data_ptr() for ai in a])
        op = (C.c_void_p * self.local)(*[oi.data_ptr() for oi in out])
        check(fn(self._s, ap, op))
        return out

    def forward(self, x: list, y: list | None = None) -> list:
        return self._run(lib().spl_stack_forward, x, y)

    def backward(self, dy: list, dx: list | None = None) -> list:
        return self._run(lib().spl_stack_backward, dy, dx)

    def memory(self, r: int = 0) -> dict:
        out = (C.c_int64 * 7)()
        check(lib().spl_stack_memory(self._s, r, out))
        keys = ["ledger", "physical_saved", "uncounted_saved", "workspace", "params", "grads",
                "layer_workspace"]
        return dict(zip(keys, list(out)))
