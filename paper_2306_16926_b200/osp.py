"""Python front of the B200 OSP sync path, over the C-ABI (include/osp_c.h).

Names and error classes follow the reference pslab API
(/root/reference/proj/include/pslab/*.hpp). Vectors are torch CUDA tensors
(fp32); torch supplies device memory and the current stream — the arithmetic
runs in this package's sm_100a kernels only.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi
from ._capi import P, c_dbl, c_i64, c_int, c_u32, c_u64, c_void_p


# ---- errors: 1:1 with pslab::Error (errors.hpp:11-69) -------------------------

class Error(RuntimeError):
    pass


class PartitionError(Error):
    pass


class ShapeError(Error):
    pass


class LayerError(Error):
    pass


class ParseError(Error):
    pass


class ConfigError(Error):
    pass


class FormatError(Error):
    pass


class ProtocolError(Error):
    pass


class NumericError(Error):
    pass


class CudaError(Error):
    pass


class InvalidArgument(Error):
    pass


_STATUS = {1: PartitionError, 2: ShapeError, 3: LayerError, 4: ParseError, 5: ConfigError,
           6: FormatError, 7: ProtocolError, 8: NumericError, 20: CudaError, 21: InvalidArgument}


def lib():
    return _capi.load()


def _check(status: int):
    if status != 0:
        msg = lib().osp_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


def _stream(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _dev_f32(t: torch.Tensor, name: str):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise InvalidArgument(f"{name} must be a float32 CUDA tensor")
    if not t.is_contiguous():
        raise InvalidArgument(f"{name} must be contiguous")


class _DevArray:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, shape, typestr: str, strides=None, owner=None):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": strides}
        self._owner = owner


class _Handle:
    """Owns one library handle. Zero-copy views reference this holder, not the
    Python wrapper: a view's storage keeps its owner alive from C, where the
    garbage collector cannot see it, so a wrapper <-> view cycle would never be
    collected (and the device memory never freed)."""

    __slots__ = ("h", "_destroy", "_parent")

    def __init__(self, h, destroy: Optional[str] = None, parent=None):
        self.h, self._destroy, self._parent = h, destroy, parent

    def close(self):
        h, self.h = self.h, None
        if h and self._destroy is not None and _capi._lib is not None:
            getattr(_capi._lib, self._destroy)(h)

    def __del__(self):
        self.close()


def _view(ptr, shape, typestr, strides=None, owner=None) -> torch.Tensor:
    return torch.as_tensor(_DevArray(ptr, shape, typestr, strides, owner), device="cuda")


def _u8(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint8))
    return a, a.ctypes.data_as(P(ctypes.c_uint8))


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    if a.size == 0:
        a = np.zeros(1, dtype=np.int32)
    return a, a.ctypes.data_as(P(ctypes.c_int32))


# ---- partition ---------------------------------------------------------------

class Partition:
    """LayerPartition (param.hpp:19-46)."""

    def __init__(self, layer_counts: Sequence[int], bytes_per_element: int = 4):
        counts = np.ascontiguousarray(np.asarray(list(layer_counts), dtype=np.uint64))
        h = c_void_p()
        _check(lib().osp_partition_create(counts.ctypes.data_as(P(c_u64)), counts.size,
                                          bytes_per_element, ctypes.byref(h)))
        self._h = h
        self.counts = counts
        self.offsets = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)

    @property
    def handle(self):
        return self._h

    def layer_count(self) -> int:
        return int(lib().osp_partition_layer_count(self._h))

    def total_count(self) -> int:
        return int(lib().osp_partition_total_count(self._h))

    def total_bytes(self) -> int:
        return int(lib().osp_partition_total_bytes(self._h))

    def bytes_per_element(self) -> int:
        return int(lib().osp_partition_bytes_per_element(self._h))

    def layer(self, layer_id: int):
        off, cnt = c_u64(), c_u64()
        _check(lib().osp_partition_layer(self._h, layer_id, ctypes.byref(off), ctypes.byref(cnt)))
        return int(off.value), int(cnt.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _capi._lib is not None:
            _capi._lib.osp_partition_destroy(h)
            self._h = None


# ---- free functions (one kernel each) ------------------------------------------

def aggregate_layer(contribs: Sequence[torch.Tensor], weights: Sequence[float],
                    stream=None) -> torch.Tensor:
    """aggregate_layer (protocol.cpp:9-30)."""
    n = len(contribs)
    if n == 0:
        _check(lib().osp_aggregate_layer(None, 0, None, 0, None, None))
    size = contribs[0].numel()
    for c in contribs:
        _dev_f32(c, "contribution")
        if c.numel() != size:
            raise ProtocolError("contribution size mismatch in aggregation")
    if len(weights) != n:
        raise ProtocolError("aggregation needs one contribution per worker")
    out = torch.empty(size, dtype=torch.float32, device=contribs[0].device)
    ptrs = (c_void_p * n)(*[_ptr(c) for c in contribs])
    w = (c_dbl * n)(*weights)
    _check(lib().osp_aggregate_layer(ptrs, n, w, size, _ptr(out), _stream(stream)))
    return out


def apply_delta(p: torch.Tensor, d: torch.Tensor, scale: float, stream=None) -> None:
    """apply_delta dense form (param.cpp:127-137), in place."""
    _dev_f32(p, "params")
    _dev_f32(d, "delta")
    if p.numel() != d.numel():
        raise ShapeError(f"delta length {d.numel()} does not match param length {p.numel()}")
    _check(lib().osp_apply_delta(_ptr(p), _ptr(d), p.numel(), scale, _stream(stream)))


def sgd_delta(grad: torch.Tensor, lr: float, stream=None) -> torch.Tensor:
    """sgd_delta (learner.cpp:391-398)."""
    _dev_f32(grad, "grad")
    out = torch.empty_like(grad)
    _check(lib().osp_sgd_delta(_ptr(grad), grad.numel(), lr, _ptr(out), _stream(stream)))
    return out


def synth_delta(seed: int, worker: int, iteration: int, n: int, first: int = 0,
                stream=None) -> torch.Tensor:
    """Synthetic delta source (runner.cpp:312-321)."""
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _check(lib().osp_synth_delta(seed, worker, iteration, first, n, _ptr(out), _stream(stream)))
    return out


def synth_deltas(seed: int, n_workers: int, iteration: int, n: int, out: torch.Tensor = None,
                 stream=None) -> torch.Tensor:
    """All workers' synthetic deltas for one iteration as an [N, n] block."""
    if out is None:
        out = torch.empty((n_workers, n), dtype=torch.float32, device="cuda")
    _check(lib().osp_synth_deltas(seed, n_workers, iteration, n, _ptr(out), out.stride(0),
                                  _stream(stream)))
    return out


def lgp_partial(part: Partition, params: torch.Tensor, global_delta: torch.Tensor,
                local_delta: torch.Tensor, ics_flags, base: torch.Tensor, stream=None) -> None:
    """lgp_partial (protocol.cpp:69-97) on flat vectors; flags 1 = local estimate."""
    f, fp = _u8(ics_flags)
    if f.size != part.layer_count():
        raise ShapeError("layer flags do not cover the partition")
    _check(lib().osp_lgp_partial(part.handle, _ptr(params), _ptr(global_delta),
                                 _ptr(local_delta), fp, _ptr(base), _stream(stream)))


def lgp_correct(part: Partition, params: torch.Tensor, base: torch.Tensor,
                global_delta: torch.Tensor, layer_ids, stream=None) -> None:
    """lgp_correct (protocol.cpp:99-116): p = base + global on the listed layers."""
    ids, ip = _i32(layer_ids)
    _check(lib().osp_lgp_correct(part.handle, _ptr(params), _ptr(base), _ptr(global_delta), ip,
                                 len(layer_ids), _stream(stream)))


def pgp_layer_importance(part: Partition, params: torch.Tensor, grads: torch.Tensor,
                         stream=None) -> np.ndarray:
    """pgp_layer_importance (importance.cpp:11-28), reference-exact scores."""
    if params.numel() != grads.numel():
        raise ShapeError("param/grad length mismatch")
    out = np.empty(part.layer_count(), dtype=np.float64)
    _check(lib().osp_pgp_layer_importance(part.handle, _ptr(params), _ptr(grads),
                                          out.ctypes.data_as(P(c_dbl)), _stream(stream)))
    return out


def rank_and_gib(part: Partition, scores, budget: int, stream=None):
    """rank_layers + build_gib (importance.cpp:30-59) -> (order, ics_flags)."""
    s = np.ascontiguousarray(np.asarray(scores, dtype=np.float64))
    if s.size != part.layer_count():
        raise ShapeError("importance covers a different layer count than the partition")
    order = np.empty(s.size, dtype=np.int32)
    flags = np.empty(s.size, dtype=np.uint8)
    _check(lib().osp_rank_and_gib(part.handle, s.ctypes.data_as(P(c_dbl)), budget,
                                  order.ctypes.data_as(P(ctypes.c_int32)),
                                  flags.ctypes.data_as(P(ctypes.c_uint8)), _stream(stream)))
    return order, flags


def pgp_rank_gib(part: Partition, params: torch.Tensor, grads: torch.Tensor, budget: int,
                 stream=None):
    """check_resolution's PGP -> rank -> GIB (protocol.cpp:407-419) on device
    vectors, certified (osp_pgp_rank_gib) -> (scores, deferred ids in rank
    order, flags)."""
    _dev_f32(params, "params")
    _dev_f32(grads, "grads")
    if params.numel() != part.total_count() or grads.numel() != part.total_count():
        raise ShapeError("vectors do not match the partition")
    L = part.layer_count()
    scores = np.empty(L, dtype=np.float64)
    order = np.empty(L, dtype=np.int32)
    flags = np.empty(L, dtype=np.uint8)
    k = c_i64()
    _check(lib().osp_pgp_rank_gib(part.handle, _ptr(params), _ptr(grads), int(budget),
                                  scores.ctypes.data_as(P(c_dbl)),
                                  order.ctypes.data_as(P(ctypes.c_int32)), ctypes.byref(k),
                                  flags.ctypes.data_as(P(ctypes.c_uint8)), _stream(stream)))
    return scores, order[: k.value].copy(), flags


def split_for_sync(part: Partition, ics_flags, ics_order, n_chunks: int):
    """split_for_sync index lists (protocol.cpp:122-166) -> (rs_ids, chunk_of, n_used)."""
    f, fp = _u8(ics_flags)
    if f.size != part.layer_count():
        raise ShapeError("gib covers a different layer count than the delta")
    o, op = _i32(ics_order)
    L = part.layer_count()
    rs = np.empty(L, dtype=np.int32)
    chunk_of = np.empty(L, dtype=np.int32)
    nrs = c_i64()
    used = c_int()
    _check(lib().osp_split_for_sync(part.handle, fp, op, len(ics_order), n_chunks,
                                    rs.ctypes.data_as(P(ctypes.c_int32)), ctypes.byref(nrs),
                                    chunk_of.ctypes.data_as(P(ctypes.c_int32)),
                                    ctypes.byref(used)))
    return rs[: nrs.value].copy(), chunk_of, int(used.value)


def gib_encode(tag: int, ics_flags) -> bytes:
    """gib_encode (importance.cpp:61-97)."""
    f, fp = _u8(ics_flags)
    n = int(lib().osp_gib_encoded_size(f.size))
    out = np.zeros(n, dtype=np.uint8)
    _check(lib().osp_gib_encode(tag, f.size, fp, out.ctypes.data_as(P(ctypes.c_uint8)), n))
    return out.tobytes()


def gib_wire_encode(tag: int, ics_flags, order) -> bytes:
    """GIB wire with the rank-order side channel: gib_encode bytes, then n and the
    deferred ids least important first (include/osp_c.h, osp_gib_wire_encode)."""
    f, fp = _u8(ics_flags)
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32).reshape(-1))
    op = o.ctypes.data_as(P(ctypes.c_int32)) if o.size else None
    n = c_u64()
    _check(lib().osp_gib_wire_encode(tag, f.size, fp, op, o.size, None, 0, ctypes.byref(n)))
    out = np.zeros(max(n.value, 1), dtype=np.uint8)
    _check(lib().osp_gib_wire_encode(tag, f.size, fp, op, o.size,
                                     out.ctypes.data_as(P(ctypes.c_uint8)), out.size,
                                     ctypes.byref(n)))
    return out[: n.value].tobytes()


def gib_wire_decode(buf: bytes):
    """-> (tag, flags, order); order is None for a bitmap-only buffer."""
    b = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
    n = b.size
    if b.size == 0:
        b = np.zeros(1, dtype=np.uint8)
    bp = b.ctypes.data_as(P(ctypes.c_uint8))
    tag, L, k = c_u32(), c_u32(), c_i64()
    _check(lib().osp_gib_wire_decode(bp, n, ctypes.byref(tag), ctypes.byref(L), None, 0, None, 0,
                                     ctypes.byref(k)))
    flags = np.zeros(max(L.value, 1), dtype=np.uint8)
    order = np.zeros(max(k.value, 1), dtype=np.int32)
    _check(lib().osp_gib_wire_decode(bp, n, None, None, flags.ctypes.data_as(P(ctypes.c_uint8)),
                                     flags.size, order.ctypes.data_as(P(ctypes.c_int32)),
                                     order.size, ctypes.byref(k)))
    return (int(tag.value), flags[: L.value].copy(),
            None if k.value < 0 else order[: k.value].copy())


def gib_decode(buf: bytes):
    """gib_decode (importance.cpp:99-117) -> (tag, flags)."""
    b = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
    if b.size == 0:
        b = np.zeros(1, dtype=np.uint8)
        n = 0
    else:
        n = b.size
    tag, L = c_u32(), c_u32()
    _check(lib().osp_gib_decode(b.ctypes.data_as(P(ctypes.c_uint8)), n, ctypes.byref(tag),
                                ctypes.byref(L), None, 0))
    flags = np.zeros(max(L.value, 1), dtype=np.uint8)
    _check(lib().osp_gib_decode(b.ctypes.data_as(P(ctypes.c_uint8)), n, ctypes.byref(tag),
                                ctypes.byref(L), flags.ctypes.data_as(P(ctypes.c_uint8)),
                                flags.size))
    return int(tag.value), flags[: L.value].copy()


def encode_payload(part: Partition, values: torch.Tensor, layer_ids, kind: int, iteration: int,
                   stream=None) -> torch.Tensor:
    """encode_payload_message (message.cpp:53-78) of device-resident layers -> device bytes."""
    _dev_f32(values, "values")
    ids, ip = _i32(layer_ids)
    n = len(layer_ids)
    size = int(lib().osp_payload_encoded_size(part.handle, ip, n))
    if size == 0:
        raise LayerError("layer id out of range")
    out = torch.empty(size, dtype=torch.uint8, device=values.device)
    got = c_u64()
    _check(lib().osp_encode_payload(part.handle, _ptr(values), ip, n, kind, iteration, _ptr(out),
                                    size, ctypes.byref(got), _stream(stream)))
    return out[: got.value]


def decode_payload(part: Partition, buf: torch.Tensor, values: torch.Tensor, stream=None):
    """decode_payload_message (message.cpp:80-99) from device bytes into a flat device
    vector -> (kind, iteration, layer ids)."""
    _dev_f32(values, "values")
    if not (buf.is_cuda and buf.dtype == torch.uint8 and buf.is_contiguous()):
        raise InvalidArgument("buf must be a contiguous uint8 CUDA tensor")
    L = part.layer_count()
    ids = np.empty(max(min(L, 65535), 1), dtype=np.int32)
    kind, it, n = ctypes.c_uint8(), c_u32(), c_i64()
    _check(lib().osp_decode_payload(part.handle, _ptr(buf), buf.numel(), _ptr(values),
                                    ctypes.byref(kind), ctypes.byref(it),
                                    ids.ctypes.data_as(P(ctypes.c_int32)), ids.size,
                                    ctypes.byref(n), _stream(stream)))
    return int(kind.value), int(it.value), ids[: n.value].copy()


def compute_umax(bandwidth_bps, t_c, n_workers, model_bytes, latency_s=0.0, loss_rate=0.0,
                 eq5_literal=False) -> int:
    """compute_umax (tuning.cpp:8-21)."""
    out = c_u64()
    _check(lib().osp_compute_umax(bandwidth_bps, latency_s, loss_rate, t_c, n_workers,
                                  model_bytes, 1 if eq5_literal else 0, ctypes.byref(out)))
    return int(out.value)


class SguSchedule:
    """SguSchedule + tune_sgu (tuning.hpp:27-38, tuning.cpp:23-48)."""

    def __init__(self, u_max: int = 0):
        self._s = _capi.osp_sgu_schedule(u_max, 0, 0.0, 0, 0)

    @property
    def u_max(self):
        return int(self._s.u_max)

    @u_max.setter
    def u_max(self, v):
        self._s.u_max = int(v)

    @property
    def initial_loss(self):
        return float(self._s.initial_loss) if self._s.has_initial_loss else None

    @property
    def current_budget(self):
        return int(self._s.current_budget)

    def tune(self, epoch: int, loss: float) -> int:
        out = c_u64()
        _check(lib().osp_tune_sgu(ctypes.byref(self._s), epoch, loss, ctypes.byref(out)))
        return int(out.value)


# ---- the batched group path -------------------------------------------------------

class OspGroup:
    """N co-resident OspWorkers + the OspServer of one GPU, stepped on the device.

    One iteration = stage1 (barrier) + stage2_chunk(c) for every chunk slot +
    resolve (PGP -> certified rank -> next GIB). See include/osp_c.h.
    """

    def __init__(self, part: Partition, n_workers: int, weights: Optional[Sequence[float]] = None,
                 n_chunks: int = 4, init_params: Optional[torch.Tensor] = None,
                 tile_elems: int = 0, sgd_lr: float = 0.0, tma: Optional[bool] = None,
                 carry: bool = True, small: bool = True, stream=None):
        """tma: None = TMA-staged stage kernels when the shape allows them, True =
        require them, False = register-staged kernels (identical results).
        carry: with the TMA family, stage 1 also keeps the ICS aggregate so stage 2
        only broadcasts it (OSP_GROUP_NO_CARRY when False; identical results).
        small: launch-bound layouts step in one single-CTA launch
        (OSP_GROUP_NO_SMALL when False; identical results)."""
        self.part = part
        self.N = n_workers
        self.M = part.total_count()
        self.L = part.layer_count()
        self.n_chunks = n_chunks
        w = list(weights) if weights is not None else [1.0 / n_workers] * n_workers
        if len(w) != n_workers:
            raise ConfigError("one weight per worker")
        self._w = (c_dbl * max(n_workers, 1))(*w)
        cfg = _capi.osp_group_config(n_workers, ctypes.cast(self._w, P(c_dbl)), n_chunks,
                                     tile_elems, sgd_lr,
                                     {None: 0, True: _capi.GROUP_TMA,
                                      False: _capi.GROUP_REGISTER}[tma]
                                     | (0 if carry else _capi.GROUP_NO_CARRY)
                                     | (0 if small else _capi.GROUP_NO_SMALL))
        init = 0
        if init_params is not None:
            _dev_f32(init_params, "init_params")
            if init_params.numel() != self.M:
                raise ShapeError("init params do not match the partition")
            init = _ptr(init_params)
        h = c_void_p()
        _check(lib().osp_group_create(part.handle, ctypes.byref(cfg), init or None,
                                      _stream(stream), ctypes.byref(h)))
        self._owned = True
        self._hnd = _Handle(h, "osp_group_destroy")
        self._attach(h)

    @classmethod
    def _borrow(cls, handle, part: Partition, n_workers: int, n_chunks: int, owner):
        """View of a group owned by another handle (the local state of a shard)."""
        self = cls.__new__(cls)
        self.part, self.N, self.n_chunks = part, n_workers, n_chunks
        self.M, self.L = part.total_count(), part.layer_count()
        self._owned = False
        self._hnd = _Handle(c_void_p(handle), None, parent=owner)  # owner: the shard's _Handle
        self._attach(c_void_p(handle))
        return self

    def _attach(self, h):
        self._h = h
        ld = c_u64()
        pp = lib().osp_group_worker_params(h, ctypes.byref(ld))
        self.ldP = int(ld.value)
        o = self._hnd
        self._g = _view(lib().osp_group_global(h), (self.M,), "<f4", owner=o)
        self._p = _view(pp, (self.N, self.M), "<f4", strides=(self.ldP * 4, 4), owner=o)
        self._scores = _view(lib().osp_group_scores(h), (self.L,), "<f8", owner=o)

    # state views (device, zero-copy)
    @property
    def global_params(self) -> torch.Tensor:
        return self._g

    @property
    def worker_params(self) -> torch.Tensor:
        return self._p

    @property
    def scores(self) -> torch.Tensor:
        return self._scores

    def _deltas(self, deltas: torch.Tensor):
        if not (deltas.is_cuda and deltas.dtype == torch.float32 and deltas.dim() == 2):
            raise InvalidArgument("deltas must be a [N, >=M] float32 CUDA tensor")
        if deltas.shape[0] != self.N or deltas.stride(1) != 1:
            raise ShapeError("deltas must have one unit-stride row per worker")
        if deltas.shape[1] < self.M:
            raise ShapeError(f"delta rows hold {deltas.shape[1]} elements, the partition {self.M}")
        return _ptr(deltas), deltas.stride(0)

    def set_budget(self, budget_bytes: int, stream=None):
        _check(lib().osp_group_set_budget(self._h, int(budget_bytes), _stream(stream)))

    def set_gib(self, ics_flags, ics_order, tag: int, stream=None):
        f, fp = _u8(ics_flags)
        if f.size != self.L:
            raise ShapeError(f"gib covers {f.size} layers, the partition {self.L}")
        o, op = _i32(ics_order)
        _check(lib().osp_group_set_gib(self._h, fp, op, len(ics_order), tag, _stream(stream)))

    def stage1(self, deltas: torch.Tensor, stream=None):
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_stage1(self._h, p, ld, _stream(stream)))

    def stage2_chunk(self, chunk: int, deltas: torch.Tensor, stream=None):
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_stage2_chunk(self._h, chunk, p, ld, _stream(stream)))

    def stage2_all(self, deltas: torch.Tensor, stream=None):
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_stage2_all(self._h, p, ld, _stream(stream)))

    def stages(self, deltas: torch.Tensor, stream=None):
        """stage1 + stage2_all."""
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_stages(self._h, p, ld, _stream(stream)))

    def resolve(self, deltas: torch.Tensor, stream=None):
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_resolve(self._h, p, ld, _stream(stream)))

    def gib_wire(self, stream=None) -> bytes:
        """The current GIB as a wire (bitmap + rank order), from the device."""
        n = c_u64()
        _check(lib().osp_group_gib_wire(self._h, None, 0, ctypes.byref(n), _stream(stream)))
        out = np.zeros(n.value, dtype=np.uint8)
        _check(lib().osp_group_gib_wire(self._h, out.ctypes.data_as(P(ctypes.c_uint8)), out.size,
                                        ctypes.byref(n), _stream(stream)))
        return out.tobytes()

    def set_gib_wire(self, buf: bytes, stream=None):
        b = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
        _check(lib().osp_group_set_gib_wire(self._h, b.ctypes.data_as(P(ctypes.c_uint8)), b.size,
                                            _stream(stream)))

    def set_momentum(self, mu: float, stream=None):
        """Heavy-ball momentum on gradient inputs, fused into stage 1 (extension;
        include/osp_c.h osp_group_set_momentum)."""
        _check(lib().osp_group_set_momentum(self._h, float(mu), _stream(stream)))

    def stage2_resolve(self, deltas: torch.Tensor, stream=None):
        """stage2_all + resolve (overlapped with the ICS carry)."""
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_stage2_resolve(self._h, p, ld, _stream(stream)))

    def step(self, deltas: torch.Tensor, stream=None):
        p, ld = self._deltas(deltas)
        _check(lib().osp_group_step(self._h, p, ld, _stream(stream)))

    def _host_args(self, host_deltas, params_out):
        if isinstance(host_deltas, torch.Tensor):
            if host_deltas.device.type != "cpu" or host_deltas.dtype != torch.float32:
                raise InvalidArgument("host deltas must be a float32 CPU tensor")
            if host_deltas.dim() != 2 or host_deltas.stride(1) != 1:
                raise ShapeError("host deltas must be [N, >=M] with unit inner stride")
            shape, ptr, ld = tuple(host_deltas.shape), host_deltas.data_ptr(), host_deltas.stride(0)
        else:
            raise InvalidArgument("the pipelined host step takes pinned torch CPU tensors")
        if shape[0] != self.N or shape[1] < self.M:
            raise ShapeError(f"host deltas are {list(shape)}, need [{self.N}, >={self.M}]")
        pout = None
        if params_out is not None:
            if not (isinstance(params_out, torch.Tensor) and params_out.device.type == "cpu"
                    and params_out.dtype == torch.float32 and params_out.is_contiguous()
                    and params_out.numel() == self.M):
                raise ShapeError("params_out must be a contiguous float32 CPU tensor of M")
            pout = params_out.data_ptr()
        return ptr, ld, pout

    def step_host_async(self, host_deltas: torch.Tensor, params_out: Optional[torch.Tensor] = None,
                        gib_out: Optional[torch.Tensor] = None, stream=None):
        """Pipelined step_host (osp_group_step_host_async): returns once issued;
        this call's H2D overlaps the previous call's step and D2H. Outputs are
        valid after host_wait()."""
        ptr, ld, pout = self._host_args(host_deltas, params_out)
        gout = gib_out.data_ptr() if gib_out is not None else None
        _check(lib().osp_group_step_host_async(self._h, ptr, ld, gout, pout, _stream(stream)))

    def host_wait(self):
        _check(lib().osp_group_host_wait(self._h))

    def step_host(self, host_deltas, stream=None, params_out=None) -> bytes:
        """End-to-end step from host memory: H2D copy of the N delta rows, the
        step, and D2H of the next GIB and of the updated global vector (every
        worker's parameters at the iteration boundary; OspServer::global_params /
        OspWorker::params). params_out: a host float32 array of M elements to
        receive it, or None to skip that copy."""
        if isinstance(host_deltas, torch.Tensor):
            if host_deltas.device.type != "cpu" or host_deltas.dtype != torch.float32:
                raise InvalidArgument("host deltas must be a float32 CPU tensor")
            if host_deltas.dim() != 2 or host_deltas.stride(1) != 1:
                raise ShapeError("host deltas must be [N, >=M] with unit inner stride")
            shape = tuple(host_deltas.shape)
            ptr, ld = host_deltas.data_ptr(), host_deltas.stride(0)
        else:
            if not (isinstance(host_deltas, np.ndarray) and host_deltas.dtype == np.float32):
                raise InvalidArgument("host deltas must be a float32 numpy array")
            if host_deltas.ndim != 2 or host_deltas.strides[1] != 4 or host_deltas.strides[0] % 4:
                raise ShapeError("host deltas must be [N, >=M] with unit inner stride")
            shape = host_deltas.shape
            ptr, ld = host_deltas.ctypes.data, host_deltas.strides[0] // 4
        if shape[0] != self.N or shape[1] < self.M:
            raise ShapeError(f"host deltas are {list(shape)}, need [{self.N}, >={self.M}]")
        pout = None
        if params_out is not None:
            if isinstance(params_out, torch.Tensor):
                if not (params_out.device.type == "cpu" and params_out.dtype == torch.float32
                        and params_out.is_contiguous() and params_out.numel() == self.M):
                    raise ShapeError("params_out must be a contiguous float32 CPU tensor of M")
                pout = params_out.data_ptr()
            else:
                if not (isinstance(params_out, np.ndarray) and params_out.dtype == np.float32
                        and params_out.flags.c_contiguous and params_out.size == self.M):
                    raise ShapeError("params_out must be a contiguous float32 array of M")
                pout = params_out.ctypes.data
        out = np.empty(int(lib().osp_gib_encoded_size(self.L)), dtype=np.uint8)
        _check(lib().osp_group_step_host(self._h, ptr, ld, out.ctypes.data_as(P(ctypes.c_uint8)),
                                         pout, _stream(stream)))
        return out.tobytes()

    def read_gib(self, stream=None) -> dict:
        L = self.L
        flags = np.empty(L, dtype=np.uint8)
        order = np.empty(L, dtype=np.int32)
        chunk_of = np.empty(L, dtype=np.int32)
        n_order, n_used, tag, deferred = c_i64(), c_int(), c_u32(), c_u64()
        _check(lib().osp_group_read_gib(self._h, flags.ctypes.data_as(P(ctypes.c_uint8)),
                                        order.ctypes.data_as(P(ctypes.c_int32)),
                                        ctypes.byref(n_order),
                                        chunk_of.ctypes.data_as(P(ctypes.c_int32)),
                                        ctypes.byref(n_used), ctypes.byref(tag),
                                        ctypes.byref(deferred), _stream(stream)))
        return dict(flags=flags, order=order[: n_order.value].copy(), chunk_of=chunk_of,
                    n_used=int(n_used.value), tag=int(tag.value),
                    deferred_bytes=int(deferred.value))

    def stats(self, stream=None) -> dict:
        r, fl, fr = c_u64(), c_u64(), c_u64()
        _check(lib().osp_group_stats(self._h, ctypes.byref(r), ctypes.byref(fl), ctypes.byref(fr),
                                     _stream(stream)))
        return dict(resolved=int(r.value), fallback_layers=int(fl.value),
                    fallback_resolves=int(fr.value))

    def deferred_history(self, first_tag: int, n: int, stream=None) -> np.ndarray:
        out = np.zeros(max(n, 1), dtype=np.uint64)
        _check(lib().osp_group_deferred_history(self._h, first_tag, n,
                                                out.ctypes.data_as(P(c_u64)), _stream(stream)))
        return out[:n]

    def geometry(self) -> dict:
        t, nt, gb, bt = c_u32(), c_u64(), c_int(), c_int()
        _check(lib().osp_group_geometry(self._h, ctypes.byref(t), ctypes.byref(nt),
                                        ctypes.byref(gb), ctypes.byref(bt)))
        return dict(tile_elems=int(t.value), n_tiles=int(nt.value), grid_blocks=int(gb.value),
                    block_threads=int(bt.value), stage_kernels=self.stage_kernels)

    @property
    def single_launch(self) -> bool:
        """True when step() runs as one single-CTA launch (OSP_GROUP_SMALL)."""
        return bool(lib().osp_group_flags(self._h) & _capi.GROUP_SMALL)

    @property
    def stage_kernels(self) -> str:
        """"tma-staged" or "register-staged"."""
        f = lib().osp_group_flags(self._h)
        return "tma-staged" if f & _capi.GROUP_TMA else "register-staged"

    def close(self):
        """Destroy now (views taken from this group must not be used afterwards);
        otherwise the handle goes when the group and its views are gone."""
        hnd = getattr(self, "_hnd", None)
        if hnd is not None and getattr(self, "_owned", True):
            hnd.close()
        self._h = None
