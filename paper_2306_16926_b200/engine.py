"""ctypes mirror of include/osp_engine.h: the message-level OspWorker / OspServer
engines (reference protocol.hpp:65-254) over libpslab_b200.so, whose state is
device-resident and whose arithmetic runs in the sm_100a kernels.

Same names and message flow as the reference engines; messages are opaque
handles that encode to the reference wire formats. Errors raise the osp.*
exception classes (1:1 with pslab::Error).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER as P
from ctypes import c_double, c_float, c_int, c_int32, c_uint8, c_uint32, c_uint64, c_void_p
from typing import List, Optional, Sequence

import numpy as np

from . import osp

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpslab_b200.so")


class ServerConfig(ctypes.Structure):
    _fields_ = [("n_workers", c_int), ("weights", P(c_double)), ("u_max", c_uint64),
                ("iterations_per_epoch", c_uint64), ("has_fixed_budget", c_int),
                ("fixed_budget_bytes", c_uint64)]


_SIGS = {
    "osp_engine_last_error": (ctypes.c_char_p, []),
    "osp_engine_partition_create": (c_int, [P(c_uint64), c_uint64, c_uint32, P(c_void_p)]),
    "osp_engine_partition_destroy": (None, [c_void_p]),
    "osp_engine_partition_total_count": (c_uint64, [c_void_p]),
    "osp_msg_kind": (c_int, [c_void_p]),
    "osp_msg_iteration": (c_uint32, [c_void_p]),
    "osp_msg_from": (c_int, [c_void_p]),
    "osp_msg_scalar": (c_double, [c_void_p]),
    "osp_msg_layer_count": (c_int, [c_void_p]),
    "osp_msg_size_bytes": (c_uint64, [c_void_p, c_void_p]),
    "osp_msg_encode": (c_int, [c_void_p, P(c_uint8), c_uint64, P(c_uint64)]),
    "osp_msg_decode": (c_int, [P(c_uint8), c_uint64, c_int, P(c_void_p)]),
    "osp_msg_gib": (c_int, [c_void_p, P(c_uint8), c_uint64, P(c_uint64)]),
    "osp_msg_rank_order": (c_int, [c_void_p, P(c_int32), c_uint64, P(c_uint64)]),
    "osp_msg_destroy": (None, [c_void_p]),
    "osp_worker_create": (c_int, [c_void_p, c_int, P(c_float), c_double, P(c_void_p)]),
    "osp_worker_destroy": (None, [c_void_p]),
    "osp_worker_compute_done": (c_int, [c_void_p, c_uint64, P(c_float), c_double, c_int,
                                        P(c_void_p), P(c_void_p), P(c_void_p), c_int, P(c_int)]),
    "osp_worker_on_pull_important": (c_int, [c_void_p, c_void_p, P(c_int)]),
    "osp_worker_on_ics_global_chunk": (c_int, [c_void_p, c_void_p]),
    "osp_worker_stashed_pull_ready": (c_int, [c_void_p]),
    "osp_worker_apply_stashed_pull": (c_int, [c_void_p]),
    "osp_worker_on_gib_update": (c_int, [c_void_p, c_void_p]),
    "osp_worker_iteration": (c_uint64, [c_void_p]),
    "osp_worker_pending_empty": (c_int, [c_void_p]),
    "osp_worker_params": (c_int, [c_void_p, P(c_float)]),
    "osp_server_create": (c_int, [c_void_p, P(c_float), P(ServerConfig), P(c_void_p)]),
    "osp_server_destroy": (None, [c_void_p]),
    "osp_server_on_push_important": (c_int, [c_void_p, c_void_p, P(c_void_p), P(c_void_p),
                                             P(c_void_p)]),
    "osp_server_on_push_ics_chunk": (c_int, [c_void_p, c_void_p, P(c_void_p), P(c_void_p),
                                             P(c_void_p)]),
    "osp_server_on_loss_report": (c_int, [c_void_p, c_void_p]),
    "osp_server_set_umax": (c_int, [c_void_p, c_uint64]),
    "osp_server_global_params": (c_int, [c_void_p, P(c_float)]),
    "osp_server_resolved_count": (c_uint64, [c_void_p]),
    "osp_server_dropped_stale": (c_uint64, [c_void_p]),
    "osp_server_budget_for_epoch": (c_uint64, [c_void_p, c_uint64]),
    "osp_server_epoch_of_iteration": (c_uint64, [c_void_p, c_uint64]),
}
EXPORTED = sorted(_SIGS)
_lib = None


def lib():
    global _lib
    if _lib is None:
        osp.lib()  # libosp_b200.so first (the façade links against it)
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} missing: run `make facade`")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _check(status: int):
    if status != 0:
        msg = lib().osp_engine_last_error().decode(errors="replace")
        raise osp._STATUS.get(status, osp.Error)(msg)


def _fvec(v: Optional[np.ndarray], n: int):
    if v is None:
        return None, None
    a = np.ascontiguousarray(v, dtype=np.float32)
    if a.size != n:
        raise osp.ShapeError(f"vector of {a.size} floats for a partition of {n}")
    return a, a.ctypes.data_as(P(c_float))


class Partition:
    """make_partition (param.hpp:43-46)."""

    def __init__(self, layer_counts: Sequence[int], bytes_per_element: int = 4):
        counts = (c_uint64 * len(layer_counts))(*[int(c) for c in layer_counts])
        h = c_void_p()
        _check(lib().osp_engine_partition_create(counts, len(layer_counts), bytes_per_element,
                                                 ctypes.byref(h)))
        self._h = h.value
        self.total = int(lib().osp_engine_partition_total_count(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.osp_engine_partition_destroy(self._h)
            self._h = None


class Message:
    """An engine message (message.hpp:30-38); owns its handle."""
    KINDS = ["PushImportant", "PushIcsChunk", "PullImportant", "IcsGlobalChunk", "GibUpdate",
             "LossReport", "PushFull", "PullFull"]

    def __init__(self, h):
        self._h = h

    @property
    def kind(self) -> str:
        return self.KINDS[lib().osp_msg_kind(self._h)]

    @property
    def iteration(self) -> int:
        return int(lib().osp_msg_iteration(self._h))

    @property
    def from_worker(self) -> int:
        return int(lib().osp_msg_from(self._h))

    @property
    def scalar(self) -> float:
        return float(lib().osp_msg_scalar(self._h))

    @property
    def layer_count(self) -> int:
        return int(lib().osp_msg_layer_count(self._h))

    def size_bytes(self, part: Partition) -> int:
        return int(lib().osp_msg_size_bytes(self._h, part._h))

    def encode(self) -> bytes:
        n = c_uint64()
        _check(lib().osp_msg_encode(self._h, None, 0, ctypes.byref(n)))
        buf = (c_uint8 * n.value)()
        _check(lib().osp_msg_encode(self._h, buf, n.value, ctypes.byref(n)))
        return bytes(buf)

    @classmethod
    def decode(cls, data: bytes, from_worker: int = -1) -> "Message":
        buf = (c_uint8 * len(data)).from_buffer_copy(data)
        h = c_void_p()
        _check(lib().osp_msg_decode(buf, len(data), from_worker, ctypes.byref(h)))
        return cls(h.value)

    def gib(self) -> bytes:
        n = c_uint64()
        _check(lib().osp_msg_gib(self._h, None, 0, ctypes.byref(n)))
        buf = (c_uint8 * n.value)()
        _check(lib().osp_msg_gib(self._h, buf, n.value, ctypes.byref(n)))
        return bytes(buf)

    def rank_order(self) -> np.ndarray:
        n = c_uint64()
        _check(lib().osp_msg_rank_order(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.int32)
        _check(lib().osp_msg_rank_order(self._h, out.ctypes.data_as(P(c_int32)), n.value,
                                        ctypes.byref(n)))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.osp_msg_destroy(self._h)
            self._h = None


def _opt(h: c_void_p) -> Optional[Message]:
    return Message(h.value) if h.value else None


class OspWorker:
    """protocol.hpp:71-109."""

    def __init__(self, part: Partition, worker_id: int, init_params=None, subset_weight=1.0):
        self.part = part
        a, p = _fvec(init_params, part.total)
        h = c_void_p()
        _check(lib().osp_worker_create(part._h, worker_id, p, float(subset_weight), ctypes.byref(h)))
        self._h = h.value

    def on_compute_done(self, iteration: int, delta, loss: float, n_chunks: int):
        """-> (rs_push, loss_report, [ics chunk messages])"""
        a, p = _fvec(delta, self.part.total)
        rs, lr = c_void_p(), c_void_p()
        chunks = (c_void_p * max(n_chunks, 1))()
        n = c_int()
        _check(lib().osp_worker_compute_done(self._h, iteration, p, float(loss), n_chunks,
                                             ctypes.byref(rs), ctypes.byref(lr), chunks,
                                             max(n_chunks, 1), ctypes.byref(n)))
        return Message(rs.value), Message(lr.value), [Message(chunks[j]) for j in range(n.value)]

    def on_pull_important(self, pull: Message) -> bool:
        applied = c_int()
        _check(lib().osp_worker_on_pull_important(self._h, pull._h, ctypes.byref(applied)))
        return bool(applied.value)

    def on_ics_global_chunk(self, chunk: Message):
        _check(lib().osp_worker_on_ics_global_chunk(self._h, chunk._h))

    def stashed_pull_ready(self) -> bool:
        return bool(lib().osp_worker_stashed_pull_ready(self._h))

    def apply_stashed_pull(self):
        _check(lib().osp_worker_apply_stashed_pull(self._h))

    def on_gib_update(self, msg: Message):
        _check(lib().osp_worker_on_gib_update(self._h, msg._h))

    @property
    def iteration(self) -> int:
        return int(lib().osp_worker_iteration(self._h))

    @property
    def pending_empty(self) -> bool:
        return bool(lib().osp_worker_pending_empty(self._h))

    def params(self) -> np.ndarray:
        out = np.zeros(self.part.total, np.float32)
        _check(lib().osp_worker_params(self._h, out.ctypes.data_as(P(c_float))))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.osp_worker_destroy(self._h)
            self._h = None


class OspServer:
    """protocol.hpp:126-180."""

    def __init__(self, part: Partition, weights: Sequence[float], init_global=None, u_max: int = 0,
                 iterations_per_epoch: int = 1, fixed_budget_bytes: Optional[int] = None):
        self.part = part
        self._w = (c_double * len(weights))(*weights)
        cfg = ServerConfig(len(weights), ctypes.cast(self._w, P(c_double)), int(u_max),
                           int(iterations_per_epoch), 0 if fixed_budget_bytes is None else 1,
                           0 if fixed_budget_bytes is None else int(fixed_budget_bytes))
        a, p = _fvec(init_global, part.total)
        h = c_void_p()
        _check(lib().osp_server_create(part._h, p, ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h.value

    def _out(self, fn, msg: Message):
        pull, ics, gib = c_void_p(), c_void_p(), c_void_p()
        _check(fn(self._h, msg._h, ctypes.byref(pull), ctypes.byref(ics), ctypes.byref(gib)))
        return {"pull_important": _opt(pull), "ics_broadcast": _opt(ics), "gib_update": _opt(gib)}

    def on_push_important(self, msg: Message) -> dict:
        return self._out(lib().osp_server_on_push_important, msg)

    def on_push_ics_chunk(self, msg: Message) -> dict:
        return self._out(lib().osp_server_on_push_ics_chunk, msg)

    def on_loss_report(self, msg: Message):
        _check(lib().osp_server_on_loss_report(self._h, msg._h))

    def set_umax(self, u_max: int):
        _check(lib().osp_server_set_umax(self._h, int(u_max)))

    def global_params(self) -> np.ndarray:
        out = np.zeros(self.part.total, np.float32)
        _check(lib().osp_server_global_params(self._h, out.ctypes.data_as(P(c_float))))
        return out

    @property
    def resolved_count(self) -> int:
        return int(lib().osp_server_resolved_count(self._h))

    @property
    def dropped_stale(self) -> int:
        return int(lib().osp_server_dropped_stale(self._h))

    def budget_for_epoch(self, epoch: int) -> int:
        return int(lib().osp_server_budget_for_epoch(self._h, epoch))

    def epoch_of_iteration(self, iteration: int) -> int:
        return int(lib().osp_server_epoch_of_iteration(self._h, iteration))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.osp_server_destroy(self._h)
            self._h = None


def run_synchronous_iteration(server: OspServer, workers: List[OspWorker], iteration: int,
                              deltas, loss: float, n_chunks: int):
    """One OSP iteration in the reference harness's synchronous message order
    (oracle/ref_driver.cpp: loss reports, RS pushes, pull broadcast, ICS chunk j
    of every worker, GIB broadcast). Returns the worker params after stage 1."""
    outs = [w.on_compute_done(iteration, deltas[k], loss, n_chunks) for k, w in enumerate(workers)]
    for rs, lr, _ in outs:
        server.on_loss_report(lr)
    pull = gib = None
    for rs, _, _ in outs:
        o = server.on_push_important(rs)
        if o["pull_important"] is not None:
            pull = o["pull_important"]
        if o["gib_update"] is not None:
            gib = o["gib_update"]
        if o["ics_broadcast"] is not None:
            raise osp.ProtocolError("ICS broadcast at the barrier")
    if pull is None:
        raise osp.ProtocolError(f"barrier did not close at iteration {iteration}")
    for w in workers:
        if not w.on_pull_important(pull):
            raise osp.ProtocolError("pull stashed in a synchronous iteration")
    stage1 = [w.params() for w in workers]
    for j in range(len(outs[0][2])):
        for k in range(len(workers)):
            o = server.on_push_ics_chunk(outs[k][2][j])
            if o["ics_broadcast"] is not None:
                for w in workers:
                    w.on_ics_global_chunk(o["ics_broadcast"])
            if o["gib_update"] is not None:
                gib = o["gib_update"]
            if o["pull_important"] is not None:
                raise osp.ProtocolError("pull during ICS")
    if gib is None or server.resolved_count != iteration + 1:
        raise osp.ProtocolError(f"iteration {iteration} did not resolve")
    for w in workers:
        w.on_gib_update(gib)
    return stage1, gib
