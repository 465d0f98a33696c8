"""Multi-GPU OSP: one process per GPU, PS sharded one shard per GPU (osp_shard_*).

torch.distributed is plumbing only: it exchanges the 512-byte CUDA-IPC handles
once at setup and provides the host barrier / max-over-ranks timing. The
exchange itself (push = reduce-scatter, pull = all-gather) happens inside the
library's kernels over NVLink peer memory.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from ._capi import P, c_dbl, c_u64, c_void_p
from .osp import (ConfigError, OspGroup, ShapeError, Partition, _check, _dev_f32, _Handle, _ptr, _stream,
                  _view, lib)


class ShardGroup:
    """This rank's slice of an N-worker OSP job spread over `world` GPUs."""

    def __init__(self, part: Partition, n_workers: int, weights: Optional[Sequence[float]] = None,
                 n_chunks: int = 4, init_params: Optional[torch.Tensor] = None,
                 tile_elems: int = 0, sgd_lr: float = 0.0, rank: Optional[int] = None,
                 world: Optional[int] = None, group=None, defer_ics: bool = False, stream=None):
        """defer_ics: stage 1 exchanges the barrier layers only and stage 2 the
        deferred chunks (OSP_SHARD_DEFER_ICS: the ICS traffic can run beside the
        next iteration's compute); default: one exchange per iteration in stage 1,
        stage 2 a local broadcast of the carry. Identical results."""
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        if n_workers % self.world:
            raise ConfigError("workers must split evenly across ranks")
        self.part = part
        self.N = n_workers
        self.n_loc = n_workers // self.world
        self.M = part.total_count()
        self.n_chunks = n_chunks
        w = list(weights) if weights is not None else [1.0 / n_workers] * n_workers
        self._w = (c_dbl * n_workers)(*w)
        cfg = _capi.osp_shard_config(self.world, self.rank, n_workers, ctypes.cast(self._w, P(c_dbl)),
                                     n_chunks, tile_elems, sgd_lr,
                                     _capi.SHARD_DEFER_ICS if defer_ics else 0)
        init = None
        if init_params is not None:
            _dev_f32(init_params, "init_params")
            if init_params.numel() != self.M:
                raise ShapeError("init params do not match the partition")
            init = _ptr(init_params)
        h = c_void_p()
        _check(lib().osp_shard_create(part.handle, ctypes.byref(cfg), init, _stream(stream),
                                      ctypes.byref(h)))
        self._h = h
        self._hnd = _Handle(h, "osp_shard_destroy")
        self.local = OspGroup._borrow(lib().osp_shard_group(h), part, self.n_loc, n_chunks,
                                      self._hnd)
        ld = c_u64()
        self._x = []
        for b in range(2):
            ptr = lib().osp_shard_deltas(h, b, ctypes.byref(ld))
            self._x.append(_view(ptr, (self.n_loc, self.M), "<f4", strides=(int(ld.value) * 4, 4),
                                 owner=self._hnd))
        self.ldX = int(ld.value)

    def export_handle(self) -> bytes:
        buf = np.zeros(_capi.SHARD_HANDLE_BYTES, dtype=np.uint8)
        _check(lib().osp_shard_export(self._h, buf.ctypes.data_as(P(ctypes.c_uint8))))
        return buf.tobytes()

    def connect(self, handles: Sequence[bytes]):
        if len(handles) != self.world:
            raise ConfigError("need one handle per rank")
        blob = np.frombuffer(b"".join(handles), dtype=np.uint8).copy()
        _check(lib().osp_shard_connect(self._h, blob.ctypes.data_as(P(ctypes.c_uint8))))

    def connect_via(self, group=None):
        """Exchange handles with torch.distributed (all_gather_object) and connect."""
        mine = self.export_handle()
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self.connect(allh)

    # ---- data -------------------------------------------------------------
    def deltas(self, buf: int) -> torch.Tensor:
        """This rank's workers' delta rows [N/P, M] of buffer 0/1 (write into it)."""
        return self._x[buf]

    def fill_synth(self, seed: int, iteration: int, buf: int, stream=None):
        """Reference synthetic deltas (runner.cpp:312-321) of this rank's workers."""
        _check(lib().osp_synth_deltas_range(seed, self.rank * self.n_loc, self.n_loc, iteration,
                                            self.M, _ptr(self._x[buf]), self.ldX, _stream(stream)))

    # ---- the step ------------------------------------------------------------
    def set_budget(self, budget: int, stream=None):
        self.local.set_budget(budget, stream)

    def stage1(self, buf: int, stream=None):
        _check(lib().osp_shard_stage1(self._h, buf, _stream(stream)))

    def stage2(self, buf: int, c0: int = 0, c1: Optional[int] = None, stream=None):
        c1 = self.n_chunks if c1 is None else c1
        _check(lib().osp_shard_stage2(self._h, c0, c1, buf, _stream(stream)))

    def resolve(self, buf: int, stream=None):
        _check(lib().osp_shard_resolve(self._h, buf, _stream(stream)))

    def step(self, buf: int, stream=None):
        _check(lib().osp_shard_step(self._h, buf, _stream(stream)))

    def profile(self, buf: int, stream=None) -> dict:
        """One step with events between the phases (ms per phase)."""
        out = (ctypes.c_float * 8)()
        _check(lib().osp_shard_profile(self._h, buf, out, _stream(stream)))
        return {n: float(v) for n, v in zip(["stage1", "stage2", "resolve"], out)}

    def debug_counters(self):
        """Exchange-kernel counters (OSP_SHARD_DEBUG=1 at create) or None."""
        out = (c_u64 * 16)()
        if not lib().osp_shard_debug_counters(self._h, out):
            return None
        names = ["b_block_cycles", "empty_wait_cycles", "full_wait_cycles", "fence_cycles",
                 "producer_cycles", "b_blocks", "a_items", "b_items", "l_items", "flushes",
                 "max_cta_ns", "next_item_cycles", "issue_cycles"]
        return {n: int(v) for n, v in zip(names, out)}

    def debug_trace(self):
        """OSP_SHARD_DEBUG=2, chain form: [8, NT] globaltimer stamps of the last
        stage-1 launch (see osp_shard_debug_trace), or None."""
        n = int(lib().osp_shard_debug_trace(self._h, None, 0))
        if not n:
            return None
        out = np.zeros(n, dtype=np.uint64)
        lib().osp_shard_debug_trace(self._h, out.ctypes.data_as(P(c_u64)), n)
        return out.reshape(8, n // 8)

    @property
    def deferred_ics(self) -> bool:
        """True: stage 2 exchanges the deferred layers; False: single exchange."""
        return bool(lib().osp_shard_deferred_ics(self._h))

    @property
    def sync_form(self) -> str:
        """Exchange synchronisation: 'tile' (per-tile flags), 'barrier' (own tiles,
        then a cross-GPU signal) or 'chain' (stage 1 as a reduction chain)."""
        return {0: "tile", 1: "barrier", 2: "chain"}[lib().osp_shard_sync_form(self._h)]

    @property
    def mode(self) -> str:
        return ("deferred ICS: stage 1 exchanges the RS layers, stage 2 the ICS chunks"
                if self.deferred_ics else
                "single exchange: every tile in stage 1 (ICS carry), stage 2 local")

    def solo_agg(self, stage: int, buf: int, stream=None):
        """Diagnostics: this rank's push/pull of a stage alone (osp_shard_solo_agg)."""
        _check(lib().osp_shard_solo_agg(self._h, stage, buf, _stream(stream)))

    def check(self, stream=None):
        _check(lib().osp_shard_check(self._h, _stream(stream)))

    @property
    def global_params(self) -> torch.Tensor:
        return self.local.global_params

    @property
    def worker_params(self) -> torch.Tensor:
        return self.local.worker_params

    def read_gib(self):
        return self.local.read_gib()

    def close(self):
        """Destroy now (views must not be used afterwards); otherwise the handle
        goes with the last of this object, its local group and their views."""
        hnd = getattr(self, "_hnd", None)
        if hnd is not None:
            if getattr(self, "local", None) is not None:
                self.local._h = None
            hnd.close()
        self._h = None
