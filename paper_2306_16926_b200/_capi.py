"""ctypes binding of the C-ABI (include/osp_c.h) — the only way Python reaches
the CUDA path. Loading fails loudly when the in-tree library is missing: there
is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OSP_LIB_VARIANT=checked: the bounds-checked build (make checked), for the
# test suite on the GPU pool, where compute-sanitizer is not available
LIB_PATH = os.path.join(_HERE, "libosp_b200_checked.so"
                        if os.environ.get("OSP_LIB_VARIANT") == "checked" else "libosp_b200.so")

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_float = ctypes.c_float
P = ctypes.POINTER


class osp_group_config(ctypes.Structure):
    _fields_ = [("n_workers", c_int), ("weights", P(c_dbl)), ("n_chunks", c_int),
                ("tile_elems", c_u32), ("sgd_lr", c_dbl), ("flags", c_u32)]


GROUP_TMA = 1
GROUP_REGISTER = 2
GROUP_NO_CARRY = 4
GROUP_NO_SMALL = 8
GROUP_SMALL = 16


class osp_shard_config(ctypes.Structure):
    _fields_ = [("world", c_int), ("rank", c_int), ("n_workers", c_int), ("weights", P(c_dbl)),
                ("n_chunks", c_int), ("tile_elems", c_u32), ("sgd_lr", c_dbl), ("flags", c_u32)]


SHARD_HANDLE_BYTES = 512
SHARD_DEFER_ICS = 1


class osp_sgu_schedule(ctypes.Structure):
    _fields_ = [("u_max", c_u64), ("has_initial_loss", c_int), ("initial_loss", c_dbl),
                ("current_budget", c_u64), ("epoch", c_u64)]


# name -> (restype, argtypes)
_SIGS = {
    "osp_last_error": (ctypes.c_char_p, []),
    "osp_status_name": (ctypes.c_char_p, [c_int]),
    "osp_abi_version": (c_int, []),
    "osp_device_info": (c_int, [P(c_int), P(c_int), P(c_int), P(c_int)]),
    "osp_partition_create": (c_int, [P(c_u64), c_u64, c_u32, P(c_void_p)]),
    "osp_partition_destroy": (None, [c_void_p]),
    "osp_partition_layer_count": (c_u64, [c_void_p]),
    "osp_partition_total_count": (c_u64, [c_void_p]),
    "osp_partition_total_bytes": (c_u64, [c_void_p]),
    "osp_partition_bytes_per_element": (c_u32, [c_void_p]),
    "osp_partition_layer": (c_int, [c_void_p, c_i64, P(c_u64), P(c_u64)]),
    "osp_device_alloc": (c_int, [c_u64, P(c_void_p)]),
    "osp_device_free": (c_int, [c_void_p]),
    "osp_memcpy_h2d": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_memcpy_d2d": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_memset": (c_int, [c_void_p, c_int, c_u64, c_void_p]),
    "osp_stream_sync": (c_int, [c_void_p]),
    "osp_aggregate_layer": (c_int, [P(c_void_p), c_int, P(c_dbl), c_u64, c_void_p, c_void_p]),
    "osp_aggregate_apply_layers": (c_int, [c_void_p, P(c_void_p), c_int, P(c_dbl),
                                           P(ctypes.c_int32), c_i64, c_void_p, c_void_p,
                                           c_void_p]),
    "osp_apply_delta": (c_int, [c_void_p, c_void_p, c_u64, c_float, c_void_p]),
    "osp_sgd_delta": (c_int, [c_void_p, c_u64, c_dbl, c_void_p, c_void_p]),
    "osp_mlp_create": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_u64,
                               P(c_void_p)]),
    "osp_mlp_destroy": (None, [c_void_p]),
    "osp_mlp_num_params": (c_u64, [c_void_p]),
    "osp_mlp_grad": (c_int, [c_void_p, c_void_p, c_u64, c_int, c_void_p, c_int, c_void_p, c_u64,
                             c_void_p, c_void_p]),
    "osp_mlp_check": (c_int, [c_void_p, c_void_p]),
    "osp_synth_delta": (c_int, [c_u64, c_u64, c_u64, c_u64, c_u64, c_void_p, c_void_p]),
    "osp_synth_deltas": (c_int, [c_u64, c_int, c_u64, c_u64, c_void_p, c_u64, c_void_p]),
    "osp_lgp_partial": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P(ctypes.c_uint8),
                                c_void_p, c_void_p]),
    "osp_lgp_correct": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P(ctypes.c_int32),
                                c_i64, c_void_p]),
    "osp_pgp_layer_importance": (c_int, [c_void_p, c_void_p, c_void_p, P(c_dbl), c_void_p]),
    "osp_pgp_rank_gib": (c_int, [c_void_p, c_void_p, c_void_p, c_u64, P(c_dbl), P(ctypes.c_int32),
                                 P(c_i64), P(ctypes.c_uint8), c_void_p]),
    "osp_rank_and_gib": (c_int, [c_void_p, P(c_dbl), c_u64, P(ctypes.c_int32),
                                 P(ctypes.c_uint8), c_void_p]),
    "osp_split_for_sync": (c_int, [c_void_p, P(ctypes.c_uint8), P(ctypes.c_int32), c_i64,
                                   c_int, P(ctypes.c_int32), P(c_i64), P(ctypes.c_int32),
                                   P(c_int)]),
    "osp_gib_encoded_size": (c_u64, [c_u64]),
    "osp_gib_encode": (c_int, [c_u32, c_u64, P(ctypes.c_uint8), P(ctypes.c_uint8), c_u64]),
    "osp_gib_decode": (c_int, [P(ctypes.c_uint8), c_u64, P(c_u32), P(c_u32), P(ctypes.c_uint8),
                               c_u64]),
    "osp_gib_wire_size": (c_u64, [c_u64, c_u64]),
    "osp_gib_wire_encode": (c_int, [c_u32, c_u64, P(ctypes.c_uint8), P(ctypes.c_int32), c_u64,
                                    P(ctypes.c_uint8), c_u64, P(c_u64)]),
    "osp_gib_wire_decode": (c_int, [P(ctypes.c_uint8), c_u64, P(c_u32), P(c_u32),
                                    P(ctypes.c_uint8), c_u64, P(ctypes.c_int32), c_u64, P(c_i64)]),
    "osp_group_gib_wire": (c_int, [c_void_p, P(ctypes.c_uint8), c_u64, P(c_u64), c_void_p]),
    "osp_group_gib_wire_device": (c_void_p, [c_void_p, P(c_u64)]),
    "osp_group_set_gib_wire": (c_int, [c_void_p, P(ctypes.c_uint8), c_u64, c_void_p]),
    "osp_payload_encoded_size": (c_u64, [c_void_p, P(ctypes.c_int32), c_i64]),
    "osp_encode_payload": (c_int, [c_void_p, c_void_p, P(ctypes.c_int32), c_i64, ctypes.c_uint8,
                                   c_u32, c_void_p, c_u64, P(c_u64), c_void_p]),
    "osp_decode_payload": (c_int, [c_void_p, c_void_p, c_u64, c_void_p, P(ctypes.c_uint8),
                                   P(c_u32), P(ctypes.c_int32), c_i64, P(c_i64), c_void_p]),
    "osp_compute_umax": (c_int, [c_dbl, c_dbl, c_dbl, c_dbl, c_int, c_u64, c_int, P(c_u64)]),
    "osp_tune_sgu": (c_int, [P(osp_sgu_schedule), c_u64, c_dbl, P(c_u64)]),
    "osp_group_create": (c_int, [c_void_p, P(osp_group_config), c_void_p, c_void_p,
                                 P(c_void_p)]),
    "osp_group_destroy": (None, [c_void_p]),
    "osp_group_set_budget": (c_int, [c_void_p, c_u64, c_void_p]),
    "osp_group_set_gib": (c_int, [c_void_p, P(ctypes.c_uint8), P(ctypes.c_int32), c_i64, c_u32,
                                  c_void_p]),
    "osp_group_stage1": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_stage2_chunk": (c_int, [c_void_p, c_int, c_void_p, c_u64, c_void_p]),
    "osp_group_stage2_all": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_resolve": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_step": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_stages": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_stage2_resolve": (c_int, [c_void_p, c_void_p, c_u64, c_void_p]),
    "osp_group_set_momentum": (c_int, [c_void_p, c_dbl, c_void_p]),
    "osp_group_step_host": (c_int, [c_void_p, c_void_p, c_u64, P(ctypes.c_uint8), c_void_p,
                                    c_void_p]),
    "osp_group_step_host_async": (c_int, [c_void_p, c_void_p, c_u64, c_void_p, c_void_p,
                                          c_void_p]),
    "osp_group_host_wait": (c_int, [c_void_p]),
    "osp_group_global": (c_void_p, [c_void_p]),
    "osp_group_worker_params": (c_void_p, [c_void_p, P(c_u64)]),
    "osp_group_scores": (c_void_p, [c_void_p]),
    "osp_group_read_gib": (c_int, [c_void_p, P(ctypes.c_uint8), P(ctypes.c_int32), P(c_i64),
                                   P(ctypes.c_int32), P(c_int), P(c_u32), P(c_u64), c_void_p]),
    "osp_group_stats": (c_int, [c_void_p, P(c_u64), P(c_u64), P(c_u64), c_void_p]),
    "osp_group_deferred_history": (c_int, [c_void_p, c_u32, c_int, P(c_u64), c_void_p]),
    "osp_group_geometry": (c_int, [c_void_p, P(c_u32), P(c_u64), P(c_int), P(c_int)]),
    "osp_group_flags": (c_u32, [c_void_p]),
    "osp_shard_create": (c_int, [c_void_p, P(osp_shard_config), c_void_p, c_void_p,
                                 P(c_void_p)]),
    "osp_shard_destroy": (None, [c_void_p]),
    "osp_shard_handle_size": (c_u64, []),
    "osp_shard_export": (c_int, [c_void_p, P(ctypes.c_uint8)]),
    "osp_shard_connect": (c_int, [c_void_p, P(ctypes.c_uint8)]),
    "osp_shard_deltas": (c_void_p, [c_void_p, c_int, P(c_u64)]),
    "osp_shard_group": (c_void_p, [c_void_p]),
    "osp_shard_stage1": (c_int, [c_void_p, c_int, c_void_p]),
    "osp_shard_stage2": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p]),
    "osp_shard_resolve": (c_int, [c_void_p, c_int, c_void_p]),
    "osp_shard_step": (c_int, [c_void_p, c_int, c_void_p]),
    "osp_shard_check": (c_int, [c_void_p, c_void_p]),
    "osp_shard_deferred_ics": (c_int, [c_void_p]),
    "osp_shard_sync_form": (c_int, [c_void_p]),
    "osp_shard_debug_counters": (c_int, [c_void_p, P(c_u64)]),
    "osp_shard_debug_trace": (c_u64, [c_void_p, P(c_u64), c_u64]),
    "osp_shard_profile": (c_int, [c_void_p, c_int, P(ctypes.c_float), c_void_p]),
    "osp_shard_solo_agg": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "osp_synth_deltas_range": (c_int, [c_u64, c_int, c_int, c_u64, c_u64, c_void_p, c_u64,
                                       c_void_p]),
}

EXPORTED = sorted(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the in-tree CUDA library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make lib` (or __graft_entry__.build()). "
            "The OSP sync path has no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
