"""ctypes/numpy front of the C oracle (oracle/osp_oracle.c).

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py — never by the product package. Each wrapper names
the reference function (file:line under /root/reference/proj) it restates.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> str:
    """Compile liboracle.so (gcc, -ffp-contract=off) if missing or stale."""
    src = os.path.join(_HERE, "osp_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oo_derive_seed.restype = ctypes.c_uint64
        L.oo_derive_seed.argtypes = [ctypes.c_uint64] * 4
        L.oo_synth_delta.argtypes = [ctypes.c_uint64] * 5 + [_f32p]
        L.oo_sgd_delta.argtypes = [_f32p, ctypes.c_uint64, ctypes.c_double, _f32p]
        L.oo_lr_at_epoch.restype = ctypes.c_double
        L.oo_lr_at_epoch.argtypes = [ctypes.c_double, ctypes.c_uint64]
        L.oo_aggregate_layer.restype = ctypes.c_int
        L.oo_aggregate_layer.argtypes = [ctypes.c_int, ctypes.POINTER(_f32p), _f64p,
                                         ctypes.c_uint64, _f32p]
        L.oo_pgp.argtypes = [ctypes.c_int64, _u64p, _f32p, _f32p, _f64p]
        L.oo_pgp_accum.argtypes = [ctypes.c_uint64, _f32p, _f32p, _f64p]
        L.oo_rank.argtypes = [ctypes.c_int64, _f64p, _i32p]
        L.oo_build_gib.argtypes = [ctypes.c_int64, _f64p, _u64p, ctypes.c_uint32,
                                   ctypes.c_uint64, _u8p]
        L.oo_gib_encoded_size.restype = ctypes.c_uint64
        L.oo_gib_encoded_size.argtypes = [ctypes.c_uint64]
        L.oo_gib_encode.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u8p, _u8p]
        L.oo_gib_decode.restype = ctypes.c_int
        L.oo_gib_decode.argtypes = [_u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32),
                                    ctypes.POINTER(ctypes.c_uint32), _u8p, ctypes.c_uint64]
        L.oo_split.restype = ctypes.c_int
        L.oo_split.argtypes = [ctypes.c_int64, _u64p, ctypes.c_uint32, _u8p, _i32p,
                               ctypes.c_int64, ctypes.c_int, _i32p, _i64p, _i32p]
        L.oo_compute_umax.restype = ctypes.c_uint64
        L.oo_compute_umax.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.oo_tune_sgu.restype = ctypes.c_int64
        L.oo_tune_sgu.argtypes = [_f64p, ctypes.POINTER(ctypes.c_int), ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_double]
        L.oo_encode_payload.restype = ctypes.c_uint64
        L.oo_encode_payload.argtypes = [ctypes.c_uint8, ctypes.c_uint32, ctypes.c_int64, _u64p,
                                        _f32p, _i32p, ctypes.c_int64, _u8p]
        L.oo_step.restype = ctypes.c_int
        L.oo_step.argtypes = [ctypes.c_int64, _u64p, ctypes.c_uint32, ctypes.c_int, _f64p,
                              _f32p, _f32p, _f32p, _u8p, _i32p, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_uint64, _f32p, _f32p, _f64p, _u8p, _i32p, _i64p, _i32p]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _c(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def derive_seed(root: int, tag: int, a: int = 0, b: int = 0) -> int:
    """rng.hpp:27-36"""
    return int(lib().oo_derive_seed(root, tag, a, b))


def synth_delta(seed: int, worker: int, iteration: int, n: int, first: int = 0) -> np.ndarray:
    """runner.cpp:312-321"""
    out = np.empty(n, dtype=np.float32)
    lib().oo_synth_delta(seed, worker, iteration, first, n, _p(out, _f32p))
    return out


def sgd_delta(grad, lr: float) -> np.ndarray:
    """learner.cpp:391-398"""
    g = _c(grad, np.float32)
    out = np.empty_like(g)
    lib().oo_sgd_delta(_p(g, _f32p), g.size, lr, _p(out, _f32p))
    return out


def lr_at_epoch(lr: float, epoch: int) -> float:
    """learner.cpp:400-403"""
    return float(lib().oo_lr_at_epoch(lr, epoch))


def aggregate_layer(contribs, weights) -> np.ndarray:
    """protocol.cpp:9-30 (raises ValueError where the reference throws ProtocolError)"""
    cs = [_c(c, np.float32) for c in contribs]
    w = _c(weights, np.float64)
    if len(cs) == 0 or len(cs) != w.size or any(c.size != cs[0].size for c in cs):
        raise ValueError("aggregation needs one same-sized contribution per worker")
    arr = (_f32p * len(cs))(*[_p(c, _f32p) for c in cs])
    out = np.empty(cs[0].size, dtype=np.float32)
    rc = lib().oo_aggregate_layer(len(cs), arr, _p(w, _f64p), cs[0].size, _p(out, _f32p))
    if rc != 0:
        raise ValueError("aggregation weights must sum > 0")
    return out


def pgp(counts, params, grads) -> np.ndarray:
    """importance.cpp:11-28"""
    c = _c(counts, np.uint64)
    p = _c(params, np.float32)
    g = _c(grads, np.float32)
    out = np.empty(c.size, dtype=np.float64)
    lib().oo_pgp(c.size, _p(c, _u64p), _p(p, _f32p), _p(g, _f32p), _p(out, _f64p))
    return out


def pgp_accum(params, grads, acc: float) -> float:
    """importance.cpp:20-25, continued: acc + the sequential sum over this piece"""
    p = _c(params, np.float32)
    g = _c(grads, np.float32)
    a = ctypes.c_double(acc)
    lib().oo_pgp_accum(p.size, _p(p, _f32p), _p(g, _f32p), ctypes.byref(a))
    return a.value


def rank(scores) -> np.ndarray:
    """importance.cpp:30-40"""
    s = _c(scores, np.float64)
    out = np.empty(s.size, dtype=np.int32)
    lib().oo_rank(s.size, _p(s, _f64p), _p(out, _i32p))
    return out


def build_gib(scores, counts, bpe: int, budget: int) -> np.ndarray:
    """importance.cpp:42-59 -> uint8 flags (1 = deferred to ICS)"""
    s = _c(scores, np.float64)
    c = _c(counts, np.uint64)
    out = np.empty(s.size, dtype=np.uint8)
    lib().oo_build_gib(s.size, _p(s, _f64p), _p(c, _u64p), bpe, budget, _p(out, _u8p))
    return out


def gib_encode(tag: int, flags) -> bytes:
    """importance.cpp:61-97"""
    f = _c(flags, np.uint8)
    n = int(lib().oo_gib_encoded_size(f.size))
    out = np.empty(n, dtype=np.uint8)
    lib().oo_gib_encode(tag, f.size, _p(f, _u8p), _p(out, _u8p))
    return out.tobytes()


def gib_decode(buf: bytes):
    """importance.cpp:99-117 -> (tag, flags); ValueError where the reference throws FormatError"""
    b = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
    if b.size < 8:
        raise ValueError("gib buffer truncated")
    cap = int.from_bytes(bytes(b[4:8]), "little")
    flags = np.zeros(max(cap, 1), dtype=np.uint8)
    tag = ctypes.c_uint32()
    nl = ctypes.c_uint32()
    rc = lib().oo_gib_decode(_p(b, _u8p), b.size, ctypes.byref(tag), ctypes.byref(nl),
                             _p(flags, _u8p), flags.size)
    if rc != 0:
        raise ValueError("gib bitmap truncated")
    return int(tag.value), flags[: nl.value].copy()


def split(counts, bpe: int, flags, ics_order, n_chunks: int):
    """protocol.cpp:122-166 -> (rs_ids, chunk_of, n_used_chunks)"""
    c = _c(counts, np.uint64)
    f = _c(flags, np.uint8)
    o = _c(ics_order if len(ics_order) else [0], np.int32)
    rs = np.empty(c.size + 1, dtype=np.int32)
    nrs = ctypes.c_int64()
    chunk_of = np.empty(c.size, dtype=np.int32)
    used = lib().oo_split(c.size, _p(c, _u64p), bpe, _p(f, _u8p), _p(o, _i32p), len(ics_order),
                          n_chunks, _p(rs, _i32p), ctypes.byref(nrs), _p(chunk_of, _i32p))
    if used < 0:
        raise ValueError("need at least one chunk slot")
    return rs[: nrs.value].copy(), chunk_of, int(used)


def compute_umax(bandwidth_bps, loss_rate, t_c, n_workers, model_bytes, eq5_literal=False) -> int:
    """tuning.cpp:8-21"""
    return int(lib().oo_compute_umax(bandwidth_bps, loss_rate, t_c, n_workers, model_bytes,
                                     1 if eq5_literal else 0))


class SguSchedule:
    """tuning.cpp:23-48"""

    def __init__(self, u_max: int):
        self.u_max = u_max
        self._init = ctypes.c_double(0.0)
        self._has = ctypes.c_int(0)

    @property
    def initial_loss(self):
        return self._init.value if self._has.value else None

    def tune(self, epoch: int, loss: float) -> int:
        rc = lib().oo_tune_sgu(ctypes.byref(self._init), ctypes.byref(self._has), self.u_max,
                               epoch, loss)
        if rc < 0:
            raise ValueError({-1: "ConfigError", -2: "NumericError", -3: "ProtocolError"}[int(rc)])
        return int(rc)


def encode_payload(kind: int, iteration: int, counts, values, ids) -> bytes:
    """message.cpp:53-78 (payload wire encoding of the listed layers of a flat vector)"""
    c = _c(counts, np.uint64)
    v = _c(values, np.float32)
    i = _c(ids if len(ids) else [0], np.int32)
    n = 7 + sum(8 + 4 * int(c[k]) for k in ids)
    out = np.zeros(n, dtype=np.uint8)
    got = lib().oo_encode_payload(kind, iteration, c.size, _p(c, _u64p), _p(v, _f32p),
                                  _p(i, _i32p), len(ids), _p(out, _u8p))
    assert got == n
    return out.tobytes()


def step(counts, bpe, weights, deltas, G, P, flags_in, order_in, n_chunks, budget):
    """One synchronous OSP iteration (protocol.cpp:172-447, order of oracle/ref_driver.cpp).

    deltas: [N, M] f32; G: [M] f32; P: [N, M] f32 (both updated in place).
    Returns dict(p_stage1, agg, scores, flags_out, order_out, chunk_of, n_chunks_used).
    """
    c = _c(counts, np.uint64)
    L = c.size
    w = _c(weights, np.float64)
    d = _c(deltas, np.float32)
    N, M = d.shape
    assert G.dtype == np.float32 and G.flags.c_contiguous and G.size == M
    assert P.dtype == np.float32 and P.flags.c_contiguous and P.shape == (N, M)
    fi = _c(flags_in, np.uint8)
    oi = _c(order_in if len(order_in) else [0], np.int32)
    p1 = np.empty((N, M), dtype=np.float32)
    agg = np.zeros(M, dtype=np.float32)
    scores = np.empty(L, dtype=np.float64)
    fo = np.empty(L, dtype=np.uint8)
    oo = np.empty(L + 1, dtype=np.int32)
    no = ctypes.c_int64()
    chunk_of = np.empty(L, dtype=np.int32)
    used = lib().oo_step(L, _p(c, _u64p), bpe, N, _p(w, _f64p), _p(d, _f32p), _p(G, _f32p),
                         _p(P, _f32p), _p(fi, _u8p), _p(oi, _i32p), len(order_in), n_chunks,
                         budget, _p(p1, _f32p), _p(agg, _f32p), _p(scores, _f64p), _p(fo, _u8p),
                         _p(oo, _i32p), ctypes.byref(no), _p(chunk_of, _i32p))
    if used < 0:
        raise ValueError("oracle step failed")
    return dict(p_stage1=p1, agg=agg, scores=scores, flags_out=fo, order_out=oo[: no.value].copy(),
                chunk_of=chunk_of, n_chunks_used=int(used))
