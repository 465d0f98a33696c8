"""CPU-side checks of the drop-in boundary: the in-tree C-ABI library loads and
exports every function include/osp_c.h declares (no compute without a GPU)."""
import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "osp_c.h")
ENGINE_HEADER = os.path.join(REPO, "include", "osp_engine.h")


def declared_functions(header=HEADER):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(osp_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_functions():
    names = declared_functions()
    assert "osp_group_step" in names and "osp_aggregate_layer" in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol():
    from paper_2306_16926_b200 import _capi
    assert os.path.exists(_capi.LIB_PATH), "run `make lib` first"
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_checked_build_exports_the_same_symbols():
    """The bounds-checked build (make checked; OSP_LIB_VARIANT=checked) is a
    drop-in for the product library."""
    from paper_2306_16926_b200 import _capi
    path = os.path.join(os.path.dirname(_capi.LIB_PATH), "libosp_b200_checked.so")
    if not os.path.exists(path):
        pytest.skip("checked build not built (make checked)")
    lib = ctypes.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2306_16926_b200 import _capi
    assert set(declared_functions()) == set(_capi.EXPORTED)


def test_host_only_entry_points_without_gpu():
    """GIB codec and tuning are host logic; they run without a device."""
    from paper_2306_16926_b200 import _capi
    lib = _capi.load()
    assert lib.osp_abi_version() == 2
    assert lib.osp_gib_encoded_size(1000) == 133
    assert lib.osp_status_name(7) == b"ProtocolError"
    out = ctypes.c_uint64()
    assert lib.osp_compute_umax(1.25e9, 0.0, 0.0, 0.1, 8, 100_000_000, 0, ctypes.byref(out)) == 0
    assert out.value == 15_625_000


def test_gib_wire_with_rank_order_without_gpu():
    """GIB + rank-order side channel (README.md:207-210's gap): bitmap prefix is
    the reference encoding (read by the reference decoder, here its restatement
    in oracle/), the tail carries the emission order; malformed tails fail."""
    import struct

    import numpy as np

    from oracle import oracle
    from paper_2306_16926_b200 import osp
    L = 1000
    flags = np.zeros(L, np.uint8)
    order = np.array([977, 3, 500, 4, 999], np.int32)
    flags[order] = 1
    w = osp.gib_wire_encode(12, flags, order)
    assert len(w) == 133 + 4 + 4 * 5
    assert w[:133] == osp.gib_encode(12, flags) == oracle.gib_encode(12, flags)
    assert w[133:] == struct.pack("<I5I", 5, *order.tolist())
    tag, f2 = oracle.gib_decode(w)  # the reference decoder reads the bitmap prefix
    assert tag == 12 and np.array_equal(f2, flags)
    tag, f3, o3 = osp.gib_wire_decode(w)
    assert tag == 12 and np.array_equal(f3, flags) and np.array_equal(o3, order)
    tag, f4, o4 = osp.gib_wire_decode(w[:133])
    assert o4 is None and np.array_equal(f4, flags)
    e = osp.gib_wire_encode(0, np.zeros(9, np.uint8), [])
    assert osp.gib_wire_decode(e)[2].size == 0
    for bad in (w[:135], w[:-1], w + b"\0", w[:137] + struct.pack("<I", 1000) + w[141:],
                w[:137] + struct.pack("<I", 5) + w[141:], w[:133] + struct.pack("<I", 2000)):
        with pytest.raises(osp.FormatError):
            osp.gib_wire_decode(bad)
    with pytest.raises(osp.LayerError):
        osp.gib_wire_encode(1, flags, [1000])
    with pytest.raises(osp.ProtocolError):
        osp.gib_wire_encode(1, flags, [5])        # not deferred
    with pytest.raises(osp.ProtocolError):
        osp.gib_wire_encode(1, flags, [3, 3])     # repeated


def test_python_front_errors_without_gpu():
    pytest.importorskip("torch")
    from paper_2306_16926_b200 import osp
    assert osp.gib_encode(42, [1] * 1000)[:4] == bytes([42, 0, 0, 0])
    tag, flags = osp.gib_decode(osp.gib_encode(7, [1, 0, 0, 1, 0, 0, 0, 0]))
    assert tag == 7 and list(flags) == [1, 0, 0, 1, 0, 0, 0, 0]
    with pytest.raises(osp.FormatError):
        osp.gib_decode(bytes([1, 2, 3]))
    s = osp.SguSchedule(1000)
    assert s.tune(1, 1.0) == 0
    assert s.tune(7, 0.25) == 750
    with pytest.raises(osp.ProtocolError):
        osp.SguSchedule(10).tune(2, 0.5)
    with pytest.raises(osp.ConfigError):
        osp.SguSchedule(10).tune(0, 0.5)
    with pytest.raises(osp.NumericError):
        osp.SguSchedule(10).tune(1, -0.5)
    assert osp.compute_umax(1.25e9, 0.1, 8, 1_000_000_000, loss_rate=0.25) == 12_500_000
    assert osp.compute_umax(1.25e9, 0.1, 8, 1_000_000_000, loss_rate=0.25,
                            eq5_literal=True) == 19_531_250
    with pytest.raises(osp.ConfigError):
        osp.compute_umax(-1.0, 0.1, 8, 100)


def test_engine_library_exports_every_declared_symbol():
    """include/osp_engine.h (message-level worker/server C-ABI) is exported by
    the façade library and fully bound by paper_2306_16926_b200/engine.py."""
    from paper_2306_16926_b200 import engine
    names = declared_functions(ENGINE_HEADER)
    assert "osp_worker_compute_done" in names and "osp_server_on_push_important" in names
    lib = engine.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(engine.EXPORTED)


def test_engine_messages_without_gpu():
    """Partition and message codec are host logic: payload wire round trip
    (message.cpp:53-99 layout) and its error class."""
    import struct
    from paper_2306_16926_b200 import engine, osp
    part = engine.Partition([3, 2])
    assert part.total == 5
    raw = (struct.pack("<BIH", 0, 7, 2) + struct.pack("<II", 0, 3) + struct.pack("<3f", 1, 2, 3)
           + struct.pack("<II", 1, 2) + struct.pack("<2f", -1, 0.5))
    m = engine.Message.decode(raw, from_worker=2)
    assert (m.kind, m.iteration, m.from_worker, m.layer_count) == ("PushImportant", 7, 2, 2)
    assert m.size_bytes(part) == 20
    assert m.encode() == raw
    with pytest.raises(osp.FormatError):
        engine.Message.decode(raw[:-3])
