"""Pins the C oracle (oracle/osp_oracle.c) before it is trusted as the checker.

1. Hand vectors of the reference unit tests (tests/test_protocol.cpp,
   test_importance.cpp, test_tuning.cpp, test_learner.cpp under
   /root/reference/proj — cited per test).
2. Golden dumps of the unmodified reference engine (tests/golden/*.npz,
   oracle/gen_golden.py): every artefact bit-exact, every iteration.
"""
import numpy as np
import pytest

from oracle import oracle
from osp_testlib import Golden


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


# ---- hand vectors -----------------------------------------------------------

def test_aggregation_hand_vectors():
    # test_protocol.cpp:21-40
    a, b = [1, 3], [3, 5]
    assert list(oracle.aggregate_layer([a, b], [1.0, 1.0])) == [2, 4]
    assert list(oracle.aggregate_layer([a, b], [1.0, 3.0])) == [2.5, 4.5]
    assert list(oracle.aggregate_layer([a], [0.7])) == [1, 3]
    with pytest.raises(ValueError):
        oracle.aggregate_layer([a, [0, 0, 0]], [1.0, 1.0])


def test_pgp_hand_vectors():
    # test_importance.cpp:8-20
    assert oracle.pgp([2], [1.0, -2.0], [0.5, 0.25])[0] == pytest.approx(1.0)
    assert oracle.pgp([2], [1.0, -2.0], [0.0, 0.0])[0] == 0.0
    assert oracle.pgp([2], [-1.0, 2.0], [0.5, 0.25])[0] == pytest.approx(1.0)


def test_rank_tie_break():
    # test_importance.cpp:39-44
    assert list(oracle.rank([5.0, 1.0, 0.2])) == [2, 1, 0]
    assert list(oracle.rank([1.0, 1.0, 1.0])) == [0, 1, 2]
    assert list(oracle.rank([9.0])) == [0]


def test_build_gib_prefix_rule():
    # test_importance.cpp:46-64: sizes 40/60/48 B, rank [2,1,0]
    counts, scores = [10, 15, 12], [5.0, 1.0, 0.2]
    assert list(oracle.build_gib(scores, counts, 4, 100)) == [0, 0, 1]
    assert list(oracle.build_gib(scores, counts, 4, 0)) == [0, 0, 0]
    assert list(oracle.build_gib(scores, counts, 4, 148)) == [1, 1, 1]


def test_build_gib_monotone_random():
    # test_importance.cpp:66-87
    rng = np.random.default_rng(77)
    for _ in range(30):
        L = int(rng.integers(1, 11))
        counts = rng.integers(1, 65, L)
        scores = rng.uniform(0, 10, L)
        total = int(counts.sum()) * 4
        b1 = int(rng.integers(0, total + 1))
        b2 = b1 + int(rng.integers(0, total + 1))
        g1 = oracle.build_gib(scores, counts, 4, b1)
        g2 = oracle.build_gib(scores, counts, 4, b2)
        assert int((counts * 4 * g1).sum()) <= b1
        assert int((counts * 4 * g2).sum()) <= b2
        assert np.all(g2[g1 == 1] == 1)


def test_gib_wire_format():
    # test_importance.cpp:89-121
    assert len(oracle.gib_encode(42, np.ones(1000, np.uint8))) == 133
    e = oracle.gib_encode(0, np.zeros(8, np.uint8))
    assert len(e) == 9 and e[8] == 0
    f = np.zeros(8, np.uint8)
    f[[0, 3]] = 1
    assert oracle.gib_encode(0, f)[8] == 0x09
    full = oracle.gib_encode(0, np.ones(64, np.uint8))
    with pytest.raises(ValueError):
        oracle.gib_decode(full[:-1])
    with pytest.raises(ValueError):
        oracle.gib_decode(bytes([1, 2, 3]))


def test_gib_round_trip_1_to_1000():
    # test_importance.cpp:123-135
    rng = np.random.default_rng(123)
    for L in range(1, 1001):
        f = rng.integers(0, 2, L).astype(np.uint8)
        tag, back = oracle.gib_decode(oracle.gib_encode(L, f))
        assert tag == L and np.array_equal(back, f)


def test_split_cases():
    # test_protocol.cpp:42-79
    rs, chunk_of, used = oracle.split([2, 2], 4, [0, 0], [], 4)
    assert list(rs) == [0, 1] and used == 0
    rs, chunk_of, used = oracle.split([2, 2], 4, [1, 1], [0, 1], 1)
    assert len(rs) == 0 and used == 1 and list(chunk_of) == [0, 0]
    rs, chunk_of, used = oracle.split([4, 4, 4, 4], 4, [0, 0, 1, 1], [3, 2], 2)
    assert list(rs) == [0, 1] and used == 2
    assert chunk_of[3] == 0 and chunk_of[2] == 1
    with pytest.raises(ValueError):
        oracle.split([2], 4, [0], [], 0)


def test_tuning_hand_vectors():
    # test_tuning.cpp:7-72
    assert oracle.compute_umax(1.25e9, 0.0, 0.1, 8, 100_000_000) == 15_625_000
    assert oracle.compute_umax(1.25e9, 0.0, 0.0, 8, 100_000_000) == 0
    assert oracle.compute_umax(1.25e9, 0.0, 1.0, 1, 1_000_000_000) == 800_000_000
    assert oracle.compute_umax(1.25e9, 0.25, 0.1, 8, 1_000_000_000) == 12_500_000
    assert oracle.compute_umax(1.25e9, 0.25, 0.1, 8, 1_000_000_000, True) == 19_531_250
    s = oracle.SguSchedule(1000)
    assert s.tune(1, 1.0) == 0 and s.initial_loss == 1.0
    assert s.tune(5, 1.0) == 0
    assert s.tune(6, 0.0) == 1000
    assert s.tune(7, 0.25) == 750
    assert s.tune(8, 3.0) == 0
    s2 = oracle.SguSchedule(1000)
    with pytest.raises(ValueError, match="ProtocolError"):
        s2.tune(2, 0.5)
    with pytest.raises(ValueError, match="ConfigError"):
        s2.tune(0, 0.5)
    with pytest.raises(ValueError, match="NumericError"):
        s2.tune(1, -0.5)


def test_sgd_delta_and_lr():
    # test_learner.cpp:203-218
    d = oracle.sgd_delta([2.0, -4.0], 0.1)
    assert d[0] == pytest.approx(-0.2) and d[1] == pytest.approx(0.4)
    assert oracle.lr_at_epoch(0.1, 9) == pytest.approx(0.1)
    assert oracle.lr_at_epoch(0.1, 10) == pytest.approx(0.05)
    assert oracle.lr_at_epoch(0.1, 20) == pytest.approx(0.025)
    assert list(oracle.sgd_delta([0.0, 0.0], 0.5)) == [0.0, 0.0]


# ---- reference-engine goldens ------------------------------------------------

def test_synth_generator_matches_reference(golden):
    # runner.cpp:312-321: the dumped deltas are the reference Rng stream
    for it in range(golden.iters):
        d = golden.get(it, "deltas")
        if d is None:
            continue
        for w in range(golden.N):
            assert np.array_equal(bits(oracle.synth_delta(golden.seed, w, it, golden.M)), bits(d[w]))
        # element offsets: a window of the stream equals the slice
        if golden.M > 8:
            win = oracle.synth_delta(golden.seed, 0, it, 5, first=3)
            assert np.array_equal(bits(win), bits(d[0][3:8]))


def test_oracle_step_matches_reference_engine(golden: Golden):
    """Run the restated step iteration by iteration; every artefact must be
    bit-identical to the reference engine's dump."""
    g = golden
    G = g.p0.copy()
    P = np.tile(g.p0, (g.N, 1))
    tag, flags = oracle.gib_decode(bytes(g.get(0, "gib_in")))
    order = g.get(0, "order_in")
    for it in range(g.iters):
        tag_in, flags_in = oracle.gib_decode(bytes(g.get(it, "gib_in")))
        assert np.array_equal(flags_in, flags) and tag_in == (0 if it == 0 else it)
        assert np.array_equal(order, g.get(it, "order_in"))
        budget = int(g.get(it, "budget")[0])
        r = oracle.step(g.counts, g.bpe, g.weights, g.deltas(it), G, P, flags, order,
                        g.n_chunks, budget)
        # split: RS ids and chunk membership
        rs_ref = g.get(it, "rs_ids")
        assert np.array_equal(np.flatnonzero(flags == 0), np.sort(rs_ref))
        chunks_ref = Golden.decode_chunks(g.get(it, "chunks"))
        assert r["n_chunks_used"] == len(chunks_ref)
        for c, ids in enumerate(chunks_ref):
            assert sorted(np.flatnonzero(r["chunk_of"] == c).tolist()) == ids
        # stage-1 worker params
        st1 = g.get(it, "params_stage1")
        if st1 is not None:
            assert np.array_equal(bits(r["p_stage1"]), bits(st1))
        else:
            assert np.array_equal(bits(r["p_stage1"][0]), bits(g.get(it, "params_stage1_w0")))
            assert np.array_equal(bits(r["p_stage1"][-1]), bits(g.get(it, "params_stage1_wlast")))
        # server state after resolution
        assert np.array_equal(bits(G), bits(g.get(it, "global")))
        assert np.array_equal(bits(r["agg"]), bits(g.get(it, "agg")))
        assert np.array_equal(bits(r["scores"]), bits(g.get(it, "scores")))
        if int(g.get(it, "final_eq_global")[0]):
            for w in range(g.N):
                assert np.array_equal(bits(P[w]), bits(G))
        else:
            assert np.array_equal(bits(P), bits(g.get(it, "params_final")))
        # next GIB (tag = i + 1) and the rank-ordered ICS list
        assert oracle.gib_encode(it + 1, r["flags_out"]) == bytes(g.get(it, "gib_out"))
        assert np.array_equal(r["order_out"], g.get(it, "order_out"))
        flags, order = r["flags_out"], r["order_out"]


def test_payload_encoding_hand_vector():
    # test_message.cpp:10-35: PushImportant, iteration 0x01020304, layer 7 = {1.0f}
    counts = [1] * 8
    vals = np.zeros(8, np.float32)
    vals[7] = 1.0
    b = oracle.encode_payload(0, 0x01020304, counts, vals, [7])
    assert len(b) == 7 + 8 + 4
    assert b[0] == 0 and list(b[1:5]) == [4, 3, 2, 1] and list(b[5:7]) == [1, 0]
    assert b[7] == 7 and b[11] == 1
    assert b[15] == 0x00 and b[17] == 0x80 and b[18] == 0x3f
