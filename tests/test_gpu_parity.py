"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference-engine goldens. Bit-exact for everything: masks, index lists, chunk
maps, GIB bytes, aggregated/updated fp32 vectors. The only non-bit-exact
quantity is the group's per-layer PGP score (a parallel tree sum, documented
tolerance 1e-12 relative; the ranking built from it is certified exact)."""
import struct

import numpy as np
import pytest
import torch

from oracle import oracle
from osp_testlib import Golden

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-12  # tree vs sequential fp64 sum of non-negative terms


def bits(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.fixture(scope="module")
def osp():
    from paper_2306_16926_b200 import osp as m
    m.lib()
    return m


def cuda(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


# ---- per-function primitives -------------------------------------------------

def test_aggregate_hand_vectors(osp):
    # test_protocol.cpp:21-40
    a, b = cuda(np.float32([1, 3])), cuda(np.float32([3, 5]))
    assert osp.aggregate_layer([a, b], [1.0, 1.0]).tolist() == [2, 4]
    assert osp.aggregate_layer([a, b], [1.0, 3.0]).tolist() == [2.5, 4.5]
    assert osp.aggregate_layer([a], [0.7]).tolist() == [1, 3]
    with pytest.raises(osp.ProtocolError):
        osp.aggregate_layer([a, cuda(np.float32([0, 0, 0]))], [1.0, 1.0])
    with pytest.raises(osp.ProtocolError):
        osp.aggregate_layer([a, b], [0.0, 0.0])


def test_aggregate_random_bit_exact(osp):
    # checks.cpp:220-264 (aggregation oracle): random weights and sizes
    rng = np.random.default_rng(4242)
    for _ in range(20):
        n = int(rng.integers(1, 9))
        size = int(rng.integers(1, 5000))
        w = list(0.1 + rng.random(n))
        xs = [rng.uniform(-2, 2, size).astype(np.float32) for _ in range(n)]
        got = osp.aggregate_layer([cuda(x) for x in xs], w)
        want = oracle.aggregate_layer(xs, w)
        assert np.array_equal(bits(got), bits(want))


def test_synth_delta_matches_reference_stream(osp, golden):
    d = golden.get(0, "deltas")
    if d is None:
        pytest.skip("fixture without stored deltas")
    got = osp.synth_deltas(golden.seed, golden.N, 0, golden.M)
    assert np.array_equal(bits(got), bits(d))
    win = osp.synth_delta(golden.seed, golden.N - 1, 0, 7, first=2) if golden.M > 9 else None
    if win is not None:
        assert np.array_equal(bits(win), bits(d[-1][2:9]))


def test_synth_large_vs_oracle(osp):
    n = 3_000_001
    got = osp.synth_deltas(11, 3, 5, n)
    for w in range(3):
        assert np.array_equal(bits(got[w]), bits(oracle.synth_delta(11, w, 5, n)))


def test_apply_and_sgd(osp):
    # test_param.cpp:94-107, test_learner.cpp:203-218
    p = cuda(np.float32([1, 1]))
    d = cuda(np.float32([0.5, -0.5]))
    osp.apply_delta(p, d, 1.0)
    assert p.tolist() == [1.5, 0.5]
    osp.apply_delta(p, d, 0.0)
    assert p.tolist() == [1.5, 0.5]
    with pytest.raises(osp.ShapeError):
        osp.apply_delta(p, cuda(np.float32([1, 2, 3])), 1.0)
    g = np.random.default_rng(1).normal(size=100_003).astype(np.float32)
    assert np.array_equal(bits(osp.sgd_delta(cuda(g), 0.05)), bits(oracle.sgd_delta(g, 0.05)))
    with pytest.raises(osp.ConfigError):
        osp.sgd_delta(cuda(g), 0.0)


def test_lgp_hand_vectors(osp):
    # test_protocol.cpp:81-142
    part = osp.Partition([2, 2])
    p = cuda(np.float32([1, 1, 1, 1]))
    gd = cuda(np.float32([0.1, -0.2, 0, 0]))
    ld = cuda(np.float32([0, 0, 0.05, 0.05]))
    base = torch.zeros(4, device="cuda")
    osp.lgp_partial(part, p, gd, ld, [0, 1], base)
    v = p.tolist()
    assert v[0] == pytest.approx(1.1) and v[1] == pytest.approx(0.8)
    assert v[2] == pytest.approx(1.05) and v[3] == pytest.approx(1.05)
    osp.lgp_correct(part, p, base, cuda(np.float32([0, 0, 0.02, -0.01])), [1])
    v = p.tolist()
    assert v[2] == pytest.approx(1.02) and v[3] == pytest.approx(0.99)
    # correcting with the local delta is an exact no-op (test_protocol.cpp:126-135)
    part1 = osp.Partition([2])
    q = cuda(np.float32([1, 1]))
    loc = cuda(np.float32([0.3, -0.7]))
    b1 = torch.zeros(2, device="cuda")
    osp.lgp_partial(part1, q, torch.zeros(2, device="cuda"), loc, [1], b1)
    before = q.clone()
    osp.lgp_correct(part1, q, b1, loc, [0])
    assert np.array_equal(bits(q), bits(before))
    with pytest.raises(osp.LayerError):
        osp.lgp_correct(part1, q, b1, loc, [5])


def test_pgp_exact_vs_oracle(osp):
    rng = np.random.default_rng(3)
    counts = [1, 7, 300, 4096, 33, 100_000]
    M = sum(counts)
    p = rng.uniform(-1, 1, M).astype(np.float32)
    g = rng.uniform(-1e-3, 1e-3, M).astype(np.float32)
    part = osp.Partition(counts)
    got = osp.pgp_layer_importance(part, cuda(p), cuda(g))
    assert np.array_equal(bits(got), bits(oracle.pgp(counts, p, g)))
    # test_importance.cpp:8-20
    part2 = osp.Partition([2])
    s = osp.pgp_layer_importance(part2, cuda(np.float32([1, -2])), cuda(np.float32([0.5, 0.25])))
    assert s[0] == pytest.approx(1.0)


def test_rank_gib_vs_oracle(osp):
    # test_importance.cpp:39-87
    part = osp.Partition([10, 15, 12])
    order, flags = osp.rank_and_gib(part, [5.0, 1.0, 0.2], 100)
    assert list(order) == [2, 1, 0] and list(flags) == [0, 0, 1]
    _, flags = osp.rank_and_gib(part, [5.0, 1.0, 0.2], 0)
    assert list(flags) == [0, 0, 0]
    _, flags = osp.rank_and_gib(part, [5.0, 1.0, 0.2], part.total_bytes())
    assert list(flags) == [1, 1, 1]
    order, _ = osp.rank_and_gib(osp.Partition([1, 1, 1]), [1.0, 1.0, 1.0], 0)
    assert list(order) == [0, 1, 2]
    rng = np.random.default_rng(77)
    for _ in range(30):
        L = int(rng.integers(1, 600))
        counts = rng.integers(1, 65, L)
        scores = rng.uniform(0, 10, L)
        scores[rng.integers(0, L, L // 4)] = 1.5  # ties
        budget = int(rng.integers(0, int(counts.sum()) * 4 + 1))
        part = osp.Partition(counts)
        order, flags = osp.rank_and_gib(part, scores, budget)
        assert np.array_equal(order, oracle.rank(scores))
        assert np.array_equal(flags, oracle.build_gib(scores, counts, 4, budget))


def test_split_vs_oracle(osp):
    # test_protocol.cpp:42-79 and random
    part = osp.Partition([4, 4, 4, 4])
    rs, chunk_of, used = osp.split_for_sync(part, [0, 0, 1, 1], [3, 2], 2)
    assert list(rs) == [0, 1] and used == 2 and chunk_of[3] == 0 and chunk_of[2] == 1
    rs, chunk_of, used = osp.split_for_sync(osp.Partition([2, 2]), [0, 0], [], 4)
    assert list(rs) == [0, 1] and used == 0
    with pytest.raises(osp.ConfigError):
        osp.split_for_sync(part, [0, 0, 0, 0], [], 0)
    with pytest.raises(osp.ShapeError):
        osp.split_for_sync(part, [0, 0], [], 1)
    rng = np.random.default_rng(9)
    for _ in range(40):
        L = int(rng.integers(1, 300))
        counts = rng.integers(1, 5000, L)
        flags = (rng.random(L) < 0.5).astype(np.uint8)
        perm = rng.permutation(L).astype(np.int32)
        order = perm[: int(rng.integers(0, L + 1))]  # partial rank list: missing ids appended
        nc = int(rng.integers(1, 9))
        bpe = int(rng.choice([1, 4, 1000]))
        p = osp.Partition(counts, bpe)
        rs, co, used = osp.split_for_sync(p, flags, order, nc)
        rs_o, co_o, used_o = oracle.split(counts, bpe, flags, order, nc)
        assert np.array_equal(rs, rs_o) and np.array_equal(co, co_o) and used == used_o


# ---- the group step against the reference-engine goldens ----------------------

def run_group_against_golden(osp, g: Golden, tile_elems=0, pad_ld=0, tma=None, carry=True,
                             stage2_zeros=False):
    part = osp.Partition(g.counts, g.bpe)
    grp = osp.OspGroup(part, g.N, list(g.weights), n_chunks=g.n_chunks,
                       init_params=cuda(g.p0), tile_elems=tile_elems, tma=tma, carry=carry)
    for it in range(g.iters):
        d = g.deltas(it)
        X = torch.zeros((g.N, g.M + pad_ld), dtype=torch.float32, device="cuda")
        X[:, : g.M] = cuda(d)
        # the GIB this iteration splits with (tag it) must be what the group holds
        st = grp.read_gib()
        tag_in, flags_in = oracle.gib_decode(bytes(g.get(it, "gib_in")))
        assert st["tag"] == tag_in
        assert np.array_equal(st["flags"], flags_in)
        assert np.array_equal(st["order"], g.get(it, "order_in"))
        chunks_ref = Golden.decode_chunks(g.get(it, "chunks"))
        assert st["n_used"] == len(chunks_ref)
        for c, ids in enumerate(chunks_ref):
            assert sorted(np.flatnonzero(st["chunk_of"] == c).tolist()) == ids
        grp.set_budget(int(g.get(it, "budget")[0]))
        grp.stage1(X)
        st1 = g.get(it, "params_stage1")
        P1 = grp.worker_params.cpu().numpy()
        if st1 is not None:
            assert np.array_equal(bits(P1), bits(st1)), f"stage-1 worker params, it {it}"
        else:
            assert np.array_equal(bits(P1[0]), bits(g.get(it, "params_stage1_w0")))
            assert np.array_equal(bits(P1[-1]), bits(g.get(it, "params_stage1_wlast")))
        # with the ICS carry, stage 2 applies the payload split at stage 1 (as the
        # reference's split_for_sync copies it) and never reads its deltas argument
        X2 = torch.zeros_like(X) if stage2_zeros else X
        for c in range(g.n_chunks):
            grp.stage2_chunk(c, X2)
        grp.resolve(X)
        G = grp.global_params.cpu().numpy()
        assert np.array_equal(bits(G), bits(g.get(it, "global"))), f"global, it {it}"
        assert int(g.get(it, "final_eq_global")[0]) == 1
        P = grp.worker_params.cpu().numpy()
        for w in range(g.N):
            assert np.array_equal(bits(P[w]), bits(G)), f"worker {w} after corrections"
        np.testing.assert_allclose(grp.scores.cpu().numpy(), g.get(it, "scores"), rtol=SCORE_RTOL,
                                   atol=0)
        nxt = grp.read_gib()
        tag_out, flags_out = oracle.gib_decode(bytes(g.get(it, "gib_out")))
        assert nxt["tag"] == tag_out == it + 1
        assert np.array_equal(nxt["flags"], flags_out), f"GIB flags, it {it}"
        assert np.array_equal(nxt["order"], g.get(it, "order_out")), f"ICS order, it {it}"
        # the device-written wire: the reference's GIB bytes + the rank order
        order_out = np.asarray(g.get(it, "order_out"), dtype="<u4")
        assert grp.gib_wire() == (bytes(g.get(it, "gib_out")) + struct.pack("<I", order_out.size)
                                  + order_out.tobytes()), f"GIB wire, it {it}"
    return grp


@pytest.mark.parametrize("tma", [None, False])
def test_group_matches_reference_engine(osp, golden, tma):
    run_group_against_golden(osp, golden, tma=tma)


def test_group_small_tiles_and_unaligned_rows(osp, golden):
    # multi-tile layers, and rows whose stride breaks 16-byte alignment (scalar path)
    run_group_against_golden(osp, golden, tile_elems=1024, pad_ld=1, tma=False)


# ---- the group step against the oracle at larger sizes ---------------------------

def oracle_vs_group(osp, counts, N, weights, budget_frac, n_chunks, iters, seed, p0=None,
                    sgd_lr=0.0, tile_elems=0, tma=None, carry=True):
    counts = np.asarray(counts, dtype=np.uint64)
    M = int(counts.sum())
    bpe = 4
    budget = int(budget_frac * M * bpe)
    G = np.zeros(M, np.float32) if p0 is None else p0.copy()
    P = np.tile(G, (N, 1))
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, weights, n_chunks=n_chunks, init_params=cuda(G),
                       sgd_lr=sgd_lr, tile_elems=tile_elems, tma=tma, carry=carry)
    flags = np.zeros(len(counts), np.uint8)
    order = np.zeros(0, np.int32)
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    for it in range(iters):
        osp.synth_deltas(seed, N, it, M, out=X)
        if sgd_lr > 0:
            X.mul_(37.0)  # treat as raw gradients
            deltas = np.stack([oracle.sgd_delta(X[w].cpu().numpy(), sgd_lr) for w in range(N)])
        else:
            deltas = X.cpu().numpy()
        r = oracle.step(counts, bpe, weights, deltas, G, P, flags, order, n_chunks, budget)
        grp.set_budget(budget)
        grp.step(X)
        assert np.array_equal(bits(grp.global_params), bits(G)), f"global, it {it}"
        Pg = grp.worker_params.cpu().numpy()
        for w in range(N):
            assert np.array_equal(bits(Pg[w]), bits(P[w])), f"worker {w}, it {it}"
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"]), f"flags, it {it}"
        assert np.array_equal(nxt["order"], r["order_out"]), f"order, it {it}"
        np.testing.assert_allclose(grp.scores.cpu().numpy(), r["scores"], rtol=SCORE_RTOL, atol=0)
        flags, order = r["flags_out"], r["order_out"]
    return grp


def test_group_resnet50_layout_vs_oracle(osp):
    from paper_2306_16926_b200 import layouts
    grp = oracle_vs_group(osp, layouts.resnet50(), 8, [0.125] * 8, 0.5, 4, 3, seed=11, tma=False)
    assert grp.stats()["resolved"] == 3
    assert grp.stage_kernels == "register-staged"


def test_group_odd_workers_unequal_weights(osp):
    rng = np.random.default_rng(5)
    counts = rng.integers(1, 20000, 57)
    w = list(0.1 + rng.random(5))
    p0 = rng.uniform(-1, 1, int(counts.sum())).astype(np.float32)
    grp = oracle_vs_group(osp, counts, 5, w, 0.6, 3, 4, seed=3, p0=p0, tile_elems=2048, tma=False)
    assert grp.stage_kernels == "register-staged"
    grp = oracle_vs_group(osp, counts, 5, w, 0.6, 3, 4, seed=3, p0=p0, tile_elems=2048)
    assert grp.stage_kernels == "tma-staged"  # N=5: default TMA shape


def test_group_fused_sgd(osp):
    rng = np.random.default_rng(8)
    counts = rng.integers(1, 9000, 40)
    oracle_vs_group(osp, counts, 4, [0.25] * 4, 0.5, 4, 3, seed=19, sgd_lr=0.05, tma=False)


@pytest.mark.parametrize("L", [1, 2, 33, 2500, 3072, 3073, 20000])
def test_group_many_layers(osp, L):
    """Layer counts from 1 up: bitonic rank padding, stage kernels with global
    layer tables (L > 2048), the resolve's per-layer arrays in shared memory up to
    3072 layers and in a global scratch buffer above (3073, 20000)."""
    rng = np.random.default_rng(L)
    counts = rng.integers(1, 400, L)
    oracle_vs_group(osp, counts, 4, [0.25] * 4, 0.5, 3, 2, seed=L)


def test_many_layers_free_functions(osp):
    """rank_and_gib and split_for_sync above the shared-memory layer count."""
    rng = np.random.default_rng(9)
    L = 7000
    counts = rng.integers(1, 50, L).astype(np.uint64)
    scores = rng.random(L)
    scores[100:110] = scores[5]  # ties
    part = osp.Partition(counts)
    budget = int(counts.sum()) * 2
    order, flags = osp.rank_and_gib(part, scores, budget)
    assert np.array_equal(order, oracle.rank(scores))
    assert np.array_equal(flags, oracle.build_gib(scores, counts, 4, budget))
    ics_order = order[: int(flags.sum())]
    rs, chunk_of, used = osp.split_for_sync(part, flags, ics_order, 5)
    rs_o, chunk_o, used_o = oracle.split(counts, 4, flags, ics_order, 5)
    assert np.array_equal(rs, rs_o) and np.array_equal(chunk_of, chunk_o) and used == used_o


def test_group_too_many_layers(osp):
    with pytest.raises(osp.InvalidArgument):
        osp.OspGroup(osp.Partition([1] * 65537), 2)


def test_group_budget_edges(osp):
    counts = [4096, 12, 70000, 1, 333, 8192, 5]
    for frac in (0.0, 1.0, 0.33):
        oracle_vs_group(osp, counts, 2, [0.5, 0.5], frac, 4, 3, seed=23, tma=False)
    oracle_vs_group(osp, counts, 1, [1.0], 0.7, 1, 3, seed=29, tma=False)
    oracle_vs_group(osp, counts, 3, [0.2, 0.3, 0.5], 0.9, 9, 3, seed=31)


def test_certificate_fallback_on_exact_ties(osp):
    """Two layers with identical contents tie exactly in the reference (stable
    order by id); the tree sums cannot certify the order, so the exact
    sequential fallback must run and reproduce the reference ranking."""
    half = 50_000
    counts = [half, half, 1000, half]
    M = sum(counts)
    N = 4
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    osp.synth_deltas(7, N, 0, M, out=X)
    X[:, half: 2 * half] = X[:, :half]           # layer 1 == layer 0
    X[:, 2 * half + 1000:] = X[:, :half]         # layer 3 == layer 0
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=2)
    G = np.zeros(M, np.float32)
    P = np.zeros((N, M), np.float32)
    budget = int(0.6 * M * 4)
    r = oracle.step(counts, 4, [0.25] * N, X.cpu().numpy(), G, P, np.zeros(4, np.uint8),
                    np.zeros(0, np.int32), 2, budget)
    assert r["scores"][0] == r["scores"][1] == r["scores"][3]
    grp.set_budget(budget)
    grp.step(X)
    nxt = grp.read_gib()
    assert np.array_equal(nxt["flags"], r["flags_out"])
    assert np.array_equal(nxt["order"], r["order_out"])
    st = grp.stats()
    assert st["fallback_resolves"] == 1 and st["fallback_layers"] >= 3


@pytest.mark.parametrize("carry", [True, False])
def test_certificate_fallback_on_deferred_layers(osp, carry):
    """Exact ties again in iteration 1, where a tied layer is deferred: the exact
    fallback must score it against its post-update values. With the ICS carry
    the step overlaps the resolve with the stage-2 broadcast, so those values
    come from the carry buffer, not from G (still being written)."""
    half = 50_000
    counts = [half, half, 1000, half]
    M = sum(counts)
    N = 4
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=2, carry=carry)
    G = np.zeros(M, np.float32)
    P = np.zeros((N, M), np.float32)
    flags, order = np.zeros(4, np.uint8), np.zeros(0, np.int32)
    budget = int(0.6 * M * 4)
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    deferred_tie = False
    for it in range(3):
        osp.synth_deltas(7, N, it, M, out=X)
        X[:, half: 2 * half] = X[:, :half]
        X[:, 2 * half + 1000:] = X[:, :half]
        deferred_tie |= bool(flags[0] or flags[1] or flags[3])
        r = oracle.step(counts, 4, [0.25] * N, X.cpu().numpy(), G, P, flags, order, 2, budget)
        grp.set_budget(budget)
        grp.step(X)
        assert np.array_equal(bits(grp.global_params), bits(G)), f"global, it {it}"
        assert np.array_equal(bits(grp.worker_params), bits(P)), f"workers, it {it}"
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"]), f"flags, it {it}"
        assert np.array_equal(nxt["order"], r["order_out"]), f"order, it {it}"
        flags, order = r["flags_out"], r["order_out"]
    assert deferred_tie
    st = grp.stats()
    assert st["fallback_resolves"] == 3


@pytest.mark.parametrize("carry", [True, False])
def test_group_step_captured_in_cuda_graph(osp, carry):
    """The step has no host sync and fixed arguments, so it can be captured in
    a CUDA graph (programmatic-dependent launches become graph edges, incl. the
    carry's resolve-beside-stage-2 join); replays equal direct steps bit for bit."""
    from paper_2306_16926_b200 import layouts
    counts = layouts.resnet50()[:60]
    M, N = sum(counts), 8
    part = osp.Partition(counts)
    X = [osp.synth_deltas(11, N, i, M) for i in range(2)]
    a = osp.OspGroup(part, N, n_chunks=4, carry=carry)
    b = osp.OspGroup(part, N, n_chunks=4, carry=carry)
    for grp in (a, b):
        grp.set_budget(M * 2)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cs, capture_error_mode="thread_local"):
        b.step(X[0])
        b.step(X[1])
    torch.cuda.synchronize()
    assert b.read_gib()["tag"] == 0  # capture launches nothing
    for r in range(3):
        a.step(X[0])
        a.step(X[1])
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(bits(a.global_params), bits(b.global_params)), f"replay {r}"
        assert np.array_equal(bits(a.worker_params), bits(b.worker_params)), f"replay {r}"
        ra, rb = a.read_gib(), b.read_gib()
        assert ra["tag"] == rb["tag"] == 2 * (r + 1)
        assert np.array_equal(ra["order"], rb["order"]) and np.array_equal(ra["flags"], rb["flags"])


@pytest.mark.parametrize("carry", [True, False])
def test_momentum_matches_oracle_on_momentum_deltas(osp, carry):
    """Momentum (extension): v <- fl(fl(mu*v) + g), delta = sgd_delta(v), fused
    into stage 1. Pinned to the oracle step fed with deltas from the same rule
    restated in numpy (fp32 multiply then add, as in the kernel); mu = 0 is the
    plain sgd_delta path bit for bit."""
    rng = np.random.default_rng(17)
    counts = [int(c) for c in rng.integers(1, 7000, 23)] + [4096, 8192, 12]
    M, N, lr, mu = sum(counts), 4, 0.05, 0.9
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=3, sgd_lr=lr, carry=carry)
    plain = osp.OspGroup(part, N, [0.25] * N, n_chunks=3, sgd_lr=lr, carry=carry)
    grp.set_momentum(mu)
    plain.set_momentum(0.0)
    G = np.zeros(M, np.float32)
    Pw = np.zeros((N, M), np.float32)
    V = np.zeros((N, M), np.float32)
    flags, order = np.zeros(len(counts), np.uint8), np.zeros(0, np.int32)
    budget = int(0.5 * M * 4)
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    for it in range(4):
        osp.synth_deltas(41, N, it, M, out=X)
        X.mul_(29.0)  # gradients
        g = X.cpu().numpy()
        V = (np.float32(mu) * V).astype(np.float32) + g          # fp32 mul, then fp32 add
        deltas = np.stack([oracle.sgd_delta(V[w], lr) for w in range(N)])
        r = oracle.step(counts, 4, [0.25] * N, deltas, G, Pw, flags, order, 3, budget)
        for grp_ in (grp, plain):
            grp_.set_budget(budget)
            grp_.step(X)
        assert np.array_equal(bits(grp.global_params), bits(G)), f"global, it {it}"
        assert np.array_equal(bits(grp.worker_params), bits(Pw)), f"workers, it {it}"
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"]) and np.array_equal(nxt["order"], r["order_out"])
        flags, order = r["flags_out"], r["order_out"]
    # mu = 0: the group that never had momentum and one that turned it off agree
    ref0 = osp.OspGroup(part, N, [0.25] * N, n_chunks=3, sgd_lr=lr, carry=carry)
    for it in range(4):
        osp.synth_deltas(41, N, it, M, out=X)
        X.mul_(29.0)
        ref0.set_budget(budget)
        ref0.step(X)
    assert np.array_equal(bits(ref0.global_params), bits(plain.global_params))
    assert np.array_equal(bits(ref0.worker_params), bits(plain.worker_params))
    with pytest.raises(osp.ConfigError):
        osp.OspGroup(part, N, [0.25] * N).set_momentum(0.9)       # deltas, not gradients
    with pytest.raises(osp.ConfigError):
        grp.set_momentum(1.5)
    with pytest.raises(osp.InvalidArgument):
        osp.OspGroup(part, N, [0.25] * N, sgd_lr=lr, tma=False).set_momentum(0.9)
    with pytest.raises(osp.InvalidArgument):  # 17 rows x 8 KB x 2 slots: no room for the ring
        osp.OspGroup(part, 8, [0.125] * 8, sgd_lr=lr, tile_elems=2048).set_momentum(0.9)


def test_repeated_stage2_resolve_is_refused(osp):
    """Misuse guard for the carry's device-side join: a second stage2_resolve
    without a stage 1 in between is a ProtocolError raised on the host (no
    launch, no hang, state untouched); the group then continues normally."""
    counts = [4096, 1000, 8192, 12, 2048]
    M, N = sum(counts), 4
    grp = osp.OspGroup(osp.Partition(counts), N, [0.25] * N, n_chunks=2, small=False)
    grp.set_budget(M * 2)
    X = osp.synth_deltas(3, N, 0, M)
    grp.step(X)
    grp.step(osp.synth_deltas(3, N, 1, M))
    torch.cuda.synchronize()
    G = grp.global_params.clone()
    P = grp.worker_params.clone()
    tag = grp.read_gib()["tag"]
    with pytest.raises(osp.ProtocolError):
        grp.stage2_resolve(X)
    torch.cuda.synchronize()
    assert torch.equal(G, grp.global_params) and torch.equal(P, grp.worker_params)
    assert grp.read_gib()["tag"] == tag
    grp.step(osp.synth_deltas(3, N, 2, M))
    assert grp.read_gib()["tag"] == tag + 1


def test_group_device_memory_released_without_gc(osp):
    """Dropping a group (and its zero-copy views) frees its device memory at
    once: the views keep a handle holder alive, not the group, so there is no
    reference cycle for the garbage collector to find."""
    import gc
    gc.disable()
    try:
        part = osp.Partition([1 << 22] * 16)  # 67 M params: ~2.5 GB per group
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        for _ in range(4):
            g = osp.OspGroup(part, 8)
            v = g.worker_params
            g.step(osp.synth_deltas(1, 8, 0, part.total_count()))
            torch.cuda.synchronize()
            del g, v
        torch.cuda.empty_cache()
        free1 = torch.cuda.mem_get_info()[0]
        assert free0 - free1 < (256 << 20), (free0, free1)
        g = osp.OspGroup(part, 8)
        v = g.global_params
        del g                     # the view alone keeps the group's memory valid
        assert float(v.sum()) == 0.0
        del v
    finally:
        gc.enable()


def test_gib_wire_installs_like_set_gib(osp):
    """A wire read from one group and installed into another reproduces the
    GIB, rank order and chunk map; a bitmap-only wire installs ascending ids."""
    from paper_2306_16926_b200 import layouts
    counts = layouts.resnet50()[:40]
    M, N = sum(counts), 4
    part = osp.Partition(counts)
    a = osp.OspGroup(part, N, [0.25] * N, n_chunks=3)
    b = osp.OspGroup(part, N, [0.25] * N, n_chunks=3)
    for it in range(3):
        a.set_budget(M * 2)
        a.step(osp.synth_deltas(3, N, it, M))
    w = a.gib_wire()
    ra = a.read_gib()
    assert w == osp.gib_wire_encode(ra["tag"], ra["flags"], ra["order"])
    b.set_gib_wire(w)
    rb = b.read_gib()
    for k in ("tag", "flags", "order", "chunk_of", "n_used"):
        assert np.array_equal(np.asarray(ra[k]), np.asarray(rb[k])), k
    assert b.gib_wire() == w
    b.set_gib_wire(w[: osp.lib().osp_gib_encoded_size(len(counts))])
    rb = b.read_gib()
    assert np.array_equal(rb["order"], np.flatnonzero(ra["flags"]))
    with pytest.raises(osp.ShapeError):
        osp.OspGroup(osp.Partition(counts[:5]), N).set_gib_wire(w)


def test_step_host_async_pipelined(osp):
    """osp_group_step_host_async: five pipelined calls (each call's H2D beside
    the previous step and D2H), then the wait: every call's updated global
    vector and GIB bytes equal the device step's, iteration by iteration."""
    from paper_2306_16926_b200 import layouts
    counts = layouts.resnet50()[:30]
    M, N, K = sum(counts), 8, 5
    part = osp.Partition(counts)
    a = osp.OspGroup(part, N, [0.125] * N, n_chunks=4)
    b = osp.OspGroup(part, N, [0.125] * N, n_chunks=4)
    a.set_budget(M * 2)
    b.set_budget(M * 2)
    hosts = [osp.synth_deltas(11, N, it, M).cpu().pin_memory() for it in range(K)]
    outs = [torch.empty(M, dtype=torch.float32).pin_memory() for _ in range(K)]
    gibs = [torch.empty(int(osp.lib().osp_gib_encoded_size(len(counts))), dtype=torch.uint8).pin_memory()
            for _ in range(K)]
    for it in range(K):
        b.step_host_async(hosts[it], params_out=outs[it], gib_out=gibs[it])
    b.host_wait()
    for it in range(K):
        a.step(hosts[it].cuda())
        assert np.array_equal(outs[it].numpy().view(np.uint32),
                              a.global_params.cpu().numpy().view(np.uint32)), f"params, it {it}"
        ra = a.read_gib()
        assert bytes(gibs[it].numpy()) == oracle.gib_encode(ra["tag"], ra["flags"]), f"gib, it {it}"
    assert np.array_equal(bits(a.worker_params), bits(b.worker_params))


def test_step_host_matches_device_step(osp):
    from paper_2306_16926_b200 import layouts
    counts = layouts.resnet50()[:40]
    M = sum(counts)
    N = 8
    part = osp.Partition(counts)
    a = osp.OspGroup(part, N, [0.125] * N, n_chunks=4)
    b = osp.OspGroup(part, N, [0.125] * N, n_chunks=4)
    for it in range(3):
        X = osp.synth_deltas(11, N, it, M)
        host = X.cpu().numpy()
        a.set_budget(M * 2)
        b.set_budget(M * 2)
        a.step(X)
        params = np.empty(M, np.float32)
        gib = b.step_host(host, params_out=params)
        assert np.array_equal(bits(a.global_params), bits(b.global_params))
        assert np.array_equal(params.view(np.uint32), a.global_params.cpu().numpy().view(np.uint32))
        ra = a.read_gib()
        assert gib == oracle.gib_encode(ra["tag"], ra["flags"])
    # shape errors are raised before any copy (no host out-of-bounds read)
    with pytest.raises(osp.ShapeError):
        b.step_host(np.zeros((N - 1, M), np.float32))
    with pytest.raises(osp.ShapeError):
        b.step_host(np.zeros((N, M - 1), np.float32))
    with pytest.raises(osp.ShapeError):
        b.step_host(np.zeros((N, M), np.float32), params_out=np.zeros(M - 1, np.float32))
    with pytest.raises(osp.ShapeError):
        b.set_gib(np.zeros(len(counts) - 1, np.uint8), [], 0)
    with pytest.raises(osp.ShapeError):
        b.stage1(torch.zeros((N, 2 * M), device="cuda")[:, : M - 4])


def test_stage2_needs_stage1_and_gib_install_waits(osp):
    """stage 2 before stage 1 of an iteration and a GIB install between stage 1
    and the resolve are protocol errors (the carry and its list snapshot are
    written by stage 1)."""
    counts = [4096, 64, 2048, 1000]
    M, N = sum(counts), 4
    part = osp.Partition(counts)
    g = osp.OspGroup(part, N, [0.25] * N, n_chunks=2)
    X = osp.synth_deltas(3, N, 0, M)
    with pytest.raises(osp.ProtocolError):
        g.stage2_all(X)
    with pytest.raises(osp.ProtocolError):
        g.stage2_resolve(X)
    g.stage1(X)
    with pytest.raises(osp.ProtocolError):
        g.set_gib([0, 1, 0, 0], [1], 5)
    g.stage2_resolve(X)
    g.set_gib([0, 1, 0, 0], [1], 5)
    g.step(X)
    torch.cuda.synchronize()


# ---- TMA-staged stage kernels (OSP_GROUP_TMA): same results --------------------

@pytest.mark.parametrize("carry", [True, False])
@pytest.mark.parametrize("pad_ld", [0, 1])
def test_tma_group_matches_reference_engine(osp, golden, pad_ld, carry):
    if golden.N > 8:
        with pytest.raises(osp.InvalidArgument):
            osp.OspGroup(osp.Partition(golden.counts, golden.bpe), golden.N,
                         list(golden.weights), tma=True)
        return
    # pad_ld=1: unaligned rows, every tile takes the unstaged path
    run_group_against_golden(osp, golden, pad_ld=pad_ld, tma=True, carry=carry,
                             stage2_zeros=carry)


@pytest.mark.parametrize("carry", [True, False])
@pytest.mark.parametrize("tile", [512, 1024, 2048])
def test_tma_group_resnet50_layout_vs_oracle(osp, tile, carry):
    from paper_2306_16926_b200 import layouts
    grp = oracle_vs_group(osp, layouts.resnet50(), 8, [0.125] * 8, 0.5, 4, 3, seed=11,
                          tile_elems=tile, tma=True, carry=carry)
    assert grp.stage_kernels == "tma-staged"


def test_default_group_is_tma_staged(osp):
    part = osp.Partition([1000, 5000])
    assert osp.OspGroup(part, 8).geometry()["tile_elems"] == 1024
    assert osp.OspGroup(part, 8).stage_kernels == "tma-staged"
    assert osp.OspGroup(part, 3).stage_kernels == "tma-staged"   # default shape for N = 3..7
    assert osp.OspGroup(part, 9).stage_kernels == "register-staged"
    assert osp.OspGroup(part, 9).geometry()["tile_elems"] == 512
    with pytest.raises(osp.InvalidArgument):
        osp.OspGroup(part, 8, tile_elems=256, tma=True)


def test_tma_group_ragged_sgd_and_budget_edges(osp):
    rng = np.random.default_rng(8)
    counts = rng.integers(1, 9000, 40)
    oracle_vs_group(osp, counts, 4, [0.25] * 4, 0.5, 4, 3, seed=19, sgd_lr=0.05, tma=True)
    counts = [4096, 12, 70000, 1, 333, 8192, 5]
    for frac in (0.0, 1.0, 0.33):
        oracle_vs_group(osp, counts, 2, [0.5, 0.5], frac, 4, 3, seed=23, tma=True)
    oracle_vs_group(osp, counts, 1, [1.0], 0.7, 1, 3, seed=29, tma=True)
    for frac in (0.0, 1.0):
        oracle_vs_group(osp, counts, 2, [0.5, 0.5], frac, 4, 2, seed=31, tma=True, carry=False)


def test_carry_flag_reported(osp):
    part = osp.Partition([1000, 5000])
    assert lib_flags(osp, osp.OspGroup(part, 8)) & 4 == 0
    assert lib_flags(osp, osp.OspGroup(part, 8, carry=False)) & 4 == 4
    assert lib_flags(osp, osp.OspGroup(part, 9)) & 4 == 4  # register family: no carry


def lib_flags(osp, grp):
    return osp.lib().osp_group_flags(grp._h)


@pytest.mark.parametrize("n", [3, 5, 6, 7])
def test_tma_group_non_power_of_two_workers(osp, n):
    """N in {3,5,6,7}: TMA family (default shape), ICS carry and the overlapped
    resolve, against the oracle on ragged layers with unequal weights."""
    rng = np.random.default_rng(40 + n)
    counts = [int(c) for c in rng.integers(1, 9000, 29)] + [8192, 4096]
    w = [float(x) for x in 0.1 + rng.random(n)]
    grp = oracle_vs_group(osp, counts, n, w, 0.55, 3, 3, seed=50 + n, tma=True)
    assert grp.stage_kernels == "tma-staged"


def test_tma_matches_default_kernels(osp):
    """Both kernel families on the same inputs: identical G, rows, scores bits."""
    from paper_2306_16926_b200 import layouts
    counts = layouts.resnet50()
    M = sum(counts)
    N = 8
    part = osp.Partition(counts)
    a = osp.OspGroup(part, N, [0.125] * N, n_chunks=4, tma=False)
    b = osp.OspGroup(part, N, [0.125] * N, n_chunks=4, tma=True)
    c = osp.OspGroup(part, N, [0.125] * N, n_chunks=4, tma=True, carry=False)
    for it in range(4):
        X = osp.synth_deltas(5, N, it, M)
        for grp in (a, b, c):
            grp.set_budget(M * 2)
            grp.step(X)
        for other in (b, c):
            assert np.array_equal(bits(a.global_params), bits(other.global_params))
            assert np.array_equal(bits(a.worker_params), bits(other.worker_params))
            assert np.array_equal(a.read_gib()["order"], other.read_gib()["order"])
        # same tiles and lanes: the carried stage-1 partials equal stage 2's bit for bit
        assert np.array_equal(bits(b.scores), bits(c.scores))


def test_group_errors(osp):
    part = osp.Partition([10, 10])
    with pytest.raises(osp.ConfigError):
        osp.OspGroup(part, 2, [0.5, 0.5], n_chunks=0)
    with pytest.raises(osp.ConfigError):
        osp.OspGroup(part, 2, [0.5, -0.5])
    grp = osp.OspGroup(part, 2, [0.5, 0.5])
    with pytest.raises(osp.ShapeError):
        grp.step(torch.zeros((2, 5), device="cuda"))
    with pytest.raises(osp.PartitionError):
        osp.Partition([3, 0])
    with pytest.raises(osp.PartitionError):
        osp.Partition([])
    with pytest.raises(osp.LayerError):
        part.layer(7)


@pytest.mark.parametrize("n", [9, 16, 64, 200])
def test_group_many_workers_vs_oracle(osp, n):
    """N > 8 runs the register family with a runtime worker count (dispatch_n's
    default case) up to OSP_MAX_WORKERS = 256; fixed-order fp64 aggregation over
    all N rows must stay bit-exact with the oracle (protocol.cpp:14-27)."""
    rng = np.random.default_rng(70 + n)
    counts = [int(c) for c in rng.integers(1, 3000, 13)] + [4096]
    w = [float(x) for x in 0.1 + rng.random(n)]
    grp = oracle_vs_group(osp, counts, n, w, 0.5, 3, 2, seed=80 + n)
    assert grp.stage_kernels != "tma-staged"


def test_group_more_than_max_workers_refused(osp):
    part = osp.Partition([100, 200])
    with pytest.raises(osp.InvalidArgument, match="OSP_MAX_WORKERS"):
        osp.OspGroup(part, 257, [1.0 / 257] * 257)


# ---- the single-launch step of launch-bound layouts (kernels/step_small.cu) -----

def test_small_step_matches_reference_engine(osp, golden):
    """osp_group_step as ONE single-CTA launch against the reference-engine
    goldens whose layout qualifies (L <= 32): every vector, the scores, the
    next GIB, its rank order and the device-written wire."""
    g = golden
    part = osp.Partition(g.counts, g.bpe)
    grp = osp.OspGroup(part, g.N, list(g.weights), n_chunks=g.n_chunks, init_params=cuda(g.p0))
    if not (g.L <= 32 and g.M <= 32768 and g.N <= 8):
        assert not grp.single_launch
        pytest.skip("layout above the single-launch limits")
    assert grp.single_launch
    for it in range(g.iters):
        X = cuda(g.deltas(it))
        grp.set_budget(int(g.get(it, "budget")[0]))
        grp.step(X)
        G = grp.global_params.cpu().numpy()
        assert np.array_equal(bits(G), bits(g.get(it, "global"))), f"global, it {it}"
        P = grp.worker_params.cpu().numpy()
        for w in range(g.N):
            assert np.array_equal(bits(P[w]), bits(G)), f"worker {w}, it {it}"
        np.testing.assert_allclose(grp.scores.cpu().numpy(), g.get(it, "scores"), rtol=SCORE_RTOL,
                                   atol=0)
        nxt = grp.read_gib()
        tag_out, flags_out = oracle.gib_decode(bytes(g.get(it, "gib_out")))
        assert nxt["tag"] == tag_out == it + 1
        assert np.array_equal(nxt["flags"], flags_out), f"GIB flags, it {it}"
        assert np.array_equal(nxt["order"], g.get(it, "order_out")), f"ICS order, it {it}"
        order_out = np.asarray(g.get(it, "order_out"), dtype="<u4")
        assert grp.gib_wire() == (bytes(g.get(it, "gib_out")) + struct.pack("<I", order_out.size)
                                  + order_out.tobytes()), f"GIB wire, it {it}"
        if it + 1 < g.iters:  # the chunk map the next split uses
            chunks_ref = Golden.decode_chunks(g.get(it + 1, "chunks"))
            assert nxt["n_used"] == len(chunks_ref)
            for c, ids in enumerate(chunks_ref):
                assert sorted(np.flatnonzero(nxt["chunk_of"] == c).tolist()) == ids


@pytest.mark.parametrize("N,L,frac,chunks,sgd", [(8, 4, 0.5, 4, 0.0), (4, 6, 0.9, 3, 0.0),
                                                  (1, 1, 1.0, 2, 0.0), (3, 32, 0.33, 7, 0.0),
                                                  (5, 17, 0.0, 4, 0.05), (8, 32, 0.6, 9, 0.0)])
def test_small_step_vs_oracle_and_three_launch_step(osp, N, L, frac, chunks, sgd):
    """Random small layouts (odd sizes, unequal weights, random P0, budget edges,
    fused sgd): the single-launch step equals the oracle and the three-launch
    step bit for bit over 5 iterations, the two groups mixed freely."""
    rng = np.random.default_rng(1000 + 7 * N + L)
    counts = rng.integers(1, max(2, 32768 // L // 2), L)
    w = list(0.1 + rng.random(N))
    p0 = rng.uniform(-1, 1, int(counts.sum())).astype(np.float32)
    grp = oracle_vs_group(osp, counts, N, w, frac, chunks, 5, seed=L, p0=p0, sgd_lr=sgd)
    assert grp.single_launch
    M = int(counts.sum())
    part = osp.Partition(counts)
    a = osp.OspGroup(part, N, w, n_chunks=chunks, init_params=cuda(p0), sgd_lr=sgd)
    b = osp.OspGroup(part, N, w, n_chunks=chunks, init_params=cuda(p0), sgd_lr=sgd, small=False)
    assert a.single_launch and not b.single_launch
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    for it in range(6):
        osp.synth_deltas(L, N, it, M, out=X)
        for grp in (a, b):
            grp.set_budget(int(frac * M * 4))
        a.step(X)
        if it % 2:  # the per-stage API on the small group continues from its lists
            b.step(X)
        else:
            b.stage1(X)
            b.stage2_resolve(X)
        assert np.array_equal(bits(a.global_params), bits(b.global_params)), f"it {it}"
        assert np.array_equal(bits(a.worker_params), bits(b.worker_params)), f"it {it}"
        ra, rb = a.read_gib(), b.read_gib()
        for k in ("flags", "order", "chunk_of", "n_used", "tag", "deferred_bytes"):
            assert np.array_equal(ra[k], rb[k]), f"{k} it {it}"
        assert a.gib_wire() == b.gib_wire()
        assert np.array_equal(a.deferred_history(ra["tag"], 1), b.deferred_history(rb["tag"], 1))
    a.stage1(X)  # the per-stage path after single-launch steps
    a.stage2_resolve(X)
    b.step(X)
    assert np.array_equal(bits(a.global_params), bits(b.global_params))


def test_small_step_certificate_fallback(osp):
    """Exact ties (identical layers) in a small layout: the warp resolve cannot
    certify the order from tile sums, recomputes the tied layers sequentially
    and reproduces the reference's stable order."""
    counts = [700, 700, 33, 700]
    M, N = sum(counts), 4
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=2)
    assert grp.single_launch
    G = np.zeros(M, np.float32)
    P = np.zeros((N, M), np.float32)
    flags, order = np.zeros(4, np.uint8), np.zeros(0, np.int32)
    budget = int(0.6 * M * 4)
    X = torch.empty((N, M), dtype=torch.float32, device="cuda")
    for it in range(3):
        osp.synth_deltas(7, N, it, M, out=X)
        X[:, 700:1400] = X[:, :700]
        X[:, 1433:] = X[:, :700]
        r = oracle.step(counts, 4, [0.25] * N, X.cpu().numpy(), G, P, flags, order, 2, budget)
        grp.set_budget(budget)
        grp.step(X)
        assert np.array_equal(bits(grp.global_params), bits(G)), f"global, it {it}"
        assert np.array_equal(bits(grp.worker_params), bits(P)), f"workers, it {it}"
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"]), f"flags, it {it}"
        assert np.array_equal(nxt["order"], r["order_out"]), f"order, it {it}"
        flags, order = r["flags_out"], r["order_out"]
    st = grp.stats()
    assert st["fallback_resolves"] == 3 and st["fallback_layers"] >= 9


def test_small_step_in_cuda_graph(osp):
    """The single-launch step replayed from a CUDA graph equals direct steps."""
    counts = [256, 32, 128, 4]
    M, N = sum(counts), 8
    part = osp.Partition(counts)
    X = [osp.synth_deltas(11, N, i, M) for i in range(2)]
    a = osp.OspGroup(part, N, n_chunks=4)
    b = osp.OspGroup(part, N, n_chunks=4)
    assert b.single_launch
    for grp in (a, b):
        grp.set_budget(M * 2)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cs, capture_error_mode="thread_local"):
        b.step(X[0])
        b.step(X[1])
    torch.cuda.synchronize()
    for r in range(3):
        a.step(X[0])
        a.step(X[1])
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(bits(a.global_params), bits(b.global_params)), f"replay {r}"
        assert np.array_equal(bits(a.worker_params), bits(b.worker_params)), f"replay {r}"
        assert a.gib_wire() == b.gib_wire()


@pytest.mark.parametrize("case", ["random", "ties", "edges"])
def test_pgp_rank_gib_certified_vs_oracle(osp, case):
    """osp_pgp_rank_gib (the façade's resolution step): certified tree sums +
    exact fallback reproduce the reference's deferred set and rank order
    (importance.cpp:11-59) on arbitrary vectors, incl. exact ties."""
    rng = np.random.default_rng({"random": 1, "ties": 2, "edges": 3}[case])
    counts = [int(c) for c in rng.integers(1, 30000, 41)]
    if case == "ties":
        counts[5] = counts[9] = counts[20] = 4096
    M = sum(counts)
    p = rng.uniform(-1, 1, M).astype(np.float32)
    g = rng.uniform(-1e-3, 1e-3, M).astype(np.float32)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    if case == "ties":
        for l in (9, 20):
            p[offs[l]:offs[l + 1]] = p[offs[5]:offs[6]]
            g[offs[l]:offs[l + 1]] = g[offs[5]:offs[6]]
    part = osp.Partition(counts)
    ref_scores = oracle.pgp(counts, p, g)
    budgets = [int(0.5 * M * 4)] if case != "edges" else [0, 1, M * 4, M * 4 - 1, int(0.37 * M * 4)]
    for budget in budgets:
        scores, order, flags = osp.pgp_rank_gib(part, cuda(p), cuda(g), budget)
        want_flags = oracle.build_gib(ref_scores, counts, 4, budget)
        want_order = oracle.rank(ref_scores)[: int(want_flags.sum())]
        assert np.array_equal(flags, want_flags), f"flags at budget {budget}"
        assert np.array_equal(order, want_order), f"order at budget {budget}"
        np.testing.assert_allclose(scores, ref_scores, rtol=SCORE_RTOL, atol=0)
        if case == "ties":
            assert scores[5] == scores[9] == scores[20] == ref_scores[5]
