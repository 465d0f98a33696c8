"""The message-level engine C-ABI (include/osp_engine.h, engine.py) driven in
the reference harness's synchronous message order must reproduce the
reference-engine dumps (tests/golden/*.npz, oracle/ref_driver.cpp) bit for
bit: stage-1 worker params, the global vector and the GIB bytes of every
iteration, with the reference's server options (fixed or tuned budget)."""
import math

import numpy as np
import pytest

from osp_testlib import Golden

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def engine():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2306_16926_b200 import engine as e
    return e


def make_engines(engine, g: Golden):
    cfg = g.cfg
    part = engine.Partition([int(c) for c in g.counts], g.bpe)
    fixed = None
    if "budget" in cfg:
        fixed = int(cfg["budget"])
    elif "budget_frac" in cfg:
        fixed = int(math.floor(cfg["budget_frac"] * float(g.M * g.bpe)))
    server = engine.OspServer(part, list(g.weights), init_global=g.p0, u_max=int(cfg.get("umax", 0)),
                              iterations_per_epoch=int(cfg.get("ipe", 1)), fixed_budget_bytes=fixed)
    workers = [engine.OspWorker(part, w, init_params=g.p0, subset_weight=float(g.weights[w]))
               for w in range(g.N)]
    return part, server, workers


def test_engine_capi_matches_reference_engine(engine, golden):
    from oracle import oracle
    part, server, workers = make_engines(engine, golden)
    for it in range(golden.iters):
        loss = 0.7 ** (server.epoch_of_iteration(it) - 1)
        stage1, gib = engine.run_synchronous_iteration(server, workers, it, golden.deltas(it), loss,
                                                       golden.n_chunks)
        ref1 = golden.get(it, "params_stage1")
        if ref1 is not None:
            for w in range(golden.N):
                assert np.array_equal(bits(stage1[w]), bits(ref1[w])), f"stage-1 worker {w}, it {it}"
        else:
            assert np.array_equal(bits(stage1[0]), bits(golden.get(it, "params_stage1_w0")))
        G = server.global_params()
        assert np.array_equal(bits(G), bits(golden.get(it, "global"))), f"global, it {it}"
        for w in workers:
            assert np.array_equal(bits(w.params()), bits(G)), f"worker params, it {it}"
        assert gib.gib() == bytes(golden.get(it, "gib_out")), f"GIB bytes, it {it}"
        assert np.array_equal(gib.rank_order(), golden.get(it, "order_out")), f"order, it {it}"
        assert gib.kind == "GibUpdate" and gib.iteration == it + 1
    tag, _ = oracle.gib_decode(gib.gib())
    assert tag == golden.iters


def test_engine_capi_errors(engine):
    from paper_2306_16926_b200 import osp
    part = engine.Partition([4, 4])
    w = engine.OspWorker(part, 0, subset_weight=1.0)
    with pytest.raises(osp.ShapeError):
        w.on_compute_done(0, np.zeros(3, np.float32), 1.0, 2)
    server = engine.OspServer(part, [1.0], fixed_budget_bytes=0)
    rs, lr, chunks = w.on_compute_done(0, np.ones(8, np.float32), 1.0, 2)
    assert rs.kind == "PushImportant" and lr.kind == "LossReport" and chunks == []
    out = server.on_push_important(rs)
    assert out["pull_important"] is not None and out["pull_important"].kind == "PullImportant"
    with pytest.raises(osp.ProtocolError):
        w.on_compute_done(5, np.ones(8, np.float32), 1.0, 2)  # worker is at iteration 0
