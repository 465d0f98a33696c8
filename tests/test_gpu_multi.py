"""Multi-GPU parity: the sharded path (osp_shard_*, NVLink peer memory) must be
bit-identical to the oracle — global replica on every rank, every rank's
worker rows, and the next GIB — for several iterations, in both exchange modes
(single exchange with the ICS carry; deferred ICS). The *_oversubscribed tests
run on any box (ranks share the GPUs that exist), the others need world GPUs."""
import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    try:
        sys.path.insert(0, REPO)
        import torch.distributed as dist

        from oracle import oracle
        from paper_2306_16926_b200 import dist as odist
        from paper_2306_16926_b200 import osp

        torch.cuda.set_device(rank % torch.cuda.device_count())
        if cfg.get("sync"):
            os.environ["OSP_SHARD_SYNC"] = cfg["sync"]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        counts = np.asarray(cfg["counts"], dtype=np.uint64)
        N, M, nc = cfg["N"], int(counts.sum()), cfg["chunks"]
        w = cfg["weights"]
        budget = int(cfg["budget_frac"] * M * 4)
        rng = np.random.default_rng(cfg["p0_seed"])
        p0 = rng.uniform(-1, 1, M).astype(np.float32) if cfg["p0_seed"] else np.zeros(M, np.float32)
        part = osp.Partition(counts)
        sh = odist.ShardGroup(part, N, w, n_chunks=nc, init_params=torch.as_tensor(p0, device="cuda"),
                              tile_elems=cfg.get("tile", 0), defer_ics=cfg.get("defer", False),
                              sgd_lr=cfg.get("sgd_lr", 0.0))
        sh.connect_via()
        assert sh.deferred_ics == bool(cfg.get("defer", False)), "shard exchange mode"
        if cfg.get("sync") and not cfg.get("defer"):
            assert sh.sync_form == cfg["sync"], (sh.sync_form, cfg["sync"])
        if cfg.get("expect_sync"):
            assert sh.sync_form == cfg["expect_sync"], (sh.sync_form, cfg["expect_sync"])
        G = p0.copy()
        P = np.tile(p0, (N, 1))
        flags = np.zeros(len(counts), np.uint8)
        order = np.zeros(0, np.int32)
        for it in range(cfg["iters"]):
            buf = it % 2
            if rank == cfg.get("lag_rank", -1):  # this rank's host falls behind its peers
                import time
                torch.cuda.synchronize()
                time.sleep(0.3)
            sh.fill_synth(cfg["seed"], it, buf)
            deltas = np.stack([oracle.synth_delta(cfg["seed"], k, it, M) for k in range(N)])
            for (dst, src, n) in cfg.get("copy_layers", []):  # identical layers: exact PGP ties
                x = sh.deltas(buf)
                x[:, dst:dst + n] = x[:, src:src + n]
                deltas[:, dst:dst + n] = deltas[:, src:src + n]
            if cfg.get("sgd_lr"):  # the rows are gradients: the step applies sgd_delta
                x = sh.deltas(buf)
                x.mul_(37.0)
                raw = deltas * np.float32(37.0)
                deltas = np.stack([oracle.sgd_delta(raw[k], cfg["sgd_lr"]) for k in range(N)])
            r = oracle.step(counts, 4, w, deltas, G, P, flags, order, nc, budget)
            sh.set_budget(budget)
            if cfg.get("per_chunk"):
                sh.stage1(buf)
                sh.check()
                # stage-1 state: RS layers G', deferred layers the local estimate
                p1 = sh.worker_params.cpu().numpy()
                mine1 = r["p_stage1"][rank * sh.n_loc:(rank + 1) * sh.n_loc]
                assert np.array_equal(p1.view(np.uint32), mine1.view(np.uint32)), \
                    f"stage-1 rows rank {rank} it {it}"
                for c in range(nc):
                    sh.stage2(buf, c, c + 1)
                sh.resolve(buf)
            else:
                sh.step(buf)
            sh.check()
            g_dev = sh.global_params.cpu().numpy()
            assert np.array_equal(g_dev.view(np.uint32), G.view(np.uint32)), f"G rank {rank} it {it}"
            p_dev = sh.worker_params.cpu().numpy()
            mine = P[rank * sh.n_loc:(rank + 1) * sh.n_loc]
            assert np.array_equal(p_dev.view(np.uint32), mine.view(np.uint32)), f"P rank {rank}"
            nxt = sh.read_gib()
            assert np.array_equal(nxt["flags"], r["flags_out"]), f"flags rank {rank} it {it}"
            assert np.array_equal(nxt["order"], r["order_out"]), f"order rank {rank} it {it}"
            flags, order = r["flags_out"], r["order_out"]
        if cfg.get("copy_layers"):
            assert sh.local.stats()["fallback_layers"] > 0, "ties must take the exact fallback"
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def run_world(cfg, world=2, oversubscribe=False):
    if torch.cuda.device_count() < world and not oversubscribe:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    bad = {r: m for r, m in results.items() if m != "ok"}
    assert not bad, bad


@pytest.mark.parametrize("defer,sync", [(False, None), (True, None), (False, "tile"),
                                        (False, "barrier")])
def test_shard_two_gpus_resnet_like(defer, sync):
    """Default form at 2 ranks (the chain for the single exchange), the
    deferred-ICS mode, and the single exchange in the other two forms."""
    from paper_2306_16926_b200 import layouts
    run_world(dict(counts=layouts.resnet50()[:60], N=8, weights=[0.125] * 8, chunks=4,
                   budget_frac=0.5, iters=3, seed=11, p0_seed=0, defer=defer, sync=sync))


@pytest.mark.parametrize("defer", [False, True])
def test_shard_two_gpus_ragged_unequal_weights_per_chunk(defer):
    # odd layer sizes: unstaged (scalar) tiles next to staged ones; per-chunk stage 2
    rng = np.random.default_rng(3)
    counts = [int(c) for c in rng.integers(1, 7000, 37)]
    w = [float(x) for x in 0.1 + rng.random(4)]
    run_world(dict(counts=counts, N=4, weights=w, chunks=3, budget_frac=0.7, iters=4, seed=5,
                   p0_seed=9, tile=512, per_chunk=True, defer=defer))


@pytest.mark.parametrize("frac", [0.0, 1.0])
def test_shard_budget_edges(frac):
    # 0.0: every layer in the barrier; 1.0: every layer deferred
    from paper_2306_16926_b200 import layouts
    for defer in (False, True):
        run_world(dict(counts=layouts.resnet50()[:50], N=8, weights=[0.125] * 8, chunks=4,
                       budget_frac=frac, iters=3, seed=13, p0_seed=7, defer=defer))


@pytest.mark.parametrize("defer", [False, True])
def test_shard_four_gpus(defer):
    from paper_2306_16926_b200 import layouts
    run_world(dict(counts=layouts.resnet50()[:80], N=8, weights=[0.125] * 8, chunks=4,
                   budget_frac=0.5, iters=3, seed=11, p0_seed=0, defer=defer), world=4)


@pytest.mark.parametrize("per_chunk", [False, True])
def test_shard_chain_two_gpus(per_chunk):
    """The reduction-chain form of stage 1 (kernels/shard_chain.cu): rank 1
    continues rank 0's fp64 running sum; ragged layers, unequal weights, P0."""
    rng = np.random.default_rng(41)
    counts = [int(c) for c in rng.integers(1, 30000, 37)]
    w = [float(x) for x in 0.1 + rng.random(8)]
    run_world(dict(counts=counts, N=8, weights=w, chunks=4, budget_frac=0.5, iters=4, seed=13,
                   p0_seed=2, per_chunk=per_chunk, sync="chain"))


def test_shard_chain_four_gpus():
    """Chain over 4 ranks: two middle ranks continue the running sum."""
    rng = np.random.default_rng(43)
    counts = [int(c) for c in rng.integers(1, 30000, 29)]
    w = [float(x) for x in 0.1 + rng.random(8)]
    run_world(dict(counts=counts, N=8, weights=w, chunks=4, budget_frac=0.4, iters=3, seed=17,
                   p0_seed=3, sync="chain"), world=4)


def test_shard_four_gpus_ragged_per_chunk():
    rng = np.random.default_rng(12)
    counts = [int(c) for c in rng.integers(1, 20000, 30)]
    w = [float(x) for x in 0.1 + rng.random(8)]
    run_world(dict(counts=counts, N=8, weights=w, chunks=4, budget_frac=0.5, iters=3, seed=3,
                   p0_seed=5, per_chunk=True), world=4)


def test_shard_many_workers_unstaged():
    """N = 16 workers (more rows than a ring slot holds): the exchange reads
    every row straight from (peer) global memory."""
    rng = np.random.default_rng(77)
    counts = [int(c) for c in rng.integers(1, 3000, 19)]
    w = [float(x) for x in 0.1 + rng.random(16)]
    run_world(dict(counts=counts, N=16, weights=w, chunks=3, budget_frac=0.5, iters=3, seed=9,
                   p0_seed=1), world=2, oversubscribe=True)


# ---- runs on any box: ranks share the GPUs that exist (time-sliced contexts,
# CUDA IPC between processes on one device), so the sharded kernels are
# checked bit-exact against the oracle even on the 1-GPU box; timing meaningless

def _ragged(seed, n_layers, hi):
    rng = np.random.default_rng(seed)
    return [int(c) for c in rng.integers(1, hi, n_layers)]


@pytest.mark.parametrize("world,N,frac", [(2, 8, 0.5), (2, 4, 0.0), (2, 4, 1.0)])
def test_shard_oversubscribed_ragged(world, N, frac):
    """world ranks on however many GPUs exist: ragged layers (odd sizes, scalar
    tails), unequal weights, random P0, per-chunk and fused steps, 3 iterations,
    bit-exact vs the oracle's fixed-order aggregation (protocol.cpp:9-30)."""
    rng = np.random.default_rng(31 + N)
    w = [float(x) for x in 0.1 + rng.random(N)]
    cfg = dict(counts=_ragged(7 + N, 23, 5000), N=N, weights=w, chunks=3, budget_frac=frac,
               iters=3, seed=5, p0_seed=4)
    run_world(cfg, world=world, oversubscribe=True)
    run_world(dict(cfg, per_chunk=True, defer=True), world=world, oversubscribe=True)
    run_world(dict(cfg, per_chunk=True), world=world, oversubscribe=True)


@pytest.mark.parametrize("per_chunk", [False, True])
def test_shard_deferred_all_ics_lagging_rank(per_chunk):
    """Budget = the whole model in the deferred-ICS mode: from iteration 1 stage 1
    exchanges no barrier tile, so its launch must still establish that every
    peer's deltas of the iteration are in place before stage 2 reads them; rank 1's
    host lags every iteration to expose a missing wait."""
    rng = np.random.default_rng(61)
    w = [float(x) for x in 0.1 + rng.random(4)]
    cfg = dict(counts=_ragged(17, 15, 6000), N=4, weights=w, chunks=3, budget_frac=1.0,
               iters=4, seed=3, p0_seed=2, defer=True, per_chunk=per_chunk, lag_rank=1)
    run_world(cfg, world=2, oversubscribe=True)


@pytest.mark.parametrize("world,sync,defer", [(2, "chain", False), (2, "tile", False), (4, None, False),
                                              (2, None, True)])
def test_shard_fused_sgd_oversubscribed(world, sync, defer):
    """Gradients as the rows, sgd_delta fused into the exchange (learner.cpp:
    391-398): every form (chain, per-tile flags, the barrier form at 4 ranks,
    the deferred mode), bit-exact vs the oracle fed with the CPU sgd_delta."""
    rng = np.random.default_rng(91 + world)
    w = [float(x) for x in 0.1 + rng.random(8)]
    cfg = dict(counts=_ragged(29 + world, 19, 5000), N=8, weights=w, chunks=3, budget_frac=0.5,
               iters=3, seed=13, p0_seed=6, sgd_lr=0.05, sync=sync, defer=defer)
    run_world(cfg, world=world, oversubscribe=True)


def test_shard_chain_falls_back_above_eight_local_workers():
    """32 workers on 2 ranks (16 per rank): more local rows than the TMA stage
    family holds, so the local group has no carry buffer and the shard runs
    the deferred-ICS mode with per-tile flags (unstaged rows), not the chain —
    still bit-exact."""
    rng = np.random.default_rng(5)
    w = [float(x) for x in 0.1 + rng.random(32)]
    run_world(dict(counts=_ragged(41, 9, 1500), N=32, weights=w, chunks=2, budget_frac=0.5,
                   iters=2, seed=21, p0_seed=3, defer=True, expect_sync="tile"), world=2,
              oversubscribe=True)


@pytest.mark.parametrize("sync", ["chain", "tile"])
def test_shard_exact_ties_oversubscribed(sync):
    """Identical layers tie exactly: every rank's resolve must take the exact
    sequential fallback, which reads the applied aggregate (in the chain form
    the last rank's, over NVLink) and reproduce the reference's stable order."""
    h = 30_000
    cfg = dict(counts=[h, h, 1000, h], N=8, weights=[0.125] * 8, chunks=2, budget_frac=0.6,
               iters=3, seed=7, p0_seed=0, sync=sync,
               copy_layers=[(h, 0, h), (2 * h + 1000, 0, h)])
    run_world(cfg, world=2, oversubscribe=True)


@pytest.mark.parametrize("world,N,frac", [(2, 8, 0.5), (4, 8, 0.3), (2, 2, 1.0), (8, 8, 0.6)])
def test_shard_chain_oversubscribed(world, N, frac):
    """The chain form on however many GPUs exist: first, middle and last ranks,
    ragged layers (unstaged scalar tiles), budgets 0.3..1.0, per-chunk and fused
    steps, bit-exact vs the oracle."""
    rng = np.random.default_rng(51 + world + N)
    w = [float(x) for x in 0.1 + rng.random(N)]
    cfg = dict(counts=_ragged(13 + world, 21, 4000), N=N, weights=w, chunks=3, budget_frac=frac,
               iters=3, seed=7, p0_seed=9, sync="chain")
    run_world(cfg, world=world, oversubscribe=True)
    run_world(dict(cfg, per_chunk=True), world=world, oversubscribe=True)


def test_shard_eight_ranks_oversubscribed():
    """World size 8 (one worker per rank) on whatever GPUs exist: exercises the
    P = 8 host logic, handle exchange and n_loc = 1 kernels; timing meaningless."""
    from paper_2306_16926_b200 import layouts
    run_world(dict(counts=layouts.resnet50()[:20], N=8, weights=[0.125] * 8, chunks=4,
                   budget_frac=0.5, iters=2, seed=11, p0_seed=0), world=8, oversubscribe=True)
    rng = np.random.default_rng(8)
    w = [float(x) for x in 0.1 + rng.random(8)]
    run_world(dict(counts=_ragged(9, 17, 3000), N=8, weights=w, chunks=4, budget_frac=0.6,
                   iters=2, seed=3, p0_seed=6, defer=True, per_chunk=True), world=8,
              oversubscribe=True)
