"""Smoke-size workloads for compute-sanitizer (tools/sanitize.sh): every kernel
family of the step on a tiny ragged layout, checked against the oracle so a
sanitizer run also proves the results unchanged.

  python tools/sanitize_step.py group      TMA stage 1 / overlapped resolve + stage-3 join
  python tools/sanitize_step.py register   register-staged stage kernels + resolve
  python tools/sanitize_step.py small      the single-launch small step
  python tools/sanitize_step.py shard      (one rank of a 2-rank oversubscribed shard job,
                                            launched by tools/sanitize.sh)
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402


def group_case(kind):
    from paper_2306_16926_b200 import osp
    counts = [2100, 64, 3, 5000, 17, 1024, 777] if kind != "small" else [256, 32, 128, 4]
    N, M = 4, None
    M = sum(counts)
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=3,
                       tma={"group": True, "register": False, "small": None}[kind],
                       small=kind == "small")
    if kind == "small":
        assert grp.single_launch
    G = np.zeros(M, np.float32)
    P = np.zeros((N, M), np.float32)
    flags, order = np.zeros(len(counts), np.uint8), np.zeros(0, np.int32)
    budget = int(0.5 * M * 4)
    for it in range(3):
        X = osp.synth_deltas(5, N, it, M)
        r = oracle.step(counts, 4, [0.25] * N, X.cpu().numpy(), G, P, flags, order, 3, budget)
        grp.set_budget(budget)
        grp.step(X)
        torch.cuda.synchronize()
        assert np.array_equal(grp.global_params.cpu().numpy().view(np.uint32), G.view(np.uint32))
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"])
        assert np.array_equal(nxt["order"], r["order_out"])
        flags, order = r["flags_out"], r["order_out"]
    print(f"sanitize {kind}: ok")


def shard_case():
    import torch.distributed as dist

    from paper_2306_16926_b200 import dist as odist
    from paper_2306_16926_b200 import osp
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    counts = [2100, 64, 3, 5000, 17, 1024, 777]
    N, M = 4, sum(counts)
    w = [0.25] * N
    part = osp.Partition(counts)
    for defer in (False, True):
        sh = odist.ShardGroup(part, N, w, n_chunks=3, defer_ics=defer)
        sh.connect_via()
        G = np.zeros(M, np.float32)
        P = np.zeros((N, M), np.float32)
        flags, order = np.zeros(len(counts), np.uint8), np.zeros(0, np.int32)
        budget = int(0.5 * M * 4)
        for it in range(2):
            sh.fill_synth(5, it, it % 2)
            X = np.stack([oracle.synth_delta(5, k, it, M) for k in range(N)])
            r = oracle.step(counts, 4, w, X, G, P, flags, order, 3, budget)
            sh.set_budget(budget)
            sh.step(it % 2)
            sh.check()
            assert np.array_equal(sh.global_params.cpu().numpy().view(np.uint32), G.view(np.uint32))
            flags, order = r["flags_out"], r["order_out"]
        dist.barrier()
        sh.close()
    dist.destroy_process_group()
    print(f"sanitize shard rank {rank}: ok")


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "shard":
        shard_case()
    else:
        group_case(kind)
