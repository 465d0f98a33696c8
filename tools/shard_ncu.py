"""ncu evidence for the multi-GPU aggregate kernel (k_shard_agg). The step's
kernels order themselves across GPUs in-kernel, and ncu serialises kernels, so
a profiled multi-rank step times out by design (bounded waits). Instead every
rank sets up, connects and fills its delta rows; then rank 0 alone launches
its stage-1 push/pull (osp_shard_solo_agg: peers' rows over NVLink, fixed-order
fp64 aggregate, fp32 result stored into every rank) while the others wait on a
host barrier. Run under torchrun with ncu filtered to k_shard_agg, e.g.
  ncu --target-processes all -k regex:k_shard_agg --metrics ... \
      python -m torch.distributed.run --nproc-per-node 2 tools/shard_ncu.py
Without ncu it prints the solo launch's event time and NVLink byte rate.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16926_b200 import layouts, osp  # noqa: E402
from paper_2306_16926_b200.dist import ShardGroup  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    layout = os.environ.get("LAYOUT", "resnet50")
    counts = layouts.get(layout)
    M, N = sum(counts), 8
    part = osp.Partition(counts)
    sh = ShardGroup(part, N, None, n_chunks=4)
    sh.connect_via()
    sh.fill_synth(11, 0, 0)
    torch.cuda.synchronize()
    dist.barrier()
    if os.environ.get("BOTH") == "1":
        # every rank launches its solo push/pull at once: the bidirectional
        # exchange without the step's cross-GPU ordering
        reps = int(os.environ.get("REPS", "5"))
        res = []
        for r in range(reps):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sh.solo_agg(1, 0)
            b.record()
            torch.cuda.synchronize()
            res.append(a.elapsed_time(b))
        t = torch.tensor([min(res)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            P, nl = world, N // world
            per_dir = 4.0 * M * ((N - nl) / P + (P - 1) / P)
            print(json.dumps({"layout": layout, "P": P, "both_solo_agg_ms_max": float(t[0]),
                              "per_direction_GBps": per_dir / (float(t[0]) * 1e-3) / 1e9}),
                  flush=True)
    elif rank == 0:
        reps = int(os.environ.get("REPS", "3"))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        for r in range(reps):
            ev[2 * r].record()
            sh.solo_agg(1, 0)  # bootstrap GIB: every layer in stage 1
            ev[2 * r + 1].record()
        torch.cuda.synchronize()
        ms = min(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps))
        P, nl = world, N // world
        # this owner's range: M/P elements; reads (N - N/P) peer rows, writes P-1 peer copies
        rx = 4.0 * (M / P) * (N - nl)
        tx = 4.0 * (M / P) * (P - 1)
        print(json.dumps({"layout": layout, "P": P, "solo_agg_ms": ms,
                          "nvlink_rx_GBps": rx / (ms * 1e-3) / 1e9,
                          "nvlink_tx_GBps": tx / (ms * 1e-3) / 1e9,
                          "note": "one owner alone (peers idle): one-way read rate, not the "
                                  "bidirectional step"}), flush=True)
    dist.barrier()
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
