"""Sharded exchange kernel diagnostics (torchrun, one process per GPU):
step time, phases, the kernel's debug counters per step, and the exchange alone
(every rank's own tiles, no flags; all ranks at once) for a layout / tile / lag /
ring-depth variant given by the environment.

  OSP_SHARD_DEBUG=1 torchrun --nproc-per-node 2 tools/shard_x_diag.py [layout] [tile]
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from paper_2306_16926_b200 import layouts, osp
    from paper_2306_16926_b200.dist import ShardGroup
    layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    counts = layouts.get(layout)
    M = sum(counts)
    part = osp.Partition(counts)
    sh = ShardGroup(part, 8, None, n_chunks=4, tile_elems=tile)
    sh.connect_via()
    for b in range(2):
        sh.fill_synth(11, b, b)
    sh.set_budget(int(0.5 * 4 * M))
    for k in range(10):
        sh.step(k % 2)
    sh.check()
    sh.debug_counters()
    torch.cuda.synchronize()
    dist.barrier()
    K = 100
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(K):
        sh.step(k % 2)
    e.record()
    torch.cuda.synchronize()
    sh.check()
    step_ms = s.elapsed_time(e) / K
    dbg = sh.debug_counters()
    if dbg:
        dbg = {k: v / K for k, v in dbg.items()}
    phases = [sh.profile(k % 2) for k in range(5)]
    ph = {k: sum(p[k] for p in phases) / 5 for k in phases[0]}
    # the exchange alone: own tiles only, all ranks together
    dist.barrier()
    torch.cuda.synchronize()
    dist.barrier()
    s.record()
    for k in range(20):
        sh.solo_agg(1, k % 2)
    e.record()
    torch.cuda.synchronize()
    solo_ms = s.elapsed_time(e) / 20
    solo_dbg = sh.debug_counters()
    solo_t = torch.tensor([solo_ms], dtype=torch.float64, device="cuda")
    solo_all = [torch.zeros_like(solo_t) for _ in range(world)]
    dist.all_gather(solo_all, solo_t)
    solo_per_rank = [float(x.item()) for x in solo_all]
    sk = sorted(solo_dbg) if solo_dbg else []
    sv = torch.tensor([solo_dbg[k] / 20 for k in sk] if solo_dbg else [0.0], dtype=torch.float64, device="cuda")
    sva = [torch.zeros_like(sv) for _ in range(world)]
    dist.all_gather(sva, sv)
    solo_dbg_all = [dict(zip(sk, v.tolist())) for v in sva] if solo_dbg else None
    t = torch.tensor([step_ms, solo_ms] + [ph[k] for k in ph], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # every rank's counters (the chain form's ranks play different roles)
    keys = sorted(dbg) if dbg else []
    dv = torch.tensor([dbg[k] for k in keys] if dbg else [0.0], dtype=torch.float64, device="cuda")
    allv = [torch.zeros_like(dv) for _ in range(world)]
    dist.all_gather(allv, dv)
    dbg_all = [dict(zip(keys, v.tolist())) for v in allv] if dbg else None
    if rank == 0:
        n_loc = 8 // world
        nvl = 4.0 * M * ((8 - n_loc) / world + (world - 1) / world)
        vals = t.tolist()
        print(json.dumps({"layout": layout, "tile": sh.local.geometry()["tile_elems"],
                          "lag": os.environ.get("OSP_SHARD_LAG", "2"),
                          "world": world, "step_ms": vals[0], "solo_exchange_ms": vals[1],
                          "phases_ms": dict(zip(ph, vals[2:])),
                          "nvlink_GBps_step": nvl / (vals[0] * 1e-3) / 1e9,
                          "sync": sh.sync_form, "solo_ms_per_rank": solo_per_rank,
                          "solo_debug_per_step": solo_dbg_all,
                          "debug_per_step": dbg_all}), flush=True)
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
