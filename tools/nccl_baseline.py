"""NCCL baseline for the sharded exchange (diagnostic; torchrun, one rank per GPU).

The exact-mode exchange of SURVEY §8(e) done with NCCL instead of our fused
peer-memory kernels: every rank packs its N/P worker rows per owner shard,
`all_to_all_single` moves them to the owners (push = reduce-scatter input), and
`all_gather_into_tensor` returns the owners' aggregates (pull). Only the
communication (+ packing) is timed — the fixed-order fp64 aggregation, the
apply and the resolve would come on top. Compare with bench.py --gpus P
(our whole step).
Usage: torchrun --nproc-per-node P tools/nccl_baseline.py [layout]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2306_16926_b200 import layouts  # noqa: E402

layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
M = sum(layouts.get(layout))
N = 8
n_loc = N // world
shard = (M + world - 1) // world
X = torch.randn(n_loc, shard * world, device="cuda")      # this rank's worker rows
send = torch.empty(world, n_loc, shard, device="cuda")   # packed per owner
recv = torch.empty(world, n_loc, shard, device="cuda")   # every worker's rows of my shard
agg = torch.randn(shard, device="cuda")
full = torch.empty(shard * world, device="cuda")


def exchange():
    send.copy_(X.view(n_loc, world, shard).transpose(0, 1))       # pack
    dist.all_to_all_single(recv.view(-1), send.view(-1))           # push (rows to owners)
    dist.all_gather_into_tensor(full, agg)                         # pull (aggregates)


for _ in range(5):
    exchange()
torch.cuda.synchronize()
dist.barrier()
K = 50
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(K):
    exchange()
b.record()
torch.cuda.synchronize()
ms = torch.tensor([a.elapsed_time(b) / K], device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
if rank == 0:
    bytes_dir = 4.0 * n_loc * shard * (world - 1) + 4.0 * shard * (world - 1)
    print(json.dumps({"layout": layout, "P": world, "nccl_exchange_ms": round(ms.item(), 4),
                      "bytes_per_direction_per_gpu": bytes_dir,
                      "gbs_per_direction": round(bytes_dir / (ms.item() * 1e-3) / 1e9, 1),
                      "note": "pack + all_to_all rows + all_gather aggregates; no aggregation, "
                              "apply or resolve"}), flush=True)
dist.barrier()
dist.destroy_process_group()
