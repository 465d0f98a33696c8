"""Chain form, each role alone (osp_shard_solo_agg: PRE / FIN items without
flags), for ncu: OSP_SHARD_SYNC=chain torchrun --nproc-per-node 2 tools/chain_solo.py"""
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
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    counts = layouts.get(layout)
    part = osp.Partition(counts)
    sh = ShardGroup(part, 8, None, n_chunks=4)
    sh.connect_via()
    for b in range(2):
        sh.fill_synth(11, b, b)
    sh.set_budget(int(0.5 * 4 * sum(counts)))
    for k in range(4):
        sh.step(k % 2)
    torch.cuda.synchronize()
    dist.barrier()
    for k in range(3):
        sh.solo_agg(1, k % 2)
    torch.cuda.synchronize()
    dist.barrier()
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
