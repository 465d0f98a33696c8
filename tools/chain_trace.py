"""Timeline of the chain form's stage 1 (diagnostics; torchrun, one process per GPU).

OSP_SHARD_DEBUG=2 OSP_SHARD_SYNC=chain torchrun --nproc-per-node 2 tools/chain_trace.py [layout]

Runs warm-up steps, then one step, and gathers every rank's per-tile globaltimer
stamps (osp_shard_debug_trace) to rank 0, which writes them to
gpurun_out/r2_chain_trace.npz and prints the fronts: when each fraction of the
tiles was PRE-published (rank 0), FIN-acquired / FIN-published (last rank) and
APPLY-done (rank 0), relative to the first PRE issue.
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from paper_2306_16926_b200 import layouts, osp
    from paper_2306_16926_b200.dist import ShardGroup
    layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    counts = layouts.get(layout)
    M = sum(counts)
    part = osp.Partition(counts)
    sh = ShardGroup(part, 8, None, n_chunks=4)
    sh.connect_via()
    assert sh.sync_form == "chain", sh.sync_form
    for b in range(2):
        sh.fill_synth(11, b, b)
    sh.set_budget(int(0.5 * 4 * M))
    for k in range(20):
        sh.step(k % 2)
    sh.check()
    torch.cuda.synchronize()
    dist.barrier()
    # two back-to-back steps; the trace keeps the second's stage 1, the host
    # stamps bracket both
    for k in range(2):
        sh.step(k % 2)
    torch.cuda.synchronize()
    sh.check()
    tr = torch.as_tensor(sh.debug_trace().astype(np.int64), device="cuda")
    allt = [torch.zeros_like(tr) for _ in range(world)]
    dist.all_gather(allt, tr)
    if rank == 0:
        a = [x.cpu().numpy() for x in allt]
        os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
        np.savez(os.path.join(REPO, "gpurun_out", f"r2_chain_trace_{layout}.npz"),
                 **{f"rank{r}": a[r] for r in range(world)})
        t0 = a[0][0][a[0][0] > 0].min()
        fin = a[world - 1]

        def front(x):
            x = np.sort(x[x > 0] - t0) / 1e3
            if len(x) == 0:
                return None
            return {f"p{p}": round(float(np.percentile(x, p)), 1) for p in (0, 10, 25, 50, 75, 90, 100)}

        out = {"layout": layout, "world": world, "NT": int(a[0].shape[1]),
               "us_since_first_pre_issue": {
                   "pre_issue_r0": front(a[0][0]), "pre_pub_r0": front(a[0][2]),
                   "fin_acq": front(fin[3]), "fin_pub": front(fin[4]),
                   "apply_acq_r0": front(a[0][5]), "apply_done_r0": front(a[0][6])}}
        lag = (fin[3] - a[world - 2][2]).astype(np.float64) / 1e3
        out["fin_acq_minus_prev_pre_pub_us"] = {f"p{p}": round(float(np.percentile(lag, p)), 2)
                                                for p in (0, 10, 50, 90, 100)}
        print(json.dumps(out), flush=True)
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
