"""Resolve kernel alone (diagnostic): back-to-back osp_group_resolve launches
after one step, event-timed, per layout."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_16926_b200 import layouts, osp  # noqa: E402

for name in (sys.argv[1:] or ["resnet50", "resnet152", "vgg16", "llama1b"]):
    counts = layouts.get(name)
    M, N = sum(counts), 8
    grp = osp.OspGroup(osp.Partition(counts), N, n_chunks=4)
    X = osp.synth_deltas(11, N, 0, M)
    grp.set_budget(int(0.5 * M * 4))
    grp.step(X)
    grp.stage1(X)
    grp.stage2_all(X)
    for _ in range(5):
        grp.resolve(X)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        grp.resolve(X)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:9s} L={len(counts):4d} tiles={grp.geometry()['n_tiles']:7d} resolve "
          f"{a.elapsed_time(b) / 100 * 1e3:.1f} us", flush=True)
    del grp, X
    torch.cuda.empty_cache()
