"""Register-staged vs TMA-staged stage kernels on one GPU (diagnostic).
Prints ms per stage-1 / stage-2 / full step for each variant and layout."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_16926_b200 import layouts, osp  # noqa: E402

K = 100


def timed(fn, k=K):
    for i in range(6):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(k):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


import argparse  # noqa: E402
import os  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layouts", default="resnet50,vgg16")
ap.add_argument("--variants", default="reg-512,tma-512,reg-1024,tma-1024")
args = ap.parse_args()
tag = f"cw={os.environ.get('OSP_TMA_CW', '-')} ks={os.environ.get('OSP_TMA_STAGES', '-')}"


def variant(v):
    kind, tile = v.split("-")
    return {"tma": kind == "tma", "tile_elems": int(tile)}


for layout in args.layouts.split(","):
    counts = layouts.get(layout)
    N, M = 8, sum(counts)
    X = [osp.synth_deltas(11, N, i, M) for i in range(2)]
    part = osp.Partition(counts)
    for name in args.variants.split(","):
        kw = variant(name)
        grp = osp.OspGroup(part, N, [1.0 / N] * N, n_chunks=4, **kw)
        grp.set_budget(int(0.5 * M * 4))
        st = timed(lambda i: grp.step(X[i % 2]))
        s1 = timed(lambda i: grp.stage1(X[i % 2]))
        s2 = timed(lambda i: grp.stage2_all(X[i % 2]))
        gbs = 4.0 * M * (2 * N + 2) / (s1 * 1e-3) / 1e9
        print(f"{layout:9s} {name:9s} {tag} step {st:.4f} ms  stage1 {s1:.4f} ms ({gbs:.0f} GB/s at u=0)  "
              f"stage2 {s2:.4f} ms", flush=True)
        del grp
        torch.cuda.synchronize()
