"""Step-time variants on one GPU (diagnostic): evented per-stage loop, plain C
step loop, CUDA-graph replay. Prints ms/step for each."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2306_16926_b200 import layouts, osp  # noqa: E402

layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = 200
counts = layouts.get(layout)
N, M = 8, sum(counts)
part = osp.Partition(counts)
grp = osp.OspGroup(part, N, [1.0 / N] * N, n_chunks=4)
X = [osp.synth_deltas(11, N, i, M) for i in range(2)]
grp.set_budget(int(0.5 * M * 4))
s = torch.cuda.current_stream()


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


def evented(i):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    x = X[i % 2]
    e[0].record()
    grp.stage1(x)
    e[1].record()
    grp.stage2_all(x)
    e[2].record()
    grp.resolve(x)


print("evented  ", round(timed(evented), 4))


def s1_evented(i):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    x = X[i % 2]
    e[0].record()
    grp.stage1(x)
    e[1].record()
    grp.stage2_all(x)
    grp.resolve(x)


print("s1-evented", round(timed(s1_evented), 4))
print("c-step   ", round(timed(lambda i: grp.step(X[i % 2])), 4))
print("3-calls  ", round(timed(lambda i: (grp.stage1(X[i % 2]), grp.stage2_all(X[i % 2]), grp.resolve(X[i % 2]))), 4))
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(s)
with torch.cuda.stream(side):
    grp.step(X[0])
    grp.step(X[1])
torch.cuda.synchronize()
with torch.cuda.graph(g):
    grp.step(X[0])
    grp.step(X[1])
torch.cuda.synchronize()
print("graph    ", round(timed(lambda i: g.replay() if i % 2 == 0 else None, 2 * K) , 4))
# stage-only timings (kernel alone, back to back)
print("stage1x  ", round(timed(lambda i: grp.stage1(X[i % 2])), 4))
print("stage2x  ", round(timed(lambda i: grp.stage2_all(X[i % 2])), 4))
print("resolvex ", round(timed(lambda i: grp.resolve(X[i % 2])), 4))
print("stats", grp.stats())
