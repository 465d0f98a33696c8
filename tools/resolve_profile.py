import ctypes, sys
sys.path.insert(0, ".")
import torch
from paper_2306_16926_b200 import layouts, osp
from paper_2306_16926_b200.osp import lib
f = lib().osp_debug_resolve_profile
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 32)()
for name in ["resnet50", "resnet152", "vgg16"]:
    counts = layouts.get(name); M = sum(counts); N = 8
    grp = osp.OspGroup(osp.Partition(counts), N, n_chunks=4)
    X = [osp.synth_deltas(11, N, i, M) for i in range(2)]
    grp.set_budget(int(0.5 * M * 4))
    for k in range(5): grp.step(X[k % 2])
    torch.cuda.synchronize(); f(buf, 1)
    for k in range(50): grp.step(X[k % 2])
    torch.cuda.synchronize(); f(buf, 1)
    n = buf[16]
    print(name, "L", len(counts), "launches", n, "us from first block start:",
          {i: round(buf[16 + i] / n / 1e3, 2) for i in range(1, 16) if buf[16 + i]}, flush=True)
    del grp
