"""Where do two golden dumps (oracle/ref_driver golden) differ? Element counts,
layers and values of every differing .bin file."""
import glob
import os
import sys

import numpy as np

a, b = sys.argv[1], sys.argv[2]
layers = np.fromfile(os.path.join(a, "layers.bin"), dtype=np.uint64)
offs = np.concatenate([[0], np.cumsum(layers)]).astype(np.int64)
for fa in sorted(glob.glob(os.path.join(a, "*.bin"))):
    fb = os.path.join(b, os.path.basename(fa))
    x, y = np.fromfile(fa, dtype=np.uint8), np.fromfile(fb, dtype=np.uint8)
    if x.size == y.size and np.array_equal(x, y):
        continue
    name = os.path.basename(fa)
    print(f"== {name}: sizes {x.size} {y.size}")
    if x.size != y.size or x.size % 4:
        continue
    xf, yf = x.view(np.float32), y.view(np.float32)
    M = int(offs[-1])
    d = np.flatnonzero(xf.view(np.uint32) != yf.view(np.uint32))
    print(f"   {d.size} differing floats of {xf.size}")
    for i in d[:12]:
        e = int(i % M) if xf.size % M == 0 else int(i)
        l = int(np.searchsorted(offs, e, side="right") - 1)
        print(f"   idx {i} (row {i // M if xf.size % M == 0 else 0}, layer {l}, elem {e - offs[l]}): "
              f"ref {xf[i]!r} ({xf.view(np.uint32)[i]:#010x}) dev {yf[i]!r} ({yf.view(np.uint32)[i]:#010x})")
    if d.size:
        ls = np.searchsorted(offs, d % M if xf.size % M == 0 else d, side="right") - 1
        u, c = np.unique(ls, return_counts=True)
        print("   per layer:", dict(zip(u.tolist(), c.tolist())))
