"""Streaming shard kernel diagnostics (torchrun, one rank per GPU): ms/step and
the producer counters of osp_shard_debug_counters (OSP_SS_DEBUG=1 is set here).
Usage: torchrun --nproc-per-node P tools/shard_diag.py [layout] [steps]"""
import ctypes
import os
import sys

os.environ.setdefault("OSP_SS_DEBUG", "1")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

sys.path.insert(0, ".")
from paper_2306_16926_b200 import layouts, osp  # noqa: E402
from paper_2306_16926_b200.osp import lib  # noqa: E402
from paper_2306_16926_b200.dist import ShardGroup  # noqa: E402

layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
counts = layouts.get(layout)
M = sum(counts)
sh = ShardGroup(osp.Partition(counts), 8, None, n_chunks=4, tile_elems=int(os.environ.get("TILE", "0")))
sh.connect_via()
for b in range(2):
    sh.fill_synth(11, b, b)
sh.set_budget(int(0.5 * M * 4))
for k in range(3):
    sh.step(k % 2)
torch.cuda.synchronize()
f = lib().osp_shard_debug_counters
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]
base = (ctypes.c_ulonglong * 96)()
f(sh._h, base)
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(K):
    sh.step(k % 2)
b.record()
torch.cuda.synchronize()
sh.check()
out = (ctypes.c_ulonglong * 96)()
f(sh._h, out)
d = [out[i] - base[i] for i in range(96)]
ms = a.elapsed_time(b) / K
prof = sh.profile(0)
mhz = 1965.0
for r in range(world):
    if r == rank:
        print(f"rank {rank} mode={os.environ.get('OSP_SS_MODE', '1')} tile={sh.local.geometry()['tile_elems']} ms/step {ms:.4f} phases "
              f"{ {k: round(v, 4) for k, v in prof.items()} }", flush=True)
        for st in range(2):
            for role in range(3):
                c = d[st * 48 + role * 16: st * 48 + role * 16 + 16]
                grid = c[12] // K
                if grid == 0:
                    continue
                us = lambda cyc: cyc / K / mhz / grid  # noqa: E731  per CTA, us per step
                print(f"  stage{st + 1} role {'ABC'[role]} ({grid} CTAs): items/step A {c[3] / K:.0f} "
                      f"B {c[4] / K:.0f} C {c[5] / K:.0f}; per CTA us: producer {us(c[6]):.1f} "
                      f"empty-wait {us(c[0]):.1f} B-wait {us(c[1]):.1f} x-wait {us(c[2]):.1f}; "
                      f"warp0 full-wait {us(c[8]):.1f} proc {us(c[9] + c[10] + c[11]):.1f}; last launch: "
                      f"max producer {out[st * 48 + role * 16 + 13] / mhz:.1f} us, start skew "
                      f"{(out[st * 48 + role * 16 + 14] - out[st * 48 + role * 16 + 15]) / 1e3:.1f} us", flush=True)
    dist.barrier()
sh.close()
dist.destroy_process_group()
