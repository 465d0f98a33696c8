"""Shared test helpers: golden fixture loader (tests/golden/*.npz)."""
import glob
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")

def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


class Golden:
    """One reference-engine dump (oracle/gen_golden.py)."""

    def __init__(self, name):
        self.name = name
        self.d = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        self.cfg = json.loads(bytes(self.d["meta"]).decode())
        self.counts = self.d["layers"].astype(np.uint64)
        self.weights = self.d["weights"]
        self.p0 = self.d["p0"]
        self.N = len(self.weights)
        self.M = int(self.counts.sum())
        self.L = len(self.counts)
        self.iters = self.cfg["iters"]
        self.bpe = int(self.cfg.get("bpe", 4))
        self.n_chunks = int(self.cfg["chunks"])
        self.seed = int(self.cfg["seed"])

    def get(self, it, key, default=None):
        k = f"it{it}_{key}"
        return self.d[k] if k in self.d else default

    def deltas(self, it):
        d = self.get(it, "deltas")
        if d is not None:
            return d
        from oracle import oracle
        return np.stack([oracle.synth_delta(self.seed, w, it, self.M) for w in range(self.N)])

    @staticmethod
    def decode_chunks(arr):
        arr = list(arr)
        n = arr[0]
        out, at = [], 1
        for _ in range(n):
            c = arr[at]
            out.append(sorted(arr[at + 1: at + 1 + c]))
            at += 1 + c
        return out
