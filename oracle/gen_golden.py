"""Generate tests/golden/*.npz from the UNMODIFIED reference engine.

Runs oracle/_ref/ref_driver (the reference pslab OspWorker/OspServer compiled
from /root/reference/proj/src by `make -C oracle ref`) on small seeded configs
and packs every per-iteration artefact into one compressed .npz per config.
Those fixtures pin the C restatement (tests/test_oracle.py) and are the
golden vectors of the GPU parity tests. Test infrastructure only; needs
/root/reference, so it runs in the build container, never on the GPU box.

    python oracle/gen_golden.py            # regenerate all fixtures
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DRIVER = os.path.join(HERE, "_ref", "ref_driver")
OUT = os.path.join(REPO, "tests", "golden")

# name -> driver flags. Small enough to stay a few hundred KB in total.
CONFIGS = {
    # ragged layers, unequal weights whose sum is not exactly 1.0 (exercises the division)
    "ragged_w3": dict(layers=[3, 5, 7, 1, 12, 4, 9, 16, 2, 6], workers=3, weights=[0.2, 0.5, 0.35],
                      p0="random:5", budget=90, chunks=3, iters=5, seed=21),
    # the small-MLP partition (checks.cpp:40-56) with synth deltas, half-model budget
    "mlp_half": dict(layers=[256, 32, 128, 4], workers=8, p0="random:7", budget_frac=0.5,
                     chunks=4, iters=6, seed=7),
    # synth workload as the bench runs it: P0 = 0, 8 workers, 0.5 x model, 4 chunks
    "synth_mixed": dict(layers=[1728, 64, 36, 64, 737, 128, 1, 256, 4096, 40, 512, 3, 1000, 4, 17,
                                2048, 2048, 9, 300, 64],
                        workers=8, p0="zeros", budget_frac=0.5, chunks=4, iters=5, seed=11),
    # budget 0: OSP degenerates to BSP (checks.cpp:82-124)
    "budget_zero": dict(layers=[100, 7, 300, 33, 64], workers=4, p0="random:3", budget=0,
                        chunks=4, iters=3, seed=5),
    # whole model deferred: empty barrier payload, every layer through ICS
    "budget_all": dict(layers=[100, 7, 300, 33, 64, 5, 17], workers=5, p0="random:9",
                       budget_frac=1.0, chunks=4, iters=4, seed=13),
    # bytes_per_element 1000 like the timing fixture (checks.cpp:60-78); 1 chunk
    "bpe1000": dict(layers=[250] * 10, workers=8, bpe=1000, p0="zeros", budget=2_000_000,
                    chunks=1, iters=4, seed=11),
    # more chunks than deferred layers (empty-chunk compaction)
    "many_chunks": dict(layers=[64, 64, 640, 8, 8, 1024], workers=2, p0="random:4",
                        budget_frac=0.8, chunks=9, iters=4, seed=17),
    # tuned budget (Alg. 1): 2 iterations per epoch, u_max 60% of the model
    "tuned": dict(layers=[200, 50, 400, 25, 75, 150], workers=4, p0="random:2", umax=3600,
                  ipe=2, chunks=2, iters=8, seed=3),
}


def _flags(cfg):
    args = []
    for k, v in cfg.items():
        key = {"budget_frac": "budget-frac", "chunks": "chunks", "p0": "p0"}.get(k, k)
        if isinstance(v, list):
            v = ",".join(repr(x) if isinstance(x, float) else str(x) for x in v)
        args += [f"--{key}", str(v)]
    return args


def _read(path, dtype):
    return np.fromfile(path, dtype=dtype) if os.path.exists(path) else np.zeros(0, dtype)


def generate(name, cfg):
    with tempfile.TemporaryDirectory() as tmp:
        cmd = [DRIVER, "golden", "--out", tmp] + _flags(cfg)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"{name}: {res.stderr}")
        layers = _read(os.path.join(tmp, "layers.bin"), np.uint64)
        weights = _read(os.path.join(tmp, "weights.bin"), np.float64)
        p0 = _read(os.path.join(tmp, "p0.bin"), np.float32)
        N = len(weights)
        M = int(layers.sum())
        data = dict(layers=layers, weights=weights, p0=p0,
                    meta=np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8))
        for it in range(cfg["iters"]):
            p = os.path.join(tmp, f"it{it:03d}_")
            small = N * M <= 12000
            if small:  # larger configs regenerate deltas from the seed (synth generator)
                data[f"it{it}_deltas"] = _read(p + "deltas.bin", np.float32).reshape(N, M)
            data[f"it{it}_gib_in"] = _read(p + "gib_in.bin", np.uint8)
            data[f"it{it}_order_in"] = _read(p + "order_in.bin", np.int32)
            data[f"it{it}_chunks"] = _read(p + "chunks.bin", np.int32)
            data[f"it{it}_rs_ids"] = _read(p + "rs_ids.bin", np.int32)
            st1 = _read(p + "params_stage1.bin", np.float32).reshape(N, M)
            fin = _read(p + "params_final.bin", np.float32).reshape(N, M)
            glob = _read(p + "global.bin", np.float32)
            if small:
                data[f"it{it}_params_stage1"] = st1
            else:  # keep worker 0 and the last worker
                data[f"it{it}_params_stage1_w0"] = st1[0]
                data[f"it{it}_params_stage1_wlast"] = st1[-1]
            # conservation: after the corrections every worker equals the global vector
            eq = all(np.array_equal(fin[w].view(np.uint32), glob.view(np.uint32)) for w in range(N))
            data[f"it{it}_final_eq_global"] = np.array([1 if eq else 0], dtype=np.uint8)
            if not eq:
                data[f"it{it}_params_final"] = fin
            data[f"it{it}_global"] = glob
            data[f"it{it}_agg"] = _read(p + "agg.bin", np.float32)
            data[f"it{it}_scores"] = _read(p + "scores.bin", np.float64)
            data[f"it{it}_gib_out"] = _read(p + "gib_out.bin", np.uint8)
            data[f"it{it}_order_out"] = _read(p + "order_out.bin", np.int32)
            data[f"it{it}_budget"] = _read(p + "budget.bin", np.uint64)
        os.makedirs(OUT, exist_ok=True)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **data)
        return M, N


def main(argv):
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    names = argv[1:] or list(CONFIGS)
    for name in names:
        M, N = generate(name, CONFIGS[name])
        print(f"{name}: M={M} N={N}")


if __name__ == "__main__":
    main(sys.argv)
