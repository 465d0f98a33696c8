"""Build tests/golden/learner/*.npz from the UNMODIFIED reference learner
(oracle/_ref/ref_fb: pslab::forward_backward on pslab's own synthetic dataset
and parameter init). Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/gen_learner_golden.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "learner")


def main():
    drv = os.path.join(REPO, "oracle", "_ref", "ref_fb")
    if not os.path.exists(drv):
        sys.exit("oracle/_ref/ref_fb missing: make -C oracle ref")
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([drv, tmp], check=True)
        for meta in sorted(f for f in os.listdir(tmp) if f.endswith(".meta")):
            name = meta[:-5]
            lines = open(os.path.join(tmp, meta)).read().split()
            widths = np.array([int(x) for x in lines[0].split(",")], np.int32)
            act, loss = lines[1], lines[2]
            n, d, workers, batch = (int(x) for x in lines[3:7])
            rd = lambda ext, dt: np.fromfile(os.path.join(tmp, f"{name}.{ext}"), dtype=dt)  # noqa: E731
            M = int(sum(widths[l] * widths[l + 1] + widths[l + 1] for l in range(len(widths) - 1)))
            np.savez_compressed(
                os.path.join(OUT, name + ".npz"), widths=widths, act=np.array(act), loss=np.array(loss),
                feat=rd("feat.f32", np.float32).reshape(n, d), label=rd("label.i32", np.int32),
                param=rd("param.f32", np.float32).reshape(workers, M),
                batch=rd("batch.i32", np.int32).reshape(workers, batch),
                grad=rd("grad.f32", np.float32).reshape(workers, M),
                loss_mean=rd("loss.f64", np.float64))
            print("wrote", name)


if __name__ == "__main__":
    main()
