"""CPU: the learner restatement (oracle/learner_oracle.py) is bit-identical to
the unmodified reference learner (pslab::forward_backward, learner.cpp:299-367)
on the golden dumps of oracle/_ref/ref_fb (tests/golden/gen_learner_golden.py):
gradients, mean losses, for relu / tanh and softmax CE / MSE, a 1-wide output."""
import glob
import os

import numpy as np
import pytest

from oracle import learner_oracle as lo

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "learner", "*.npz")))


def test_goldens_present():
    assert len(GOLD) >= 6


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-4] for p in GOLD])
def test_oracle_matches_reference_learner(path):
    c = lo.load_case(path)
    for w in range(len(c["param"])):
        g, loss = lo.forward_backward([int(x) for x in c["widths"]], str(c["act"]), str(c["loss"]),
                                      c["feat"], c["label"], c["param"][w], [int(i) for i in c["batch"][w]])
        assert np.array_equal(g.view(np.uint32), c["grad"][w].view(np.uint32)), f"worker {w}"
        assert loss == c["loss_mean"][w], f"worker {w}"
