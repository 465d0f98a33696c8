"""B200: the device gradient producer (kernels/learner.cu, osp_mlp_*) against the
reference learner's dumps (tests/golden/learner/, pinned by
tests/test_learner_oracle.py) and the restatement, and one end-to-end training
iteration: device gradients of every worker row -> the OSP step with the fused
sgd_delta, bit-exact against the oracle fed with the reference learner's math.

Tolerance: relu + MSE is exact arithmetic, so gradients and losses must be
bit-identical. tanh and the softmax's exp / log come from CUDA's libm instead
of the host's (each within an ulp or two), so there the float gradients may
differ by at most 1 ulp and the fp64 losses by 1e-13 relative."""
import glob
import os

import numpy as np
import pytest
import torch

from oracle import learner_oracle as lo
from oracle import oracle

pytestmark = pytest.mark.gpu

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "learner", "*.npz")))


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2306_16926_b200 import learner, osp
    return learner, osp


def ulp_diff(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-4] for p in GOLD])
def test_grad_vs_reference_learner(mods, path):
    learner, _ = mods
    c = lo.load_case(path)
    exact = str(c["act"]) == "relu" and str(c["loss"]) == "mse"
    mlp = learner.Mlp([int(x) for x in c["widths"]], torch.as_tensor(c["feat"]).cuda(),
                      torch.as_tensor(c["label"]).cuda(), str(c["act"]), str(c["loss"]))
    g, loss = mlp.grad(torch.as_tensor(c["param"]).cuda(), torch.as_tensor(c["batch"]).cuda())
    g, loss = g.cpu().numpy(), loss.cpu().numpy()
    if exact:
        assert np.array_equal(g.view(np.uint32), c["grad"].view(np.uint32))
        assert np.array_equal(loss, c["loss_mean"])
    else:
        assert ulp_diff(g, c["grad"]).max() <= 1
        np.testing.assert_allclose(loss, c["loss_mean"], rtol=1e-13, atol=0)


def test_grad_row_strides_and_worker_count(mods):
    """Parameter rows with a padded stride (the group's worker rows), an output
    with its own stride, 8 workers sharing the dataset."""
    learner, _ = mods
    c = lo.load_case(GOLD[[os.path.basename(p) for p in GOLD].index("mlp_relu_mse.npz")])
    M = c["param"].shape[1]
    params = torch.zeros((8, M + 12), dtype=torch.float32, device="cuda")
    batch = np.concatenate([c["batch"], c["batch"]])
    for w in range(8):
        params[w, :M] = torch.as_tensor(c["param"][w % 4])
    out = torch.full((8, M + 4), 7.0, dtype=torch.float32, device="cuda")
    mlp = learner.Mlp([8, 32, 4], torch.as_tensor(c["feat"]).cuda(), torch.as_tensor(c["label"]).cuda(),
                      "relu", "mse")
    mlp.grad(params[:, :M + 12], torch.as_tensor(batch).cuda(), out=out)
    o = out.cpu().numpy()
    for w in range(8):
        assert np.array_equal(o[w, :M].view(np.uint32), c["grad"][w % 4].view(np.uint32))
        assert np.all(o[w, M:] == 7.0)


def test_errors_as_the_reference_throws(mods):
    learner, osp = mods
    feats = torch.zeros((10, 3), dtype=torch.float32, device="cuda")
    labels = torch.zeros(10, dtype=torch.int32, device="cuda")
    with pytest.raises(osp.ConfigError):
        learner.Mlp([3], feats, labels)
    with pytest.raises(osp.ConfigError):
        learner.Mlp([3, 0, 2], feats, labels)
    mlp = learner.Mlp([3, 4, 2], feats, labels)
    P = torch.zeros((1, mlp.n_params), dtype=torch.float32, device="cuda")
    with pytest.raises(osp.ShapeError):  # batch row out of range (check_batch)
        mlp.grad(P, torch.tensor([[0, 10]], dtype=torch.int32, device="cuda"))
    labels[3] = 5
    with pytest.raises(osp.ShapeError):  # label exceeds output width
        mlp.grad(P, torch.tensor([[3]], dtype=torch.int32, device="cuda"))
    # a NaN output bias (W0 12, b0 4, W1 8, then b1): the loss is not finite
    # (a NaN in a hidden pre-activation would not be: relu maps it to 0, as in
    # the reference's z > 0 ? z : 0.0)
    P[0, 24] = float("nan")
    with pytest.raises(osp.NumericError):
        mlp.grad(P, torch.tensor([[1]], dtype=torch.int32, device="cuda"))
    # the flag is cleared once reported
    P[0, 24] = 0.0
    mlp.grad(P, torch.tensor([[1]], dtype=torch.int32, device="cuda"))


def test_training_iterations_end_to_end(mods):
    """Config #1's loop on the device: every worker's gradient from its own row
    (learner.cpp:299-367), then the OSP step with the fused sgd_delta
    (learner.cpp:391-398): G, every row and the GIB bit-exact against the oracle
    fed with the restated learner, for three iterations (relu + MSE)."""
    learner, osp = mods
    c = lo.load_case(GOLD[[os.path.basename(p) for p in GOLD].index("mlp_relu_mse.npz")])
    widths = [8, 32, 4]
    counts = np.array([w for l in range(2) for w in (widths[l] * widths[l + 1], widths[l + 1])],
                      np.uint64)
    M, N, lr, nc = int(counts.sum()), 4, 0.05, 2
    budget = int(0.4 * M * 4)
    G = c["param"][0].copy()
    P = np.tile(G, (N, 1))
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [0.25] * N, n_chunks=nc, init_params=torch.as_tensor(G).cuda(),
                       sgd_lr=lr)
    mlp = learner.Mlp(widths, torch.as_tensor(c["feat"]).cuda(), torch.as_tensor(c["label"]).cuda(),
                      "relu", "mse")
    rng = np.random.default_rng(3)
    flags, order = np.zeros(len(counts), np.uint8), np.zeros(0, np.int32)
    for it in range(3):
        batch = rng.integers(0, c["feat"].shape[0], (N, 32)).astype(np.int32)
        grads, _ = mlp.grad(grp.worker_params, torch.as_tensor(batch).cuda())
        host_g = np.stack([lo.forward_backward(widths, "relu", "mse", c["feat"], c["label"], P[w],
                                               list(batch[w]))[0] for w in range(N)])
        assert np.array_equal(grads.cpu().numpy().view(np.uint32), host_g.view(np.uint32)), f"grads it {it}"
        deltas = np.stack([oracle.sgd_delta(host_g[w], lr) for w in range(N)])
        r = oracle.step(counts, 4, [0.25] * N, deltas, G, P, flags, order, nc, budget)
        grp.set_budget(budget)
        grp.step(grads)
        assert np.array_equal(grp.global_params.cpu().numpy().view(np.uint32), G.view(np.uint32))
        assert np.array_equal(grp.worker_params.cpu().numpy().view(np.uint32), P.view(np.uint32))
        nxt = grp.read_gib()
        assert np.array_equal(nxt["flags"], r["flags_out"]) and np.array_equal(nxt["order"], r["order_out"])
        flags, order = r["flags_out"], r["order_out"]


@pytest.mark.parametrize("widths,act,loss,B", [([5, 3], "relu", "mse", 1), ([5, 3], "tanh", "ce", 7),
                                               ([6, 9, 1], "relu", "mse", 13),
                                               ([4, 7, 5, 3], "tanh", "mse", 33),
                                               ([3, 40, 2], "relu", "ce", 64)])
def test_grad_random_specs_vs_restatement(mods, widths, act, loss, B):
    """Depth 1 (no hidden layer) to 3, batches from 1 to 64 with repeated rows,
    against the reference-pinned restatement (oracle/learner_oracle.py)."""
    learner, _ = mods
    rng = np.random.default_rng(sum(widths) * 7 + B)
    n, k = 50, widths[-1]
    feats = rng.normal(size=(n, widths[0])).astype(np.float32)
    labels = rng.integers(0, max(k, 2) if k > 1 else 3, n).astype(np.int32)
    M = sum(widths[l] * widths[l + 1] + widths[l + 1] for l in range(len(widths) - 1))
    N = 3
    params = (rng.normal(size=(N, M)) * 0.5).astype(np.float32)
    batch = rng.integers(0, n, (N, B)).astype(np.int32)
    mlp = learner.Mlp(widths, torch.as_tensor(feats).cuda(), torch.as_tensor(labels).cuda(), act, loss)
    g, lv = mlp.grad(torch.as_tensor(params).cuda(), torch.as_tensor(batch).cuda())
    g, lv = g.cpu().numpy(), lv.cpu().numpy()
    for w in range(N):
        go, lo_ = lo.forward_backward(widths, act, loss, feats, labels, params[w], list(batch[w]))
        if act == "relu" and loss == "mse":
            assert np.array_equal(g[w].view(np.uint32), go.view(np.uint32)), f"worker {w}"
            assert lv[w] == lo_
        else:
            assert ulp_diff(g[w], go).max() <= 1, f"worker {w}"
            np.testing.assert_allclose(lv[w], lo_, rtol=1e-13, atol=0)
