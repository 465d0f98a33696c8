"""Python restatement of the reference learner's forward_backward
(learner.cpp:199-367) for the device gradient producer's tests.

TEST INFRASTRUCTURE ONLY (tests/ imports it; the product never does). Pure
Python floats are IEEE doubles and every operation rounds on its own (no FMA),
and math.exp / math.log / math.tanh call the same host libm as the reference
build, so this restatement is bit-identical to the reference on the same
inputs (pinned against oracle/_ref/ref_fb dumps, tests/golden/learner/).
"""
from __future__ import annotations

import math

import numpy as np


def layer_views(widths, params):
    """learner.cpp:204-218: (W [out][in], b [out]) per linear layer, W then b."""
    views, at = [], 0
    for l in range(len(widths) - 1):
        n_in, n_out = widths[l], widths[l + 1]
        W = params[at:at + n_in * n_out].reshape(n_out, n_in)
        b = params[at + n_in * n_out:at + n_in * n_out + n_out]
        views.append((W, b, at))
        at += n_in * n_out + n_out
    if at != len(params):
        raise ValueError("params do not match the mlp partition")
    return views


def act_forward(act, z):  # learner.cpp:220-222
    return (z if z > 0 else 0.0) if act == "relu" else math.tanh(z)


def act_backward(act, z, a):  # learner.cpp:224-226
    return (1.0 if z > 0 else 0.0) if act == "relu" else 1.0 - a * a


def sample_loss(loss, z, label, want_dz):  # learner.cpp:231-260
    k = len(z)
    if loss == "ce":
        zmax = max(z)
        s = 0.0
        for v in z:
            s += math.exp(v - zmax)
        logsum = math.log(s) + zmax
        if label >= k:
            raise ValueError("label exceeds output width")
        val = logsum - z[label]
        dz = [math.exp(z[c] - logsum) - (1.0 if c == label else 0.0) for c in range(k)] if want_dz else None
        return val, dz
    val, dz = 0.0, [0.0] * k
    for c in range(k):
        target = float(label) if k == 1 else (1.0 if label == c else 0.0)
        diff = z[c] - target
        val += diff * diff
        dz[c] = 2.0 * diff
    return val, dz


def forward_backward(widths, act, loss, feats, labels, params, batch):
    """learner.cpp:299-367 -> (float32 gradient vector, mean loss)."""
    params = np.asarray(params, dtype=np.float32)
    views = layer_views(widths, params)
    depth = len(views)
    Wd = [[[float(x) for x in row] for row in W] for (W, _, _) in views]
    bd = [[float(x) for x in b] for (_, b, _) in views]
    grad_acc = [0.0] * len(params)
    total = 0.0
    for bi in batch:
        acts = [[float(x) for x in feats[bi]]]
        pre = [None]
        for l in range(depth):
            n_out, n_in = len(Wd[l]), len(Wd[l][0])
            zl, al = [], []
            for o in range(n_out):
                z = bd[l][o]
                row = Wd[l][o]
                for i in range(n_in):
                    z += row[i] * acts[l][i]
                zl.append(z)
                al.append(act_forward(act, z) if l + 1 < depth else z)
            pre.append(zl)
            acts.append(al)
        val, delta_top = sample_loss(loss, acts[depth], int(labels[bi]), True)
        total += val
        delta = [None] * (depth + 1)
        delta[depth] = delta_top
        for l in range(depth - 1, -1, -1):
            n_out, n_in = len(Wd[l]), len(Wd[l][0])
            at = views[l][2]
            if l > 0:
                delta[l] = [0.0] * n_in
            for o in range(n_out):
                dz = delta[l + 1][o]
                grad_acc[at + n_in * n_out + o] += dz
                row = Wd[l][o]
                for i in range(n_in):
                    grad_acc[at + o * n_in + i] += dz * acts[l][i]
                    if l > 0:
                        delta[l][i] += dz * row[i]
            if l > 0:
                for i in range(n_in):
                    delta[l][i] *= act_backward(act, pre[l][i], acts[l][i])
    mean = total / float(len(batch))
    inv = 1.0 / float(len(batch))
    grad = np.array([g * inv for g in grad_acc], dtype=np.float64).astype(np.float32)
    return grad, mean


def load_case(path_base):
    """A tests/golden/learner/<case>.npz fixture as a dict."""
    z = np.load(path_base if path_base.endswith(".npz") else path_base + ".npz")
    return {k: z[k] for k in z.files}
