"""Synthetic layer tables of the BASELINE.json configs.

Element counts per parameter tensor in `parameters()` order: the OSP layer
partition (one layer per tensor, as LayerPartition::make, param.cpp:8-29).
"""
from __future__ import annotations


def _resnet_bottleneck(blocks):
    counts = [64 * 3 * 7 * 7, 64, 64]
    inplanes = 64
    for stage, n in enumerate(blocks):
        width = 64 * (2 ** stage)
        out = width * 4
        for b in range(n):
            counts += [inplanes * width, width, width,
                       width * width * 9, width, width,
                       width * out, out, out]
            if b == 0:
                counts += [inplanes * out, out, out]
            inplanes = out
    counts += [2048 * 1000, 1000]
    return counts


def resnet50():
    return _resnet_bottleneck([3, 4, 6, 3])


def resnet152():
    return _resnet_bottleneck([3, 8, 36, 3])


def vgg16():
    convs = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 256),
             (256, 512), (512, 512), (512, 512), (512, 512), (512, 512), (512, 512)]
    counts = []
    for cin, cout in convs:
        counts += [cin * cout * 9, cout]
    counts += [512 * 7 * 7 * 4096, 4096, 4096 * 4096, 4096, 4096 * 1000, 1000]
    return counts


def llama1b():
    h, kv, ff, vocab = 2048, 512, 8192, 128256
    per_layer = [h, h * h, kv * h, kv * h, h * h, h, ff * h, ff * h, h * ff]
    return [vocab * h] + per_layer * 16 + [h]


def small_mlp(widths=(8, 32, 4)):
    """learner.cpp mlp_partition: per layer W (out*in) then b (out)."""
    counts = []
    for i in range(len(widths) - 1):
        counts += [widths[i + 1] * widths[i], widths[i + 1]]
    return counts


LAYOUTS = {
    "resnet50": resnet50,
    "resnet152": resnet152,
    "vgg16": vgg16,
    "llama1b": llama1b,
    "mlp": small_mlp,
    # the accuracy check's wider MLP (checks.cpp:346): [16, 64, 64, 4]
    "mlp_acc": lambda: small_mlp((16, 64, 64, 4)),
}


def get(name: str):
    if name in LAYOUTS:
        return LAYOUTS[name]()
    return [int(x) for x in name.split(",") if x]
