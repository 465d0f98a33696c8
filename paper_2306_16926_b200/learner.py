"""The gradient producer on the other side of the sync path:
the reference learner's MLP forward_backward (learner.hpp:63-64,
learner.cpp:299-367) for every worker at once, on the device (osp_mlp_*).

    mlp = Mlp([8, 32, 4], features, labels)           # device-resident dataset
    grads, losses = mlp.grad(group.worker_params, batch)  # batch: [N, B] int32
    group.step(grads)                                  # group built with sgd_lr > 0
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from ._capi import c_void_p
from .osp import InvalidArgument, ShapeError, _check, _Handle, _ptr, _stream, lib

RELU, TANH = 0, 1
CE, MSE = 0, 1
_ACT = {"relu": RELU, "tanh": TANH}
_LOSS = {"ce": CE, "softmax_cross_entropy": CE, "mse": MSE}


class Mlp:
    """MlpSpec + Dataset of the reference learner, on the device."""

    def __init__(self, widths: Sequence[int], features: torch.Tensor, labels: torch.Tensor,
                 activation: str = "relu", loss: str = "ce"):
        if not (features.is_cuda and features.dtype == torch.float32 and features.is_contiguous()
                and features.dim() == 2):
            raise InvalidArgument("features must be a contiguous [n, d] float32 CUDA tensor")
        if not (labels.is_cuda and labels.dtype == torch.int32 and labels.is_contiguous()
                and labels.numel() == features.shape[0]):
            raise InvalidArgument("labels must be a contiguous [n] int32 CUDA tensor")
        if len(widths) >= 1 and features.shape[1] != widths[0]:
            raise ShapeError("dataset width differs from the input width")
        self.widths = [int(w) for w in widths]
        self._feats, self._labels = features, labels  # borrowed by the handle
        w = (ctypes.c_int32 * len(self.widths))(*self.widths)
        h = c_void_p()
        _check(lib().osp_mlp_create(w, len(self.widths), _ACT[activation], _LOSS[loss],
                                    _ptr(features), _ptr(labels), features.shape[0],
                                    ctypes.byref(h)))
        self._h = h
        self._hnd = _Handle(h, "osp_mlp_destroy")
        self.n_params = int(lib().osp_mlp_num_params(h))

    def grad(self, params: torch.Tensor, batch: torch.Tensor, out: Optional[torch.Tensor] = None,
             losses: Optional[torch.Tensor] = None, check: bool = True, stream=None):
        """Gradients of every worker's mean batch loss. params: [N, >= n_params]
        float32 rows (unit inner stride, any row stride); batch: [N, B] int32 row
        indices. Returns (grads [N, n_params] float32, losses [N] float64)."""
        if not (params.is_cuda and params.dtype == torch.float32 and params.dim() == 2
                and params.stride(1) == 1 and params.shape[1] >= self.n_params):
            raise ShapeError("params must be [N, >= n_params] float32 rows with unit stride")
        N = params.shape[0]
        if not (batch.is_cuda and batch.dtype == torch.int32 and batch.is_contiguous()
                and batch.dim() == 2 and batch.shape[0] == N):
            raise ShapeError("batch must be a contiguous [N, B] int32 CUDA tensor")
        if out is None:
            out = torch.empty((N, self.n_params), dtype=torch.float32, device=params.device)
        if not (out.dtype == torch.float32 and out.dim() == 2 and out.shape[0] == N
                and out.stride(1) == 1 and out.shape[1] >= self.n_params):
            raise ShapeError("out must be [N, >= n_params] float32 rows with unit stride")
        if losses is None:
            losses = torch.empty(N, dtype=torch.float64, device=params.device)
        _check(lib().osp_mlp_grad(self._h, _ptr(params), params.stride(0), N, _ptr(batch),
                                  batch.shape[1], _ptr(out), out.stride(0), _ptr(losses),
                                  _stream(stream)))
        if check:
            self.check(stream)
        return out, losses

    def check(self, stream=None):
        """NumericError / ShapeError flagged by earlier asynchronous calls."""
        _check(lib().osp_mlp_check(self._h, _stream(stream)))

    def close(self):
        self._hnd.close()
