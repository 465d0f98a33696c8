"""Closed-loop SGU budget from measured compute and link rates.

The reference derives the deferred-byte budget per epoch from the measured
compute time (runner.cpp:364-376, `umax_measured`): once an epoch's compute
phases are all measured, U_max = compute_umax(b, mean t_c, N, model bytes)
(tuning.cpp:8-21, Eq. 5) is handed to the server (OspServer::set_umax); at the
resolution of the epoch's last iteration the server folds the epoch's mean
loss into tune_sgu (protocol.cpp:396-405, tuning.cpp:23-48), and every
resolution builds the next GIB with budget_for_epoch(epoch(i + 1))
(protocol.cpp:413, 434-439: 0 up to epoch 1, then the tuned value).

Here t_c is the CUDA-event time of the (synthetic) compute phase and b the
measured rate of the synchronization traffic (bytes per second on the link
that carries it: NVLink per GPU for the sharded path, HBM for one GPU), both
taken on the device; the arithmetic is the library's osp_compute_umax /
osp_tune_sgu (host scalar code behind the C-ABI).
"""
from __future__ import annotations

from typing import Dict, List

from . import osp


class BudgetLoop:
    """Per-epoch Eq. 5 + Alg. 1 budget driven by measured t_c and link rate."""

    def __init__(self, iterations_per_epoch: int, n_workers: int, model_bytes: int,
                 loss_rate: float = 0.0, eq5_literal: bool = False):
        if iterations_per_epoch < 1:
            raise osp.ConfigError("iterations_per_epoch must be at least 1")
        self.ipe = iterations_per_epoch
        self.n_workers = n_workers
        self.model_bytes = model_bytes
        self.loss_rate = loss_rate
        self.eq5_literal = eq5_literal
        self.sched = osp.SguSchedule(0)
        self._tc: Dict[int, List[float]] = {}
        self._bw: Dict[int, List[float]] = {}
        self._loss: Dict[int, List[float]] = {}
        self.epoch_budget: Dict[int, int] = {}
        self.umax_history: List[dict] = []

    def epoch_of(self, iteration: int) -> int:
        """epoch_of_iteration (protocol.hpp): 1-based."""
        return iteration // self.ipe + 1

    def record(self, iteration: int, t_c_s: float, link_bytes: float, link_s: float,
               loss: float):
        """One iteration's measurements: compute time (s), the bytes the
        synchronization moved and the time it took, and the loss. Every one of
        the N co-resident workers reports the same compute time and loss, so
        they are accumulated N times, in the reference's arrival order, and the
        means are sum / count as the reference takes them (a last-bit
        difference would move tune_sgu's floor)."""
        e = self.epoch_of(iteration)
        self._tc.setdefault(e, []).extend([t_c_s] * self.n_workers)
        if link_s > 0 and link_bytes > 0:
            self._bw.setdefault(e, []).append(link_bytes / link_s)
        self._loss.setdefault(e, []).extend([loss] * self.n_workers)
        if len(self._tc[e]) == self.ipe * self.n_workers:  # epoch measured (runner.cpp:364-376)
            tcs = self._tc.pop(e)
            tc = 0.0
            for v in tcs:
                tc += v
            tc /= len(tcs)
            bws = self._bw.pop(e, [])
            bw = sum(bws) / len(bws) if bws else 0.0
            if bw > 0:
                self.sched.u_max = osp.compute_umax(bw, tc, self.n_workers, self.model_bytes,
                                                    loss_rate=self.loss_rate,
                                                    eq5_literal=self.eq5_literal)
            self.umax_history.append({"epoch": e, "t_c_s": tc, "bandwidth_Bps": bw,
                                      "u_max": self.sched.u_max})

    def on_resolution(self, iteration: int):
        """check_resolution's epoch-boundary fold (protocol.cpp:396-405)."""
        if (iteration + 1) % self.ipe == 0:
            e = self.epoch_of(iteration)
            losses = self._loss.pop(e, [])
            if losses:
                total = 0.0
                for v in losses:
                    total += v
                self.epoch_budget[e + 1] = self.sched.tune(e, total / len(losses))

    def budget_for_epoch(self, epoch: int) -> int:
        """protocol.cpp:434-439 (no fixed budget)."""
        if epoch <= 1:
            return 0
        return self.epoch_budget.get(epoch, 0)

    def budget_for_next(self, iteration: int) -> int:
        """The budget the resolution of `iteration` builds the next GIB with."""
        return self.budget_for_epoch(self.epoch_of(iteration + 1))

    def step(self, iteration: int, t_c_s: float, link_bytes: float, link_s: float,
             loss: float) -> int:
        """record + on_resolution; returns the budget for the next GIB."""
        self.record(iteration, t_c_s, link_bytes, link_s, loss)
        self.on_resolution(iteration)
        return self.budget_for_next(iteration)


def synthetic_loss(epoch: int) -> float:
    """The reference synth workload's loss: 0.7^(epoch - 1) (runner.cpp synth)."""
    return 0.7 ** (epoch - 1)
