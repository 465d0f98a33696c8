"""Stage-2 overlap with the next iteration's compute (the point of OSP).

Timeline per iteration i (two CUDA streams, event-ordered, no host sync):

  main:  [wait resolve(i-1)] stage1(i) --ev_s1--> compute(i+1) --ev_c-->
  side:                      [wait ev_s1] stage2(i) + resolve(i) --ev_r-->

Stage 1 of i+1 waits for the resolution of i (the reference gates barrier i+1
on it, protocol.cpp:365-366), so the only concurrency is the ICS
synchronization of i against the compute of i+1. Exposed stage-2 time of
iteration i = max(0, t(ev_r) - t(ev_c)). The synthetic compute is a bf16 GEMM
loop (tensor cores) of about t_c ms; it reads nothing of ours, matching the
reference's rule that corrections landing mid-compute only affect the next
iteration (runner.cpp:386-389).
"""
from __future__ import annotations

import torch


class SyntheticCompute:
    """Stand-in for a worker's forward/backward: bf16 GEMMs for about `ms`."""

    def __init__(self, ms: float, n: int = 4096):
        self.a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
        self.b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
        self.c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            torch.matmul(self.a, self.b, out=self.c)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            torch.matmul(self.a, self.b, out=self.c)
        e.record()
        torch.cuda.synchronize()
        per = s.elapsed_time(e) / 10
        self.reps = max(1, round(ms / per))
        self.ms = self.reps * per

    def __call__(self):
        for _ in range(self.reps):
            torch.matmul(self.a, self.b, out=self.c)


def run(stage1, stage2_resolve, compute, K: int, W: int):
    """Overlapped and serial timings. stage1(i) / stage2_resolve(i) enqueue on the
    current stream. Returns dict of per-iteration ms figures."""
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    T = W + K
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(T)]
    ev_c = [torch.cuda.Event(enable_timing=True) for _ in range(T)]
    ev_r = [torch.cuda.Event(enable_timing=True) for _ in range(T)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    for i in range(T):
        if i == W:
            start.record(main)
        if i > 0:
            main.wait_event(ev_r[i - 1])
        stage1(i)
        ev_s1[i].record(main)
        compute()
        ev_c[i].record(main)
        side.wait_event(ev_s1[i])
        with torch.cuda.stream(side):
            stage2_resolve(i)
            ev_r[i].record(side)
    main.wait_event(ev_r[T - 1])
    end.record(main)
    torch.cuda.synchronize()
    overlapped = start.elapsed_time(end) / K
    exposed = []
    for i in range(W, T):
        t_c = start.elapsed_time(ev_c[i])
        t_r = start.elapsed_time(ev_r[i])
        exposed.append(max(0.0, t_r - t_c))
    s2 = [ev_s1[i].elapsed_time(ev_r[i]) for i in range(W, T)]

    # serial reference: stage 2 + resolve on the main stream before the compute
    s_start = torch.cuda.Event(enable_timing=True)
    s_end = torch.cuda.Event(enable_timing=True)
    for i in range(T):
        if i == W:
            s_start.record(main)
        stage1(i)
        stage2_resolve(i)
        compute()
    s_end.record(main)
    torch.cuda.synchronize()
    serial = s_start.elapsed_time(s_end) / K
    return {"t_c_ms": None, "iter_ms_overlapped": overlapped, "iter_ms_serial": serial,
            "exposed_stage2_ms_mean": sum(exposed) / K, "exposed_stage2_ms_max": max(exposed),
            "stage2_plus_resolve_ms_mean": sum(s2) / K}


def run_closed_loop(stage1, stage2_resolve, set_budget, compute, loop, link_bytes, K: int,
                    ipe: int, agree=None):
    """The overlapped schedule of run() with the SGU budget driven by the device
    measurements (budget.BudgetLoop, runner.cpp:364-376 + protocol.cpp:396-405):
    at every epoch end the host reads the epoch's compute-phase times and
    stage-2 link rates from CUDA events (one host sync per epoch), and the
    resolution of the epoch's last iteration builds the next GIB with the tuned
    budget (set_budget is stream-ordered before it). link_bytes(i): the bytes
    the synchronization of iteration i (stage 1 + stage 2) moves on its link;
    the link rate is those bytes over the stage-1 time plus the stage-2 +
    resolve time under the overlap. agree(list) -> list: makes an epoch's
    measurements identical on every rank (the sharded path resolves the same
    GIB on every rank, so every rank must use the same budget; the reference
    has one server). Returns the per-iteration budgets and the loop's U_max
    history."""
    from .budget import synthetic_loss
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    ev_s0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_c0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_c = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_r = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    budgets = []
    budget = loop.budget_for_epoch(1)
    set_budget(budget)
    torch.cuda.synchronize()
    for i in range(K):
        if i > 0:
            main.wait_event(ev_r[i - 1])
        ev_s0[i].record(main)
        stage1(i)
        ev_s1[i].record(main)
        ev_c0[i].record(main)
        compute()
        ev_c[i].record(main)
        side.wait_event(ev_s1[i])
        if (i + 1) % ipe == 0:
            # epoch end: this epoch's compute phases are measured (ev_c[i]
            # implies every earlier stage 2 has finished: stage 1 waited on it)
            ev_c[i].synchronize()
            e0 = i + 1 - ipe
            meas = []
            for j in range(e0, i + 1):
                t_c = ev_c0[j].elapsed_time(ev_c[j]) * 1e-3
                # sync time of the epoch's earlier iterations (j < i)
                ts = ((ev_s0[j].elapsed_time(ev_s1[j]) + ev_s1[j].elapsed_time(ev_r[j])) * 1e-3
                      if j < i else 0.0)
                meas += [t_c, link_bytes(j) if j < i else 0.0, ts]
            if agree is not None:
                meas = agree(meas)
            for n, j in enumerate(range(e0, i + 1)):
                t_c, nb, ts = meas[3 * n: 3 * n + 3]
                loop.record(j, t_c, nb, ts, synthetic_loss(loop.epoch_of(j)))
            loop.on_resolution(i)
            budget = loop.budget_for_next(i)
        with torch.cuda.stream(side):
            set_budget(budget)
            stage2_resolve(i)
            ev_r[i].record(side)
        budgets.append(budget)
    main.wait_event(ev_r[K - 1])
    torch.cuda.synchronize()
    return {"iterations_per_epoch": ipe, "budgets_per_iteration": budgets,
            "epoch_budgets": {str(k): v for k, v in sorted(loop.epoch_budget.items())},
            "umax_per_epoch": loop.umax_history}
