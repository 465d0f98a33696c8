"""bench.py --gpus N (N > 1, launched by torchrun): the sharded OSP step.

N_w = 8 logical workers spread N_w/N per GPU (strong scaling: the job is one
OSP iteration over the whole model per step, whatever N). Timing: W warm-up
steps, barrier + synchronize, K steps bracketed by CUDA events on the launching
stream, max over ranks. The timed step is the single-exchange mode (one
exchange kernel, the resolve and the local stage-2 broadcast); the overlap
report runs the deferred-ICS mode (stage 2's exchange beside the next
iteration's compute) with a fixed budget and with the closed-loop budget.
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np
import torch
import torch.distributed as dist


def _max(vals, device="cuda"):
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def run(args, metric: str, unit: str):
    from bench import workload_config

    from . import layouts, osp
    from .dist import ShardGroup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # OSP_BENCH_OVERSUB=1: more ranks than GPUs (ranks share devices, gloo for the
    # host-side barrier / max-over-ranks): exercises the P-rank code path on a
    # smaller box; its timings are meaningless and the line says so
    oversub = os.environ.get("OSP_BENCH_OVERSUB") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = "cpu" if oversub else "cuda"
    counts = layouts.get(args.layout)
    N, M, L = args.workers, sum(counts), len(counts)
    n_loc = N // world
    model_bytes = 4 * M
    budget = int(args.budget_frac * model_bytes)
    part = osp.Partition(counts)
    sh = ShardGroup(part, N, None, n_chunks=args.chunks, tile_elems=args.tile)
    sh.connect_via()
    for b in range(2):
        sh.fill_synth(args.seed, b, b)
    sh.set_budget(budget)
    stream = torch.cuda.current_stream()

    def step(k):
        buf = k % 2
        if args.per_chunk:
            # message-by-message shape: stage 1, one stage-2 launch per chunk, resolve
            sh.stage1(buf)
            for c in range(args.chunks):
                sh.stage2(buf, c, c + 1)
            sh.resolve(buf)
        else:
            sh.step(buf)

    for k in range(args.warmup):
        step(k)
    sh.check()
    torch.cuda.synchronize()
    tag0 = sh.read_gib()["tag"]
    K = args.steps
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    clocks = None
    if rank == 0:
        from bench import ClockSampler
        clocks = ClockSampler(local)
        clocks.start()
        time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    start.record(stream)
    for k in range(K):
        step(args.warmup + k)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    sh.check()
    total_ms, = _max([start.elapsed_time(end)], dev)
    ms_step = total_ms / K
    u = sh.local.deferred_history(tag0, K).astype(np.float64) / model_bytes
    u_mean = float(u.mean())
    sync = sh.sync_form
    if sync == "chain":
        # the chain (kernels/shard_chain.cu): every link r -> r+1 carries the fp64
        # running sums (8 B per element) and the last rank serves its 4-byte
        # aggregate to the P-1 others: the busiest direction of any GPU
        nvl_bytes = max(8.0 * M, 4.0 * M * (world - 1))
        # rank 0's HBM bytes (the busier rank): its rows read (4 NL), the running
        # sums written and read by the next rank (16), G read for the deferred
        # tiles' local estimates and for the apply (u + 1), rows written (4 NL:
        # local estimates on deferred tiles, G' on the others), G or C written
        # (1), and the stage-2 broadcast (carry read, G + rows written)
        hbm_bytes = 4.0 * M * (2 * n_loc + 4 + u_mean + 1 + 1 + u_mean * (2 + n_loc))
    else:
        # per-GPU NVLink bytes per step, each direction: the peers' delta rows
        # this rank's shard reads + its aggregate stored into the other ranks
        nvl_bytes = 4.0 * M * ((N - n_loc) / world + (world - 1) / world)
        # per-GPU algorithmic HBM bytes per step (single exchange): local rows
        # read once (by this rank or a peer) and written once, G read, the pull
        # buffer written everywhere and read back on the peers' tiles, G (RS) /
        # carry (ICS) written, the local rows re-read for the peers' deferred
        # tiles, and the stage-2 broadcast (carry read, G + local rows written)
        hbm_bytes = 4.0 * M * (2 * n_loc + 1 + 1 + (world - 1) / world + 1
                               + u_mean * (n_loc * (world - 1) / world + 2 + n_loc))

    # ---- per-phase breakdown (events between kernels, 5 profiled steps, max over ranks)
    prof = [sh.profile(k % 2) for k in range(5)]
    keys = list(prof[0])
    phases = dict(zip(keys, _max([sum(p[k] for p in prof) / len(prof) for k in keys], dev)))

    # ---- e2e: pinned host deltas -> device (this rank's rows), step, result read-back
    host = [sh.deltas(b).cpu().pin_memory() for b in range(2)]
    params_host = torch.empty(M, dtype=torch.float32).pin_memory()
    e2e = []
    for k in range(args.e2e_steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh.deltas(k % 2).copy_(host[k % 2], non_blocking=True)
        step(k)
        if rank == 0:  # the step's result: the updated global vector (= every worker's params)
            params_host.copy_(sh.global_params, non_blocking=True)
        sh.read_gib()  # synchronising D2H of the next GIB
        t1 = time.perf_counter()
        if k > 0:
            e2e.append((t1 - t0) * 1e3)
    e2e_ms, = _max([statistics.median(e2e)], dev)
    # the same pipelined over consecutive steps: step k+1's rows go H2D on a
    # copy stream into the other delta buffer while step k runs and rank 0's
    # D2H of its global vector runs on a third stream; wall clock from the
    # first copy to the last read-back, max over ranks
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_step = [torch.cuda.Event() for _ in range(2)]
    ev_out = torch.cuda.Event()
    E = max(10, args.e2e_steps)

    def pipelined(n):
        for k in range(n):
            b = k % 2
            if k >= 2:
                h2d.wait_event(ev_step[b])  # step k-2 has read this buffer
            with torch.cuda.stream(h2d):
                sh.deltas(b).copy_(host[b], non_blocking=True)
                ev_in[b].record(h2d)
            stream.wait_event(ev_in[b])
            if k >= 1:
                stream.wait_event(ev_out)  # the previous read-back of G is done
            step(k)
            ev_step[b].record(stream)
            if rank == 0:
                d2h.wait_event(ev_step[b])
                with torch.cuda.stream(d2h):
                    params_host.copy_(sh.global_params, non_blocking=True)
            ev_out.record(d2h)
        torch.cuda.synchronize()

    pipelined(2)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipelined(E)
    e2e_pipe, = _max([(time.perf_counter() - t0) * 1e3 / E], dev)
    sh.check()
    geometry = sh.local.geometry()
    mode = sh.mode
    sh.close()
    del host
    torch.cuda.empty_cache()

    # ---- OSP overlap: the deferred-ICS mode, stage 2's exchange on a side stream
    # beside the next iteration's (synthetic) compute; fixed budget, then the
    # closed-loop budget from the measured t_c and NVLink rate
    ovl = None
    if args.overlap_ms > 0:
        from . import overlap
        from .budget import BudgetLoop
        sd = ShardGroup(part, N, None, n_chunks=args.chunks, tile_elems=args.tile, defer_ics=True)
        sd.connect_via()
        for b in range(2):
            sd.fill_synth(args.seed, b, b)
        sd.set_budget(budget)
        comp = overlap.SyntheticCompute(args.overlap_ms)

        def s2r(i):
            sd.stage2(i % 2)
            sd.resolve(i % 2)

        res = overlap.run(lambda i: sd.stage1(i % 2), s2r, comp, K=min(K, 50), W=3)
        sd.check()
        keys = ["iter_ms_overlapped", "iter_ms_serial", "exposed_stage2_ms_mean",
                "exposed_stage2_ms_max", "stage2_plus_resolve_ms_mean"]
        ovl = dict(zip(keys + ["t_c_ms"], _max([res[k] for k in keys] + [comp.ms], dev)))
        ovl["mode"] = sd.mode
        ovl["budget_frac"] = args.budget_frac
        # closed loop (runner.cpp:364-376, protocol.cpp:396-405): budgets start
        # at 0 and follow Eq. 5 / Alg. 1 from the measured t_c and NVLink rate
        # (the per-GPU NVLink bytes of an iteration do not depend on its split:
        # every element crosses the links once, in stage 1 or in stage 2)
        ipe = 5
        loop = BudgetLoop(ipe, N, model_bytes)
        def agree(vals):  # rank 0's measurements decide (every rank builds the same GIB)
            t = torch.tensor(vals, dtype=torch.float64, device=dev)
            dist.broadcast(t, 0)
            return [float(x) for x in t.tolist()]

        cl = overlap.run_closed_loop(lambda i: sd.stage1(i % 2), s2r, sd.set_budget, comp, loop,
                                     lambda j: nvl_bytes, K=30, ipe=ipe, agree=agree)
        sd.check()
        ovl["closed_loop"] = cl
        sd.close()

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except Exception:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        nvl_peak = 770.0
        hbm_gbs = hbm_bytes / (ms_step * 1e-3) / 1e9
        nvl_gbs = nvl_bytes / (ms_step * 1e-3) / 1e9
        line = {
            "metric": metric, "value": M / (ms_step * 1e-3), "unit": unit, "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64acc", "data": "synthetic",
            "config": workload_config(args, counts),
            "arm": {"parallelism": f"ps-shard{world}", "workers_per_gpu": n_loc,
                    "shard_mode": mode, "sync_form": sync, "tile_elems": geometry["tile_elems"],
                    "deltas": "2 device-resident sets (iterations 0 and 1) alternating",
                    "per_chunk": bool(args.per_chunk)},
            "roofline": {"bound": "nvlink" if nvl_bytes / nvl_peak > hbm_bytes / hbm_peak else "hbm",
                         "kernel": ("k_shard_chain (fp64 running-sum chain + pull of the aggregate, "
                                    "one launch per step)" if sync == "chain" else
                                    "k_shard_x (exchange + apply, one launch per step)"),
                         "achieved": nvl_gbs, "peak": nvl_peak, "unit": "GB/s",
                         "frac": nvl_gbs / nvl_peak, "traffic": None,
                         "note": "per-GPU NVLink bytes of the busiest direction / step time; peak = measured "
                                 "one-way peer copy 770 GB/s (B200_PROFILING.md); both directions "
                                 "load at once, where the measured ceiling is 667 GB/s",
                         "nvlink_bytes_per_gpu_per_direction": nvl_bytes,
                         "collective_bus_gbs": nvl_gbs,
                         "frac_vs_bidirectional_667": nvl_gbs / 667.0,
                         "hbm_gbs_per_gpu": hbm_gbs, "hbm_frac": hbm_gbs / hbm_peak,
                         "hbm_alg_bytes_per_gpu": hbm_bytes},
            "phase_ms": phases,
            "overlap": ovl,
            "u_mean": u_mean,
            "e2e": {"value": M / (e2e_pipe * 1e-3), "unit": unit, "ms_per_step": e2e_pipe,
                    "pipelined": True, "steps": E,
                    "sync_steps": {"ms_per_step": e2e_ms, "value": M / (e2e_ms * 1e-3),
                                   "path": "the same, one step at a time (H2D, step, GIB read "
                                           "on every rank, global vector on rank 0), median"},
                    "h2d_bytes_per_step": n_loc * M * 4 * world,
                    "d2h_bytes_per_step": 4 * M,
                    "path": "every rank: pinned host rows -> osp_shard_deltas on a copy stream "
                            "(one buffer ahead), osp_shard_step; rank 0: the updated global "
                            "vector (= every worker's params) read back on a third stream, every "
                            "step; wall clock over the pipelined steps, max over ranks"},
            # per step: the exchange kernel, the resolve, the stage-2 broadcast
            # (per chunk: one broadcast launch per chunk)
            "gpu_launches": K * (2 + (args.chunks if args.per_chunk else 1)),
            "clocks": clk,
        }
        if oversub:
            line["oversubscribed"] = (f"{world} ranks on {torch.cuda.device_count()} GPUs: "
                                      "code-path check, timings not meaningful")
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
