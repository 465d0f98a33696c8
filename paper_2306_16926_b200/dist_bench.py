"""bench.py --gpus N (N > 1, launched by torchrun): the sharded OSP step.

N_w = 8 logical workers spread N_w/N per GPU (strong scaling: the job is one
OSP iteration over the whole model per step, whatever N). Timing: W warm-up
steps, barrier + synchronize, K steps bracketed by CUDA events on the launching
stream, max over ranks.
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np
import torch
import torch.distributed as dist


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
    counts = layouts.get(args.layout)
    N, M, L = args.workers, sum(counts), len(counts)
    model_bytes = 4 * M
    budget = int(args.budget_frac * model_bytes)
    part = osp.Partition(counts)
    sh = ShardGroup(part, N, None, n_chunks=args.chunks, tile_elems=args.tile)
    sh.connect_via()
    for b in range(2):
        sh.fill_synth(args.seed, b, b)
    sh.set_budget(budget)
    stream = torch.cuda.current_stream()

    def step(k, evs=None):
        buf = k % 2
        if evs is not None:
            evs[0].record(stream)
        if args.per_chunk:
            # message-by-message shape: barrier stage, then one launch set per chunk
            sh.stage1(buf)
            if evs is not None:
                evs[1].record(stream)
            for c in range(args.chunks):
                sh.stage2(buf, c, c + 1)
            if evs is not None:
                evs[2].record(stream)
            sh.resolve(buf)
        else:
            # fused step: stage-2 push/pull inside the stage-1 apply launch
            sh.step(buf)
            if evs is not None:
                evs[1].record(stream)
                evs[2].record(stream)

    for k in range(args.warmup):
        step(k)
    sh.check()
    torch.cuda.synchronize()
    tag0 = sh.read_gib()["tag"]
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
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
    ev_every = max(1, getattr(args, "event_every", 4))
    sampled = [k for k in range(K) if k % ev_every == 0]
    for k in range(K):
        step(args.warmup + k, evs[k] if k % ev_every == 0 else None)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    sh.check()
    local_ms = start.elapsed_time(end)
    s1 = sum(evs[k][0].elapsed_time(evs[k][1]) for k in sampled) / len(sampled)
    s2 = sum(evs[k][1].elapsed_time(evs[k][2]) for k in sampled) / len(sampled)
    t = torch.tensor([local_ms, s1, s2], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, s1_max, s2_max = (float(x) for x in t.tolist())
    ms_step = total_ms / K
    u = sh.local.deferred_history(tag0, K).astype(np.float64) / model_bytes
    n_loc = N // world
    u_mean = float(u.mean())
    # per-GPU algorithmic HBM bytes per step
    if sh.streaming:
        # local rows read once (by this rank or an owner), G read + written, agg
        # written into the pull buffer (own tiles locally, the rest by the peers)
        # and read back on the peers' tiles, worker rows, local estimate on ICS
        # layers
        hbm_bytes = 4.0 * M * (2 * n_loc + 2 + 1 + (world - 1.0) / world
                               + u_mean * (2 * n_loc + 1))
    else:
        # own rows served to the shard owners, agg written + read, G read + written,
        # worker rows (+ local estimate on ICS layers)
        hbm_bytes = 4.0 * M * (4 + n_loc * (2 + 2 * u_mean))
    # per-GPU NVLink bytes per step (each direction): remote delta rows read by this
    # rank's shard + its aggregate stored to the other ranks
    nvl_bytes = 4.0 * M * ((N - n_loc) / world + (world - 1) / world)

    # ---- per-phase breakdown (events between kernels, 5 profiled steps, max over ranks)
    phases = None
    prof = [sh.profile(k % 2) for k in range(5)]
    keys = list(prof[0])
    pt = torch.tensor([sum(p[k] for p in prof) / len(prof) for k in keys], dtype=torch.float64,
                      device="cuda")
    dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    phases = {k: float(v) for k, v in zip(keys, pt.tolist())}

    # ---- stage 2 overlapped with the next iteration's (synthetic) compute
    ovl = None
    if args.overlap_ms > 0:
        from . import overlap
        comp = overlap.SyntheticCompute(args.overlap_ms)

        def s2r(i):
            sh.stage2(i % 2)
            sh.resolve(i % 2)

        res = overlap.run(lambda i: sh.stage1(i % 2), s2r, comp, K=min(K, 50), W=3)
        sh.check()
        keys = ["iter_ms_overlapped", "iter_ms_serial", "exposed_stage2_ms_mean",
                "exposed_stage2_ms_max", "stage2_plus_resolve_ms_mean"]
        ot = torch.tensor([res[k] for k in keys] + [comp.ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(ot, op=dist.ReduceOp.MAX)
        ovl = {k: float(v) for k, v in zip(keys + ["t_c_ms"], ot.tolist())}
        # Eq. 5 budget from the measured compute time and the measured per-GPU
        # NVLink rate of this run (runner.cpp:364-376 umax_measured, on hardware)
        nvl_bps = nvl_bytes / (total_ms / K * 1e-3)
        ovl["umax_measured_bytes"] = osp.compute_umax(nvl_bps, ovl["t_c_ms"] * 1e-3, N,
                                                      model_bytes)
        ovl["umax_frac_of_model"] = ovl["umax_measured_bytes"] / model_bytes

    # ---- e2e: pinned host deltas -> device (this rank's rows), step, GIB read-back
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
    e2e_t = torch.tensor([statistics.median(e2e)], dtype=torch.float64, device="cuda")
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_t.item())
    peaks = {}
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    nvl_peak = 770.0
    if rank == 0:
        hbm_gbs = hbm_bytes / (ms_step * 1e-3) / 1e9
        nvl_gbs = nvl_bytes / (ms_step * 1e-3) / 1e9
        line = {
            "metric": metric, "value": M / (ms_step * 1e-3), "unit": unit, "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64acc", "data": "synthetic",
            "config": workload_config(args, counts),
            "arm": {"parallelism": f"ps-shard{world}", "workers_per_gpu": n_loc,
                    "shard_kernels": sh.mode,
                    "deltas": "2 device-resident sets (iterations 0 and 1) alternating",
                    "tile_elems": sh.local.geometry()["tile_elems"]},
            "roofline": {"bound": "nvlink" if nvl_bytes / nvl_peak > hbm_bytes / hbm_peak else "hbm",
                         "achieved": nvl_gbs, "peak": nvl_peak, "unit": "GB/s",
                         "frac": nvl_gbs / nvl_peak, "traffic": None,
                         "note": "per-GPU NVLink bytes each direction / step time; peak = measured "
                                 "peer copy 770 GB/s (B200_PROFILING.md)",
                         "nvlink_bytes_per_gpu_per_direction": nvl_bytes,
                         "collective_bus_gbs": nvl_gbs,
                         "frac_vs_bidirectional_667": nvl_gbs / 667.0,
                         "ncu": "profiles/r1_ncu_full_shard_agg_solo.csv (k_shard_agg alone: NVLink "
                                "rx user bytes == algorithmic; a profiled multi-rank step cannot "
                                "run under ncu, see profiles/r1_multi_gpu_notes.md)",
                         "hbm_gbs_per_gpu": hbm_gbs, "hbm_frac": hbm_gbs / hbm_peak},
            "breakdown_ms": ({"stage1": s1_max, "stage2": s2_max,
                              "resolve": ms_step - s1_max - s2_max} if args.per_chunk
                             else {"step": s1_max}),
            "phase_ms": phases,
            "overlap": ovl,
            "u_mean": u_mean,
            "e2e": {"value": M / (e2e_ms * 1e-3), "unit": unit, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": n_loc * M * 4 * world,
                    "d2h_bytes_per_step": (8 + (L + 7) // 8) * world + 4 * M,
                    "path": "pinned host rows -> osp_shard_deltas, osp_shard_* step, GIB read on "
                            "every rank, updated global vector read on rank 0"},
            # streaming: stage1, stage2, resolve per step (per chunk: one stage-2 launch
            # each); barrier mode: agg1, apply1+agg2, apply2, resolve (per chunk: agg1,
            # apply1, agg2 + apply2 per chunk, resolve)
            "gpu_launches": K * (((2 + args.chunks) if args.per_chunk else 3) if sh.streaming
                                 else ((3 + 2 * args.chunks) if args.per_chunk else 4)),
            "clocks": clk,
        }
        if oversub:
            line["oversubscribed"] = (f"{world} ranks on {torch.cuda.device_count()} GPUs: "
                                      "code-path check, timings not meaningful")
        print(json.dumps(line), flush=True)
    dist.barrier()
    sh.close()
    dist.destroy_process_group()
