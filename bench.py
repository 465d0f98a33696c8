"""OSP sync+LGP step benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one OSP iteration of the synchronization hot path for N_w = 8 logical
workers over the ResNet-50 layout (BASELINE.json configs[1]): stage 1 (barrier:
RS aggregate/apply/pull + LGP partial), the 4 ICS chunks (aggregate/apply/LGP
correct), and the resolution (PGP -> certified rank -> next GIB). Inputs are the
reference synthetic deltas (runner.cpp:312-321, seed 11), resident in HBM; the
two delta sets alternate between steps and total 2 x 818 MB (> L2, so no flush is
needed). One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "OSP sync+LGP step params/sec and HBM GB/s at 1/2/4/8 B200 vs roofline"
UNIT = "params/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--budget-frac", type=float, default=0.5)
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--stage-kernels", default="auto", choices=["auto", "tma", "register"],
                    help="stage-kernel family (OSP_GROUP_TMA / OSP_GROUP_REGISTER)")
    ap.add_argument("--graph-steps", type=int, default=16,
                    help="steps per captured CUDA graph (even: the two delta sets alternate)")
    ap.add_argument("--graph", action="store_true",
                    help="capture --graph-steps steps in a CUDA graph and time replays "
                         "(launch-bound layouts such as the MLP of config #1)")
    ap.add_argument("--sgd-lr", type=float, default=0.0,
                    help="> 0: the inputs are gradients, sgd_delta fused into the stage kernels")
    ap.add_argument("--momentum", type=float, default=0.0,
                    help="heavy-ball momentum on the gradients (extension; needs --sgd-lr)")
    ap.add_argument("--event-every", type=int, default=4,
                    help="stage-1 events on every k-th timed step (events between kernels "
                         "break the programmatic-dependent overlap; 1 = every step)")
    ap.add_argument("--no-graph-pass", action="store_true",
                    help="skip the extra CUDA-graph replay pass reported under 'graph'")
    ap.add_argument("--no-carry", action="store_true",
                    help="OSP_GROUP_NO_CARRY: stage 2 re-reads the deltas (A/B of the ICS carry)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-chunk", action="store_true", help="one stage-2 launch per ICS chunk")
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--overlap-ms", type=float, default=2.0,
                    help="synthetic compute t_c for the stage-2 overlap report (0 = skip)")
    return ap.parse_args()


def ncu_traffic(key: str, kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture, or None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[key][kernel]
        return d["dram_read_bytes"] + d["dram_write_bytes"]
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- clocks during the timed region -------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(
            ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits", "-lms", "100"],
            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- CPU baseline (reference engine on the host) ---------------------------------

def host_cpu():
    """CPU model and logical core count of this host (for the cpu_baseline line)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


_CONFIG_INDEX = {"mlp": 0, "mlp_acc": 0, "resnet50": 1, "resnet152": 2, "vgg16": 3, "llama1b": 4}


def workload_config(args, counts) -> dict:
    """The workload both arms run (identical dict in the b200 and the reference
    line; arm-specific keys live under "arm")."""
    M = sum(counts)
    idx = _CONFIG_INDEX.get(args.layout)
    return {"workload": f"{args.layout}-size OSP sync+LGP step, {args.workers} logical workers "
                        f"+ PS" + (f" (BASELINE configs[{idx}])" if idx is not None else ""),
            "layout": args.layout, "params": M, "layers": len(counts), "workers": args.workers,
            "budget_frac": args.budget_frac, "chunks": args.chunks,
            "deltas": f"reference synth generator (runner.cpp:312-321), seed {args.seed}, "
                      "generated outside the timed region",
            "l2": (f"inputs larger than L2 ({args.workers * M * 4 / 1e6:.0f} MB of delta rows per "
                   "step against the 126 MB L2), no flush" if args.workers * M * 4 > 126e6 else
                   f"{args.workers * M * 4 / 1e6:.3f} MB of delta rows per step: L2-resident, "
                   "launch-bound case")}


def run_reference_cpu(layout: str, workers: int, budget_frac: float, chunks: int, seed: int,
                      iters: int, warmup: int, threads: int, allow_port: bool = True):
    """Time the UNMODIFIED reference engine (oracle/_ref/ref_driver) on host cores.
    Without a runnable oracle/_ref the C restatement is timed instead and the
    result says kind "port" (allow_port=False raises instead)."""
    from paper_2306_16926_b200 import layouts
    drv = os.path.join(REPO, "oracle", "_ref", "ref_driver")
    counts = layouts.get(layout)
    path = os.path.join("/tmp", f"osp_layers_{layout}_{os.getpid()}.txt")
    with open(path, "w") as f:
        f.write(",".join(map(str, counts)))
    why = "oracle/_ref/ref_driver missing"
    if os.path.exists(drv):
        cmd = [drv, "bench", "--layers-file", path, "--workers", str(workers), "--budget-frac",
               str(budget_frac), "--chunks", str(chunks), "--seed", str(seed), "--iters",
               str(iters), "--warmup", str(warmup), "--threads", str(threads)]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=3600)
        if res.returncode == 0:
            d = json.loads(res.stdout.strip().splitlines()[-1])
            return {"value": d["params_per_s"], "unit": UNIT, "cores": threads,
                    "kind": "reference", "ms_per_step": d["median_ms"],
                    "mean_ms": d["mean_ms"], "total_ms": d.get("total_ms"), "steps_timed": d["steps"],
                    "sample": (f"reference pslab OspWorker/OspServer engine (oracle/_ref, g++ -O3), "
                               f"{layout} layout, {workers} workers, budget {budget_frac} x model, "
                               f"{chunks} chunks, {iters} timed steps after {warmup} warm-up, "
                               f"{threads} host thread(s) for the worker-side calls; synth delta "
                               f"generation excluded")}
        why = f"oracle/_ref/ref_driver exited {res.returncode}: {res.stderr.strip()[-200:]}"
    if not allow_port:
        raise RuntimeError(why)
    print(f"bench.py: reference engine unavailable ({why}); timing the C restatement",
          file=sys.stderr)
    # the C restatement (oracle/osp_oracle.c), single thread
    import numpy as np
    from oracle import oracle
    M = sum(counts)
    G = np.zeros(M, np.float32)
    P = np.zeros((workers, M), np.float32)
    flags = np.zeros(len(counts), np.uint8)
    order = np.zeros(0, np.int32)
    budget = int(budget_frac * M * 4)
    times = []
    for it in range(warmup + iters):
        X = np.stack([oracle.synth_delta(seed, w, it, M) for w in range(workers)])
        t0 = time.perf_counter()
        r = oracle.step(counts, 4, [1.0 / workers] * workers, X, G, P, flags, order, chunks, budget)
        t1 = time.perf_counter()
        flags, order = r["flags_out"], r["order_out"]
        if it >= warmup:
            times.append(t1 - t0)
    med = statistics.median(times)
    return {"value": M / med, "unit": UNIT, "cores": 1, "kind": "port", "ms_per_step": med * 1e3,
            "mean_ms": statistics.mean(times) * 1e3, "total_ms": sum(times) * 1e3,
            "steps_timed": len(times), "unavailable_reason": why,
            "sample": f"C restatement (oracle/osp_oracle.c), {layout}, {workers} workers, "
                      f"{iters} timed steps"}


def reference_arm(args, rank: int):
    """--impl reference: the reference engine on this box's host cores, all
    threads for the worker-side calls, the b200 arm's config / metric / unit.
    Times exactly --steps steps after --warmup warm-up steps; a 1-thread sample
    (the reference as shipped is single-threaded) is reported beside it."""
    if rank != 0:
        return
    from paper_2306_16926_b200 import layouts
    threads = os.cpu_count() or 1
    t0 = time.time()
    counts = layouts.get(args.layout)
    M = sum(counts)
    cb = run_reference_cpu(args.layout, args.workers, args.budget_frac, args.chunks, args.seed,
                           args.steps, args.warmup, threads)
    # whole-run throughput over the timed steps (mean, as the b200 arm's total / K)
    mean_ms = cb["mean_ms"]
    value = M / (mean_ms * 1e-3)
    one = None
    if threads > 1 and cb["kind"] == "reference":
        k1 = max(1, min(3, args.steps))
        c1 = run_reference_cpu(args.layout, args.workers, args.budget_frac, args.chunks,
                               args.seed, k1, 1, 1)
        one = {"value": M / (c1["mean_ms"] * 1e-3), "unit": UNIT, "cores": 1,
               "ms_per_step": c1["mean_ms"], "steps_timed": c1["steps_timed"],
               "sample": c1["sample"]}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": cb["steps_timed"], "warmup": args.warmup,
            "ms_per_step": mean_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64acc", "data": "synthetic",
            "config": workload_config(args, counts),
            "arm": {"engine": "reference pslab OspWorker/OspServer (oracle/_ref)"
                    if cb["kind"] == "reference" else "C restatement (oracle/osp_oracle.c)",
                    "host_threads": cb["cores"], "median_ms": cb["ms_per_step"],
                    "total_timed_ms": cb.get("total_ms"),
                    "deltas": "regenerated per iteration by the reference generator"},
            "cpu_baseline": dict({k: cb[k] for k in ("unit", "cores", "kind", "sample")},
                                 value=value, **host_cpu()),
            "cpu_baseline_1thread": one,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
            "wall_s": round(time.time() - t0, 2)}
    if cb["kind"] != "reference":
        line["reference_unavailable"] = cb.get("unavailable_reason")
    print(json.dumps(line), flush=True)


# ---- the B200 arm ---------------------------------------------------------------

MLP_WIDTHS = {"mlp": [8, 32, 4], "mlp_acc": [16, 64, 64, 4]}


def training_pass(args, N: int, K: int):
    """Config #1's whole training iteration on the device (MLP layouts): every
    worker's gradient from its own parameter row (the reference learner's
    forward_backward, kernels/learner.cu; config.hpp:30-41's default spec, relu +
    softmax CE, batch 32) and the OSP step with the fused sgd_delta, G iterations
    per CUDA graph, two batch sets alternating. Synthetic Gaussian-blob dataset
    (the shape of pslab::synth_dataset: n 1024, classes = output width)."""
    import torch

    from paper_2306_16926_b200 import layouts, learner, osp
    widths = MLP_WIDTHS[args.layout]
    counts = layouts.get(args.layout)
    M = sum(counts)
    n, d, k, B = 1024, widths[0], widths[-1], 32
    gen = torch.Generator(device="cpu").manual_seed(args.seed)
    labels = torch.arange(n, dtype=torch.int32) % k
    feats = torch.randn((n, d), generator=gen, dtype=torch.float32)
    feats[:, 0] += 6.0 * labels.float()
    feats, labels = feats.cuda(), labels.cuda()
    batches = [torch.randint(0, n, (N, B), generator=gen, dtype=torch.int32).cuda() for _ in range(2)]
    mlp = learner.Mlp(widths, feats, labels, "relu", "ce")
    p0 = (torch.rand(M, generator=gen) * 0.2 - 0.1).cuda()
    grp = osp.OspGroup(osp.Partition(counts), N, [1.0 / N] * N, n_chunks=args.chunks,
                       init_params=p0, sgd_lr=0.05)
    grp.set_budget(int(args.budget_frac * M * 4))
    grads = torch.empty((N, M), dtype=torch.float32, device="cuda")
    losses = torch.empty(N, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def it(j, producer_only=False):
        mlp.grad(grp.worker_params, batches[j % 2], out=grads, losses=losses, check=False)
        if not producer_only:
            grp.step(grads)

    def timed(producer_only):
        G = max(2, args.graph_steps + args.graph_steps % 2)
        reps = max(1, K // G)
        for j in range(4):
            it(j, producer_only)
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
            for j in range(G):
                it(j, producer_only)
        torch.cuda.synchronize()
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / (reps * G), reps * G

    ms_it, n_it = timed(False)
    ms_prod, _ = timed(True)
    mlp.check()
    out = {"ms_per_iteration": ms_it, "us_per_iteration": ms_it * 1e3,
           "producer_us": ms_prod * 1e3, "iterations": n_it,
           "spec": {"widths": widths, "activation": "relu", "loss": "softmax_cross_entropy",
                    "batch": B, "workers": N, "sgd_lr": 0.05},
           "launches_per_iteration": 1 + (1 if grp.single_launch else 3),
           "data": "synthetic Gaussian blobs on the device (n 1024), random batches",
           "note": "osp_mlp_grad (every worker's forward_backward, learner.cpp:299-367) + "
                   "osp_group_step with the fused sgd_delta, from a CUDA graph"}
    grp.close()
    return out


def reference_learner_us(widths, N: int):
    """The reference learner's forward_backward for N workers, one host thread
    (oracle/_ref/ref_fb --bench; cpu_baseline leg only)."""
    drv = os.path.join(REPO, "oracle", "_ref", "ref_fb")
    if not os.path.exists(drv):
        return None
    r = subprocess.run([drv, "--bench", ",".join(str(w) for w in widths), "relu", "ce", "32",
                        str(N), "2000" if widths[-1] <= 4 and len(widths) == 3 else "200"],
                       capture_output=True, text=True, timeout=300)
    return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None


def b200_single(args):
    import numpy as np
    import torch

    from paper_2306_16926_b200 import layouts, osp

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    counts = layouts.get(args.layout)
    N, M, L = args.workers, sum(counts), len(counts)
    model_bytes = M * 4
    budget = int(args.budget_frac * model_bytes)
    part = osp.Partition(counts)
    grp = osp.OspGroup(part, N, [1.0 / N] * N, n_chunks=args.chunks, tile_elems=args.tile,
                       tma={"auto": None, "tma": True, "register": False}[args.stage_kernels],
                       carry=not args.no_carry, sgd_lr=args.sgd_lr)
    if args.momentum > 0:
        grp.set_momentum(args.momentum)
    carry = not (osp.lib().osp_group_flags(grp._h) & 4)
    X = [osp.synth_deltas(args.seed, N, i, M) for i in range(2)]
    grp.set_budget(budget)
    stream = torch.cuda.current_stream()

    def step(k, evs=None, full=False):
        # timed region: events around stage 1 only (the roofline kernel), then
        # stage 2 + resolve as osp_group_step issues them (overlapped with the
        # ICS carry); the breakdown pass (full=True) runs stage 2 and the resolve
        # one after the other to time each
        x = X[k % 2]
        if evs is None and not full and not args.per_chunk:
            grp.step(x)  # stage 1 + stage2_resolve (one launch on launch-bound layouts)
            return
        if evs is not None:
            evs[0].record(stream)
        grp.stage1(x)
        if evs is not None:
            evs[1].record(stream)
        if args.per_chunk:
            for c in range(args.chunks):
                grp.stage2_chunk(c, x)
        elif not full:
            grp.stage2_resolve(x)
            return
        else:
            grp.stage2_all(x)
        if evs is not None and full:
            evs[2].record(stream)
        grp.resolve(x)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    tag0 = grp.read_gib()["tag"]  # GIB used by the first timed step
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    ev_every = max(1, args.event_every)
    sampled = [k for k in range(K) if k % ev_every == 0]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    graph = None
    if args.graph:
        # the step has no host sync and fixed arguments: G steps (delta sets 0
        # and 1 alternating, tags continue on the device) captured once and
        # replayed K/G times, so the host's graph-launch cost is amortised over
        # G device steps
        n_graph = max(2, args.graph_steps + args.graph_steps % 2)
        K += (-K) % n_graph
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cs, capture_error_mode="thread_local"):
            for j in range(n_graph):
                step(j)
        torch.cuda.synchronize()
        graph.replay()  # warm replay (n_graph more untimed steps)
        torch.cuda.synchronize()
        tag0 = grp.read_gib()["tag"]
    torch.cuda.synchronize()
    start.record(stream)
    if graph is not None:
        for _ in range(K // n_graph):
            graph.replay()
    else:
        for k in range(K):
            step(args.warmup + k, evs[k] if k % ev_every == 0 else None)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    ms_step = total_ms / K
    # breakdown pass (separate, so its extra events do not perturb the timed region)
    KB = min(K, 50)
    evb = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(KB + 1)]
    for k in range(KB + 1):
        step(args.warmup + K + k, evb[k], full=True)
    torch.cuda.synchronize()
    # per-step times in the timed region (stage-1 start to the next stage-1 start)
    if graph is None and len(sampled) > 1:
        # consecutive sampled stage-1 starts are ev_every steps apart
        per = sorted(evs[a][0].elapsed_time(evs[b][0]) / (b - a)
                     for a, b in zip(sampled, sampled[1:]))
        step_pct = {"p50_ms": per[len(per) // 2], "p90_ms": per[min(len(per) - 1, int(0.9 * len(per)))],
                    "n": len(per), "steps_per_sample": ev_every}
    else:
        step_pct = None
    # the same step replayed from a CUDA graph (separate pass, not the headline:
    # a replay carries no stage-1 events for the roofline)
    graph_pass = None
    if graph is None and not args.no_graph_pass:
        gp = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.graph(gp, stream=cs, capture_error_mode="thread_local"):
            step(0)
            step(1)
        torch.cuda.synchronize()
        gp.replay()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = max(K // 2, 1)
        torch.cuda.synchronize()
        ga.record(stream)
        for _ in range(nrep):
            gp.replay()
        gb.record(stream)
        torch.cuda.synchronize()
        g_ms = ga.elapsed_time(gb) / (2 * nrep)
        graph_pass = {"ms_per_step": g_ms, "value": M / (g_ms * 1e-3), "steps": 2 * nrep,
                      "note": "osp_group_step x2 captured once, replayed; not the headline"}
        del gp
    # stage-1 launch times: from the timed region, or (graph replays carry no
    # events) from the breakdown pass
    s1 = ([evs[k][0].elapsed_time(evs[k][1]) for k in sampled] if graph is None else
          [evb[k][0].elapsed_time(evb[k][1]) for k in range(KB)])
    s2 = [evb[k][1].elapsed_time(evb[k][2]) for k in range(KB)]
    s3 = [evb[k][2].elapsed_time(evb[k + 1][0]) for k in range(KB)]
    # u of each timed step = deferred bytes of the GIB it split with (tags tag0..)
    # (the device ring keeps the last 4096 tags: a longer run takes the window's
    # mean for its earlier steps)
    nh = min(K, 4096)
    deferred = grp.deferred_history(tag0 + K - nh, nh).astype(np.float64)
    if nh < K:
        deferred = np.concatenate([np.full(K - nh, deferred.mean()), deferred])
    u = deferred / model_bytes
    # algorithmic bytes. SURVEY §8(d): stage 1 = 4M[(2N+2) - u] (N delta rows + G read,
    # N worker rows + G on RS written), stage 2 = 4M u (2N+1) (N rows + G re-read,
    # G + N rows written). With the ICS carry stage 1 also writes C on ICS
    # (4M(2N+2)) and stage 2 reads C once and writes G + N rows (4M u (N+2)).
    # momentum adds the velocity rows, read and written once in stage 1 (4M * 2N)
    mom_b = 4.0 * M * 2 * N if args.momentum > 0 else 0.0
    b_s1 = [4.0 * M * ((2 * N + 2) - (0.0 if carry else uk)) + mom_b for uk in u]
    b_step = [4.0 * M * ((2 * N + 2) + uk * ((N + 2) if carry else (2 * N + 1))) + mom_b
              for uk in u]
    b_survey = [4.0 * M * ((2 * N + 2) + uk * (2 * N + 1)) for uk in u]
    s1_avg = sum(s1) / len(s1)
    b_s1_avg = (sum(b_s1[k] for k in sampled) / len(sampled) if graph is None
                else sum(b_s1) / K)
    ach_s1 = b_s1_avg / (s1_avg * 1e-3) / 1e9
    ach_step = (sum(b_step) / K) / (ms_step * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    # the step time the SURVEY byte model allows at the measured peak
    survey_ms = (sum(b_survey) / K) / (peak * 1e9) * 1e3
    stats = grp.stats()
    # stage1, stage2, resolve (the sampled evented steps always take this path);
    # single-launch layouts: one launch on the unevented steps
    launches_3 = 1 + (args.chunks if args.per_chunk else 1) + 1
    n_evented = 0 if graph is not None else len(sampled)
    if grp.single_launch and not args.per_chunk:
        gpu_launches = n_evented * launches_3 + (K - n_evented)
    else:
        gpu_launches = K * launches_3

    # ---- stage 2 overlapped with the next iteration's (synthetic) compute
    ovl = None
    if args.overlap_ms > 0:
        from paper_2306_16926_b200 import overlap
        comp = overlap.SyntheticCompute(args.overlap_ms)

        def s2r(i):
            grp.stage2_resolve(X[i % 2])

        ovl = overlap.run(lambda i: grp.stage1(X[i % 2]), s2r, comp, K=min(K, 50), W=3)
        ovl["t_c_ms"] = comp.ms
        ovl["budget_frac"] = args.budget_frac
        # closed-loop budget (runner.cpp:364-376, protocol.cpp:396-405): the SGU
        # budget per epoch from the measured compute time and the measured rate
        # of the synchronization traffic (HBM bytes of the step on one GPU)
        from paper_2306_16926_b200.budget import BudgetLoop
        ipe = 5
        loop = BudgetLoop(ipe, N, model_bytes)
        tag_cl = grp.read_gib()["tag"]

        def link_bytes(j):
            uj = float(grp.deferred_history(tag_cl + j, 1)[0]) / model_bytes
            return 4.0 * M * ((2 * N + 2) + uj * ((N + 2) if carry else (2 * N + 1)))

        ovl["closed_loop"] = overlap.run_closed_loop(lambda i: grp.stage1(X[i % 2]), s2r,
                                                     grp.set_budget, comp, loop, link_bytes,
                                                     K=30, ipe=ipe)
        grp.set_budget(budget)

    # ---- e2e through the C-ABI with host buffers (pinned): H2D of the step's N
    # delta rows, the step, D2H of the next GIB and of the updated global vector
    # (every worker's parameters at the boundary), all inside the timed call.
    # One pinned host set for small layouts two; the 1B layout's 40 GB set is pinned once
    n_sets = 2 if N * M * 4 <= (8 << 30) else 1
    host = [X[i].cpu().pin_memory() for i in range(n_sets)]
    params_host = torch.empty(M, dtype=torch.float32).pin_memory()
    e2e_ms = []
    for k in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        grp.step_host(host[k % n_sets], params_out=params_host)
        t1 = time.perf_counter()
        if k > 0:
            e2e_ms.append((t1 - t0) * 1e3)
    e2e_step = statistics.median(e2e_ms)
    # the same calls pipelined (osp_group_step_host_async): call k's H2D beside
    # call k-1's step and D2H; wall clock from the first call to the final wait
    # (its two staging sets are skipped where they would not fit beside the
    # state: the 1B layout's rows are 40 GB per set)
    E = max(10, args.e2e_steps)
    e2e_pipe = None
    if N * M * 4 <= (8 << 30):
        params_pipe = [torch.empty(M, dtype=torch.float32).pin_memory() for _ in range(2)]
        grp.step_host_async(host[0], params_out=params_pipe[0])
        grp.host_wait()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(E):
            grp.step_host_async(host[k % n_sets], params_out=params_pipe[k % 2])
        grp.host_wait()
        e2e_pipe = (time.perf_counter() - t0) * 1e3 / E
    gib_bytes = 8 + (L + 7) // 8

    s1_kernel = "k_stage_tma<1>" if grp.stage_kernels == "tma-staged" else "k_stage1"
    line = {
        "metric": METRIC, "value": M / (ms_step * 1e-3), "unit": UNIT, "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64acc", "data": "synthetic",
        "config": workload_config(args, counts),
        "arm": {"parallelism": "single GPU", "tile_elems": grp.geometry()["tile_elems"],
                "stage_kernels": grp.stage_kernels, "ics_carry": carry,
                "deltas": "2 device-resident sets (iterations 0 and 1) alternating",
                "inputs": (f"gradients, sgd_delta lr {args.sgd_lr}" if args.sgd_lr > 0 else "deltas")
                + (f", momentum {args.momentum}" if args.momentum > 0 else ""),
                "launch": f"CUDA graph ({n_graph} steps per replay)" if graph is not None else "stream",
                "single_launch_step": grp.single_launch},
        "hbm_gbs_step": ach_step,
        "roofline": {"bound": "hbm",
                     "kernel": s1_kernel + (" (barrier: RS agg/apply + LGP + ICS carry)" if carry
                                            else " (barrier: RS agg/apply + LGP)"),
                     "achieved": ach_s1, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": ach_s1 / peak,
                     "traffic": ncu_traffic(f"{args.layout}/N{N}/b{args.budget_frac}",
                                            s1_kernel + ("" if carry or s1_kernel == "k_stage1"
                                                         else " no-carry")),
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, one launch)",
                     "alg_bytes_per_launch": b_s1_avg, "avg_launch_ms": s1_avg,
                     "launches_timed": len(s1),
                     "step_frac": ach_step / peak,
                     "step_alg_bytes": sum(b_step) / K,
                     "step_bytes_model": ("4M[(2N+2) + u(N+2)] (ICS carry)" if carry else
                                          "4M[(2N+2) + u(2N+1)] (SURVEY §8(d))"),
                     "survey_roofline_ms": survey_ms,
                     "vs_survey_roofline": survey_ms / ms_step},
        "breakdown_ms": {"stage1": s1_avg, "after_stage1": ms_step - s1_avg,
                         "stage2_alone": sum(s2) / KB, "resolve_alone_and_gaps": sum(s3) / KB,
                         "note": "stage1 and after_stage1 (stage 2 + resolve as the step issues "
                                 "them: overlapped with the ICS carry) from the timed region; "
                                 "stage2_alone / resolve_alone from a separate serial evented "
                                 "pass of min(K, 50) steps"},
        "u_mean": float(u.mean()),
        "e2e": {"value": M / ((e2e_pipe or e2e_step) * 1e-3), "unit": UNIT,
                "ms_per_step": e2e_pipe or e2e_step,
                "h2d_bytes_per_step": N * M * 4, "d2h_bytes_per_step": gib_bytes + 4 * M,
                "path": ("osp_group_step_host_async (C-ABI), pipelined over consecutive steps: "
                         "pinned host delta rows in, the updated global vector (= every worker's "
                         "params) out, every step; wall clock from the first call to the final "
                         "osp_group_host_wait") if e2e_pipe else
                        "osp_group_step_host (synchronous; see sync_call)",
                "steps": E if e2e_pipe else len(e2e_ms),
                "sync_call": {"ms_per_step": e2e_step, "value": M / (e2e_step * 1e-3),
                              "path": "osp_group_step_host (synchronous): H2D, step, D2H of the "
                                      "next GIB and the global vector, median of "
                                      f"{len(e2e_ms)} calls"}},
        "gpu_launches": gpu_launches,
        "certificate": stats,
        "graph": graph_pass,
        "step_ms_percentiles": step_pct,
        "clocks": clk,
        "overlap": ovl,
    }
    if args.layout in MLP_WIDTHS:
        line["training"] = training_pass(args, N, K)
    if not args.no_cpu_baseline:
        try:
            cb = run_reference_cpu(args.layout, N, args.budget_frac, args.chunks, args.seed,
                                   args.cpu_iters, 1, 1)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"].update(host_cpu())
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"error": str(e)[:200]}
        if args.layout in MLP_WIDTHS:
            try:
                rl = reference_learner_us(MLP_WIDTHS[args.layout], N)
                if rl and "training" in line:
                    sync_us = (M / cb["value"]) * 1e6 if "value" in line["cpu_baseline"] else None
                    line["training"]["reference_cpu"] = {
                        "learner_us": rl["us_per_iteration"], "sync_us": sync_us,
                        "us_per_iteration": rl["us_per_iteration"] + (sync_us or 0.0),
                        "kind": "reference", "cores": 1,
                        "sample": f"{rl['reps']} iterations of {N} workers' forward_backward "
                                  "(oracle/_ref/ref_fb --bench) + the sync step above"}
            except Exception as e:
                line["training"]["reference_cpu"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    if world > 1 or args.gpus > 1:
        from paper_2306_16926_b200 import dist_bench
        dist_bench.run(args, METRIC, UNIT)
        return
    b200_single(args)


if __name__ == "__main__":
    main()
