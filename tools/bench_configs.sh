#!/bin/bash
# BASELINE.json configs #2-#5 on one B200 (bench.py lines, one per config),
# plus the 1B budget sweep. Output: gpurun_out/bench_configs.jsonl
set -u
mkdir -p gpurun_out
out=gpurun_out/bench_configs.jsonl
: > $out
run() { timeout 900 python bench.py "$@" 2>gpurun_out/bench_err.log | tail -1 >> $out || echo "{\"failed\": \"$*\"}" >> $out; }
run --layout mlp --budget-frac 0.5 --cpu-iters 20 --steps 2000 --e2e-steps 20 --graph
run --layout resnet50 --budget-frac 0.5 --cpu-iters 3
run --layout resnet152 --budget-frac 0.5 --cpu-iters 2
run --layout vgg16 --budget-frac 0.5 --cpu-iters 1 --steps 100
for b in 0.0 0.2 0.4 0.5 0.6 0.8 1.0; do
  run --layout llama1b --budget-frac $b --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline
done
python - <<'PY'
import json
for ln in open("gpurun_out/bench_configs.jsonl"):
    d = json.loads(ln)
    if "failed" in d: print(d); continue
    c = d["config"]
    print(f'{c["workload"][:30]:30s} b={c["budget_frac"]} u={d["u_mean"]:.3f} ms={d["ms_per_step"]:.3f} '
          f'params/s={d["value"]:.3e} s1_frac={d["roofline"]["frac"]:.3f} step_frac={d["roofline"]["step_frac"]:.3f} vs_survey={d["roofline"].get("vs_survey_roofline",0):.3f} '
          f'e2e_ms={d["e2e"]["ms_per_step"]:.1f} cpu={d.get("cpu_baseline",{}).get("value")} fb={d["certificate"]}')
PY
