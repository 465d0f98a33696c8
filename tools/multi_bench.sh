#!/bin/bash
# Multi-GPU bench lines (one box, N GPUs): bench.py at 2 (and 4) ranks for the
# given layouts. Output: gpurun_out/multi_<layout>_n<P>.json
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for layout in ${LAYOUTS:-resnet50}; do
  for P in ${PS:-2 4}; do
    [ "$P" -le "$NG" ] || continue
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port $((29500 + P)) bench.py --gpus $P --layout $layout ${BENCH_ARGS:-} \
      > gpurun_out/multi_${layout}_n$P.log 2>&1
    echo "$layout P=$P rc=$?"
    grep '^{' gpurun_out/multi_${layout}_n$P.log | tail -1 > gpurun_out/multi_${layout}_n$P.json
    python - gpurun_out/multi_${layout}_n$P.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read())
    print(" ms/step", round(d["ms_per_step"], 4), "value", f'{d["value"]:.3e}', "roofline",
          {k: d["roofline"].get(k) for k in ("bound", "achieved", "frac", "hbm_frac")},
          "phases", d.get("phase_ms"), "ovl", (d.get("overlap") or {}).get("exposed_stage2_ms_mean"))
except Exception as e:
    print(" no json", e)
PY
  done
done
