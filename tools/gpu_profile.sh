#!/bin/bash
# One GPU session: parity tests, a tile sweep, the launch list and one full ncu
# capture of the two stage kernels. Outputs land in gpurun_out/ (scratch);
# summaries worth keeping are copied to profiles/ by hand.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for t in ${TILES:-256 512 1024}; do
  python bench.py --tile $t --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_t$t.log 2>&1
  python - "$t" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_t{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("tile", sys.argv[1], round(d["ms_per_step"], 4), {k: round(v, 4) for k, v in d["breakdown_ms"].items()},
      "s1_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["roofline"]["step_frac"], 3), d["clocks"])
PY
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
if [ "${FULL:-1}" = "1" ]; then
  $CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_stage -s 4 -c 2 -o gpurun_out/prof_stage $CMD > gpurun_out/ncu_full.log 2>&1
  echo "full capture rc=$?"
fi
