#!/bin/bash
# ncu evidence for the committed profiles (one GPU): launch list + full capture of
# the stage kernels and the resolve kernel on the default bench workload.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --overlap-ms 0 ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stage|k_resolve" -s 6 -c 3 -o gpurun_out/${OUT:-prof_r1} $CMD > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
