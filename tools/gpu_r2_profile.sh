# round-2 ncu evidence (one B200): launch list of the default bench, a full
# capture of the stage kernels + resolve, and of the single-launch MLP step
CMD="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 --overlap-ms 0 --no-graph-pass"
$CMD > gpurun_out/r2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_resnet50.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_stage_tma|k_resolve" -s 6 -c 3 -o gpurun_out/r2_prof_stage $CMD > gpurun_out/r2_ncu_full.log 2>&1
echo "full capture rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_step_small -s 40 -c 2 -o gpurun_out/r2_prof_small python bench.py --layout mlp --steps 64 --warmup 8 --no-cpu-baseline --e2e-steps 1 --overlap-ms 0 --no-graph-pass > gpurun_out/r2_ncu_small.log 2>&1
echo "small capture rc=$?"
for r in r2_prof_stage r2_prof_small; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,smsp__average_warp_latency_issue_stalled_long_scoreboard > gpurun_out/$r.csv 2>/dev/null
done
