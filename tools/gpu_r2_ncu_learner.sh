# ncu of the gradient producer (one launch each for [8,32,4] and [16,64,64,4])
mkdir -p gpurun_out
for L in mlp mlp_acc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_grad -c 1 -f -o gpurun_out/r2_learner_$L python bench.py --layout $L --steps 32 --warmup 4 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 1 > gpurun_out/r2_ncu_learner_$L.log 2>&1; echo ncu_$L=$?
ncu -i gpurun_out/r2_learner_$L.ncu-rep --page details --csv > gpurun_out/r2_learner_${L}_details.csv 2>/dev/null
grep -E '"Duration"|"Compute \(SM\) Throughput"|"Memory Throughput"|"Achieved Occupancy"|"Registers Per Thread"|"Executed Ipc Active"|"Dynamic Shared Memory Per Block"' gpurun_out/r2_learner_${L}_details.csv | cut -c1-200 | head -12
done
