# 1 GPU: small-step parity + MLP bench + ncu of the single-launch kernel; sanitizers; drop-in at full size
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or pgp_rank" 2>&1 | tail -3 > gpurun_out/r2_small2.log
for L in mlp mlp_acc; do timeout 300 python bench.py --layout $L --steps 3200 --warmup 32 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_${L}_graph.json 2> gpurun_out/r2_${L}_graph.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_small -c 4 -o gpurun_out/r2_step_small_mlpacc python bench.py --layout mlp_acc --steps 32 --warmup 8 --no-cpu-baseline --overlap-ms 0 --e2e-steps 1 --no-graph-pass > gpurun_out/r2_ncu_small.log 2>&1
bash tools/gpu_r2_sanitize.sh > gpurun_out/r2_sanitize_all.txt 2>&1
cat gpurun_out/r2_small2.log
for L in mlp mlp_acc; do python -c "
import json
d=json.loads(open('gpurun_out/r2_${L}_graph.json').read().strip().splitlines()[-1]); print('$L', d['ms_per_step']*1e3, 'us', d['certificate'])" || tail -3 gpurun_out/r2_${L}_graph.err; done
tail -3 gpurun_out/r2_ncu_small.log; cat gpurun_out/r2_sanitize_all.txt | tail -40
