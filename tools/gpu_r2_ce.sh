# copy-engine probe (2+ GPUs) + single-launch small step parity and MLP graph bench
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ce_probe.cu -o /tmp/ce_probe && timeout 300 /tmp/ce_probe > gpurun_out/r2_ce_probe.txt 2>&1
cat gpurun_out/r2_ce_probe.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small" 2>&1 | tail -3
for L in mlp mlp_acc; do timeout 300 python bench.py --layout $L --steps 3200 --warmup 32 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_${L}_graph.json 2> gpurun_out/r2_${L}_graph.err; python -c "
import json
d=json.loads(open('gpurun_out/r2_${L}_graph.json').read().strip().splitlines()[-1]); print('$L', d['ms_per_step']*1e3, 'us')" || tail -3 gpurun_out/r2_${L}_graph.err; done
