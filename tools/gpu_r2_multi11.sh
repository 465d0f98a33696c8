# 4 GPUs: final P=2 / P=4 bench lines
mkdir -p gpurun_out
for P in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2985$P bench.py --gpus $P --steps 50 --warmup 5 > gpurun_out/r2_bench_p$P.json 2> gpurun_out/r2_bench_p$P.err
python -c "
import json
d=json.loads(open('gpurun_out/r2_bench_p$P.json').read().strip().splitlines()[-1]); print($P, d['ms_per_step'], d['arm']['sync_form'], round(d['roofline']['achieved']), d['e2e']['ms_per_step'], d['e2e']['sync_steps']['ms_per_step'], d['clocks'])" || tail -3 gpurun_out/r2_bench_p$P.err
done
