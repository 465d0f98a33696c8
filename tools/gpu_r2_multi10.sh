# 4 GPUs: the whole multi-GPU suite (final code), then bench lines at P=2 and P=4
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -4 > gpurun_out/r2_multi10.log
cat gpurun_out/r2_multi10.log
for P in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2981$P bench.py --gpus $P --steps 50 --warmup 5 > gpurun_out/r2_bench_p$P.json 2> gpurun_out/r2_bench_p$P.err
python -c "
import json
d=json.loads(open('gpurun_out/r2_bench_p$P.json').read().strip().splitlines()[-1]); print($P, d['ms_per_step'], d['arm']['sync_form'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'])" || tail -3 gpurun_out/r2_bench_p$P.err
done
