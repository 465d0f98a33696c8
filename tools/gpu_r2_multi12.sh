# 2 GPUs: the multi-GPU suite with the final chain defaults, then the P=2 bench line and a trace
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -2 > gpurun_out/r2_multi12.log; cat gpurun_out/r2_multi12.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/r2_bench_p2.json 2> gpurun_out/r2_bench_p2.err
python -c "
import json
d=json.loads(open('gpurun_out/r2_bench_p2.json').read().strip().splitlines()[-1]); print(2, d['ms_per_step'], d['arm']['sync_form'], round(d['roofline']['achieved']), d['e2e']['ms_per_step'], d['clocks'])" || tail -3 gpurun_out/r2_bench_p2.err
OSP_SHARD_DEBUG=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29872 tools/chain_trace.py resnet50 2>&1 | grep layout | cut -c1-200
