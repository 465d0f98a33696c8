# 4 GPUs: multi tests (2 and 4 ranks), bench P=2 and P=4 with the new defaults
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 > gpurun_out/r2_multi5.log
for P in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2962$P bench.py --gpus $P --steps 200 --warmup 5 > gpurun_out/r2_bench_g$P.json 2> gpurun_out/r2_bench_g$P.err; done
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_diag5.txt; }
: > gpurun_out/r2_diag5.txt
VAR=p4_2048 run 29631 4 resnet50 2048
VAR=p4_1024 run 29632 4 resnet50 1024
VAR=p4_nosplit OSP_SHARD_SPLIT=0 OSP_SHARD_PUB=8,4 run 29633 4 resnet50 2048
VAR=p2_vgg run 29634 2 vgg16
VAR=p4_vgg run 29635 4 vgg16
cat gpurun_out/r2_multi5.log gpurun_out/r2_diag5.txt
for P in 2 4; do python -c "
import json
d=json.loads(open('gpurun_out/r2_bench_g$P.json').read().strip().splitlines()[-1]); o=d['overlap'] or {}; o.pop('closed_loop',None)
print($P, d['ms_per_step'], d['phase_ms'], d['roofline']['frac_vs_bidirectional_667'], d['e2e']['ms_per_step'], o)" || tail -5 gpurun_out/r2_bench_g$P.err; done
