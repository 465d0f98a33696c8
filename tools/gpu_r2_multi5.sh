# 2 GPUs: role split variants; small-step parity + MLP bench
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:2} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_diag4.txt; }
: > gpurun_out/r2_diag4.txt
VAR=split1024 OSP_SHARD_SPLIT=1 OSP_SHARD_PUB=8,4 OSP_SHARD_LAG=10 run 29601 resnet50 1024
VAR=split1024_nofence OSP_SHARD_SPLIT=1 run 29602 resnet50 1024
VAR=split2048 OSP_SHARD_SPLIT=1 OSP_SHARD_PUB=8,4 OSP_SHARD_LAG=10 run 29603 resnet50 2048
VAR=split1024_pub4 OSP_SHARD_SPLIT=1 OSP_SHARD_PUB=4,1 run 29604 resnet50 1024
VAR=split1024_s3 OSP_SHARD_SPLIT=1 OSP_SHARD_PUB=8,4 run 29605 resnet50 1024
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small or pgp_rank or step_host or stage2" 2>&1 | tail -3 > gpurun_out/r2_small.log
timeout 300 python bench.py --layout mlp --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlp_graph.json 2> gpurun_out/r2_mlp_graph.err
timeout 300 python bench.py --layout mlp_acc --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlpacc_graph.json 2> gpurun_out/r2_mlpacc_graph.err
cat gpurun_out/r2_diag4.txt gpurun_out/r2_small.log
for f in r2_mlp_graph r2_mlpacc_graph; do python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step']*1e3, 'us', d['arm'])" 2>/dev/null || tail -3 gpurun_out/$f.err; done
