# 2 GPUs: exchange-kernel publication variants (T=2048 and 1024)
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:2} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_diag3.txt; }
: > gpurun_out/r2_diag3.txt
VAR=base2048 OSP_SHARD_LAG=6 run 29601 resnet50 2048
VAR=nofence2048 OSP_SHARD_LAG=6 run 29602 resnet50 2048
VAR=pub8_4 OSP_SHARD_PUB=8,4 OSP_SHARD_LAG=10 run 29603 resnet50 2048
VAR=pub16_8 OSP_SHARD_PUB=16,8 OSP_SHARD_LAG=20 run 29604 resnet50 2048
VAR=base1024 OSP_SHARD_LAG=6 run 29605 resnet50 1024
VAR=nofence1024 OSP_SHARD_LAG=6 run 29606 resnet50 1024
VAR=pub16_8_1024 OSP_SHARD_PUB=16,8 OSP_SHARD_LAG=20 run 29607 resnet50 1024
cat gpurun_out/r2_diag3.txt
