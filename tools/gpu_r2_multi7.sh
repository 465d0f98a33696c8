# 4 GPUs: tile vs barrier sync at P=2/4; multi tests at 4
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_diag6.txt; }
: > gpurun_out/r2_diag6.txt
VAR=p4_barrier OSP_SHARD_SYNC=barrier run 29641 4 resnet50
VAR=p4_tile OSP_SHARD_SYNC=tile run 29642 4 resnet50
VAR=p4_barrier1024 OSP_SHARD_SYNC=barrier run 29643 4 resnet50 1024
VAR=p2_barrier OSP_SHARD_SYNC=barrier run 29644 2 resnet50
VAR=p2_tile OSP_SHARD_SYNC=tile run 29645 2 resnet50
VAR=p4_vgg_barrier OSP_SHARD_SYNC=barrier run 29646 4 vgg16
VAR=p2_vgg_barrier OSP_SHARD_SYNC=barrier run 29647 2 vgg16
VAR=p4_r152_barrier OSP_SHARD_SYNC=barrier run 29648 4 resnet152
VAR=p2_r152_tile run 29649 2 resnet152
OSP_SHARD_SYNC=barrier timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 > gpurun_out/r2_multi6.log
cat gpurun_out/r2_diag6.txt gpurun_out/r2_multi6.log
