# 4 GPUs: chain vs barrier/tile at P=4 and P=2; chain parity at 4 GPUs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain_four or chain_two" 2>&1 | tail -3
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag14.txt; }
: > gpurun_out/r2_chain_diag14.txt
VAR=p4_chain OSP_SHARD_SYNC=chain run 29781 4 resnet50
VAR=p4_barrier OSP_SHARD_SYNC=barrier run 29782 4 resnet50
VAR=p4_chain_vgg OSP_SHARD_SYNC=chain run 29783 4 vgg16
VAR=p4_barrier_vgg OSP_SHARD_SYNC=barrier run 29784 4 vgg16
VAR=p2_chain OSP_SHARD_SYNC=chain run 29785 2 resnet50
VAR=p2_tile OSP_SHARD_SYNC=tile run 29786 2 resnet50
VAR=p2_chain_r152 OSP_SHARD_SYNC=chain run 29787 2 resnet152
VAR=p4_chain_r152 OSP_SHARD_SYNC=chain run 29788 4 resnet152
VAR=p4_barrier_r152 OSP_SHARD_SYNC=barrier run 29789 4 resnet152
