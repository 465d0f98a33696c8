# chain form variants with per-rank counters (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag2.txt; }
: > gpurun_out/r2_chain_diag2.txt
: > gpurun_out/r2_diag.err
export OSP_SHARD_SYNC=chain
VAR=c3 OSP_SHARD_CHAIN_STAGES=3 run 29671 2 resnet50
VAR=c3_1024 OSP_SHARD_CHAIN_STAGES=3 run 29672 2 resnet50 1024
VAR=c3_pre3 OSP_SHARD_CHAIN_STAGES=3 OSP_SHARD_CHAIN_PRE=3 run 29673 2 resnet50
VAR=c3_pre1 OSP_SHARD_CHAIN_STAGES=3 OSP_SHARD_CHAIN_PRE=1 run 29674 2 resnet50
VAR=c3_1024_pre3 OSP_SHARD_CHAIN_STAGES=3 OSP_SHARD_CHAIN_PRE=3 run 29675 2 resnet50 1024
VAR=c3_pub2 OSP_SHARD_CHAIN_STAGES=3 OSP_SHARD_PUB=2,1 run 29676 2 resnet50
cut -c1-1500 gpurun_out/r2_chain_diag2.txt; grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head
