# chain form: fence scope / batch diagnostics, solo role throughput (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag3.txt; }
: > gpurun_out/r2_chain_diag3.txt
: > gpurun_out/r2_diag.err
export OSP_SHARD_SYNC=chain OSP_SHARD_CHAIN_STAGES=3
VAR=c3 run 29681 2 resnet50
VAR=c3_fgpu OSP_SHARD_CHAIN_FENCE=gpu run 29682 2 resnet50
VAR=c3_pub16 OSP_SHARD_PUB=16,8 run 29683 2 resnet50
VAR=c3_pub16_fgpu OSP_SHARD_CHAIN_FENCE=gpu OSP_SHARD_PUB=16,8 run 29684 2 resnet50
VAR=c3_pre1_fgpu OSP_SHARD_CHAIN_FENCE=gpu OSP_SHARD_CHAIN_PRE=1 run 29685 2 resnet50
cut -c1-1500 gpurun_out/r2_chain_diag3.txt; grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head
