# chain form: single-lane copy issue; 2 CTAs/SM at T=1024 (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag12.txt; }
: > gpurun_out/r2_chain_diag12.txt
export OSP_SHARD_SYNC=chain
VAR=onelane run 29761 2 resnet50
VAR=onelane_1024_a100 OSP_SHARD_CHAIN_ARENA_KB=100 run 29762 2 resnet50 1024
VAR=onelane_1024_a72 OSP_SHARD_CHAIN_ARENA_KB=72 run 29763 2 resnet50 1024
VAR=onelane_a112 OSP_SHARD_CHAIN_ARENA_KB=112 run 29764 2 resnet50
