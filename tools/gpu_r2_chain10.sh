# chain form: producer phase counters, per-rank solo (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag11.txt; }
: > gpurun_out/r2_chain_diag11.txt
export OSP_SHARD_SYNC=chain
VAR=mixed run 29751 2 resnet50
VAR=split2 OSP_SHARD_CHAIN_PRE=2 run 29752 2 resnet50
