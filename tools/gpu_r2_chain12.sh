# chain form: pushed running sums vs pulled (2 GPUs); parity of the push variant
mkdir -p gpurun_out
OSP_SHARD_CHAIN_PUSH=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain or ties" 2>&1 | tail -3
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag13.txt; }
: > gpurun_out/r2_chain_diag13.txt
export OSP_SHARD_SYNC=chain
VAR=pull run 29771 2 resnet50
VAR=push OSP_SHARD_CHAIN_PUSH=1 run 29772 2 resnet50
VAR=push_pub16 OSP_SHARD_PUB=16,8 OSP_SHARD_CHAIN_PUSH=1 run 29773 2 resnet50
VAR=push_vgg OSP_SHARD_CHAIN_PUSH=1 run 29774 2 vgg16
VAR=pull_vgg run 29775 2 vgg16
