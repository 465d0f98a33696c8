# chain form with role-sized ring slots: parity, then variants (2 GPUs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain" 2>&1 | tail -5 > gpurun_out/r2_chain_tests.log
cat gpurun_out/r2_chain_tests.log
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag4.txt; }
: > gpurun_out/r2_chain_diag4.txt
: > gpurun_out/r2_diag.err
export OSP_SHARD_SYNC=chain
VAR=a200 run 29691 2 resnet50
VAR=a200_pre3 OSP_SHARD_CHAIN_PRE=3 run 29692 2 resnet50
VAR=a200_pre1 OSP_SHARD_CHAIN_PRE=1 run 29693 2 resnet50
VAR=a120 OSP_SHARD_CHAIN_ARENA_KB=120 run 29694 2 resnet50
VAR=a200_1024 run 29695 2 resnet50 1024
VAR=a200_vgg run 29696 2 vgg16
cut -c1-1500 gpurun_out/r2_chain_diag4.txt; grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head
