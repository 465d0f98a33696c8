# chain form of the sharded stage 1: parity (2 GPUs + oversubscribed), then timing vs tile flags
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain" 2>&1 | tail -15 > gpurun_out/r2_chain_tests.log
cat gpurun_out/r2_chain_tests.log
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag.txt; }
: > gpurun_out/r2_chain_diag.txt
: > gpurun_out/r2_diag.err
if grep -q passed gpurun_out/r2_chain_tests.log && ! grep -q failed gpurun_out/r2_chain_tests.log; then
VAR=p2_chain OSP_SHARD_SYNC=chain run 29661 2 resnet50
VAR=p2_chain3 OSP_SHARD_CHAIN_STAGES=3 OSP_SHARD_SYNC=chain run 29662 2 resnet50
VAR=p2_chain1024 OSP_SHARD_SYNC=chain run 29663 2 resnet50 1024
VAR=p2_tile OSP_SHARD_SYNC=tile run 29664 2 resnet50
VAR=p2_vgg_chain OSP_SHARD_SYNC=chain run 29665 2 vgg16
fi
cut -c1-600 gpurun_out/r2_chain_diag.txt; tail -20 gpurun_out/r2_diag.err
