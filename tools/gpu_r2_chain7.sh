# chain form, mixed PRE/APPLY CTAs: parity, trace, variants (2 GPUs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain or ties" 2>&1 | tail -5 > gpurun_out/r2_chain_tests.log
cat gpurun_out/r2_chain_tests.log
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag9.txt; }
: > gpurun_out/r2_chain_diag9.txt
: > gpurun_out/r2_diag.err
export OSP_SHARD_SYNC=chain
VAR=mixed run 29721 2 resnet50
VAR=split2 OSP_SHARD_CHAIN_PRE=2 run 29722 2 resnet50
VAR=mixed_lead12 OSP_SHARD_CHAIN_LEAD=12 run 29723 2 resnet50
VAR=mixed_1024 run 29724 2 resnet50 1024
VAR=mixed_vgg run 29725 2 vgg16
cut -c1-330 gpurun_out/r2_chain_diag9.txt; grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head
OSP_SHARD_DEBUG=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29726 tools/chain_trace.py resnet50 2>&1 | grep layout | cut -c1-300
