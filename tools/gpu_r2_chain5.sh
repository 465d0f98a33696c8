# chain form timeline (2 GPUs)
mkdir -p gpurun_out
for L in resnet50 vgg16; do
OSP_SHARD_DEBUG=2 OSP_SHARD_SYNC=chain timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 tools/chain_trace.py $L 2>&1 | grep -v OMP | grep -v "^\*\*" | tail -3
done
