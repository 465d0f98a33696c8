# 4 GPUs: the chain (final defaults) at P=4 against the barrier form
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag20.txt; }
: > gpurun_out/r2_chain_diag20.txt; : > gpurun_out/r2_diag.err
VAR=p4_chain OSP_SHARD_SYNC=chain run 29901 4 resnet50
VAR=p4_barrier run 29902 4 resnet50
VAR=p4_chain_vgg OSP_SHARD_SYNC=chain run 29903 4 vgg16
VAR=p4_chain_a0_200 OSP_SHARD_SYNC=chain OSP_SHARD_CHAIN_ARENA_KB0=200 run 29904 4 resnet50
python -c "
import json
for line in open('gpurun_out/r2_chain_diag20.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'])"
