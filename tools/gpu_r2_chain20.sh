# chain form, final defaults: lead and publication-batch knobs (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag21.txt; }
: > gpurun_out/r2_chain_diag21.txt; : > gpurun_out/r2_diag.err
VAR=base run 29911 2 resnet50
VAR=lead1 OSP_SHARD_CHAIN_LEAD=1 run 29912 2 resnet50
VAR=lead8 OSP_SHARD_CHAIN_LEAD=8 run 29913 2 resnet50
VAR=pub4_2 OSP_SHARD_PUB=4,2 run 29914 2 resnet50
VAR=pub16_8 OSP_SHARD_PUB=16,8 run 29915 2 resnet50
VAR=base2 run 29916 2 resnet50
python -c "
import json
for line in open('gpurun_out/r2_chain_diag21.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],4), {k: round(v,3) for k,v in d['phases_ms'].items()})"
