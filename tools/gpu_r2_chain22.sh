# chain form (final defaults): running sums pushed (NVLink stores) vs pulled
mkdir -p gpurun_out
OSP_SHARD_CHAIN_PUSHPRE=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "chain_two" 2>&1 | tail -1
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag23.txt; }
: > gpurun_out/r2_chain_diag23.txt; : > gpurun_out/r2_diag.err
VAR=pull run 29941 2 resnet50
VAR=push OSP_SHARD_CHAIN_PUSHPRE=1 run 29942 2 resnet50
VAR=push_vgg OSP_SHARD_CHAIN_PUSHPRE=1 run 29943 2 vgg16
VAR=pull_vgg run 29944 2 vgg16
python -c "
import json
for line in open('gpurun_out/r2_chain_diag23.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],4), {k: round(v,3) for k,v in d['phases_ms'].items()})"
