# chain form: order / pieces of the remote running-sum copy
mkdir -p gpurun_out
OSP_SHARD_CHAIN_PREMODE=4 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "chain_two" 2>&1 | tail -1
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag22.txt; }
: > gpurun_out/r2_chain_diag22.txt; : > gpurun_out/r2_diag.err
VAR=pm0 run 29921 2 resnet50
VAR=pm1 OSP_SHARD_CHAIN_PREMODE=1 run 29922 2 resnet50
VAR=pm2 OSP_SHARD_CHAIN_PREMODE=2 run 29923 2 resnet50
VAR=pm4 OSP_SHARD_CHAIN_PREMODE=4 run 29924 2 resnet50
VAR=pm0b run 29925 2 resnet50
python -c "
import json
for line in open('gpurun_out/r2_chain_diag22.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],4), {k: round(v,3) for k,v in d['phases_ms'].items()})"
