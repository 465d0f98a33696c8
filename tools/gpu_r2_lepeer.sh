# 4 GPUs: barrier form with the peers' local estimates in phase 1: parity, then timing
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_lepeer_diag.txt; }
: > gpurun_out/r2_lepeer_diag.txt; : > gpurun_out/r2_diag.err
VAR=p4_le run 29931 4 resnet50
VAR=p4_nole OSP_SHARD_LE_PEER=0 run 29932 4 resnet50
VAR=p4_le_vgg run 29933 4 vgg16
VAR=p4_nole_vgg OSP_SHARD_LE_PEER=0 run 29934 4 vgg16
VAR=p4_le_b run 29935 4 resnet50
python -c "
import json
for line in open('gpurun_out/r2_lepeer_diag.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],4), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'])"
