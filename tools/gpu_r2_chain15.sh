# chain form: G from HBM in the consumers (no G row in the ring), 4096-element tiles
mkdir -p gpurun_out
OSP_SHARD_CHAIN_GGLOBAL=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain_two or chain_oversubscribed" 2>&1 | tail -2
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag16.txt; }
: > gpurun_out/r2_chain_diag16.txt; : > gpurun_out/r2_diag.err
VAR=base run 29831 2 resnet50
VAR=gg OSP_SHARD_CHAIN_GGLOBAL=1 run 29832 2 resnet50
VAR=gg4096 OSP_SHARD_CHAIN_GGLOBAL=1 run 29833 2 resnet50 4096
VAR=base_b run 29834 2 resnet50
VAR=gg4096_vgg OSP_SHARD_CHAIN_GGLOBAL=1 run 29835 2 vgg16 4096
VAR=base_vgg run 29836 2 vgg16
python -c "
import json
for line in open('gpurun_out/r2_chain_diag16.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, d['tile'], round(d['step_ms'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'], [round(c['issue_cycles']/148/1.9e3,1) for c in d['debug_per_step']])"
grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head -5
