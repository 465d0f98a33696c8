# chain form: the last rank with G from HBM and two CTAs per SM
mkdir -p gpurun_out
OSP_SHARD_CHAIN_PUSHAGG=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "chain_two or chain_oversubscribed" 2>&1 | tail -2
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag19.txt; }
: > gpurun_out/r2_chain_diag19.txt; : > gpurun_out/r2_diag.err
VAR=base run 29891 2 resnet50
VAR=pushagg OSP_SHARD_CHAIN_PUSHAGG=1 run 29892 2 resnet50
VAR=pushagg_vgg OSP_SHARD_CHAIN_PUSHAGG=1 run 29893 2 vgg16
VAR=base_vgg run 29894 2 vgg16
python -c "
import json
for line in open('gpurun_out/r2_chain_diag19.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'], d['solo_ms_per_rank'])"
grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head -5
