# 4 GPUs: segmented form parity, then timing vs the barrier form at P=4 (and P=2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "segment" 2>&1 | tail -4
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_seg_diag.txt; }
: > gpurun_out/r2_seg_diag.txt
VAR=p4_seg4 OSP_SHARD_SYNC=segment run 29821 4 resnet50
VAR=p4_seg8 OSP_SHARD_SYNC=segment OSP_SHARD_NSEG=8 run 29822 4 resnet50
VAR=p4_seg2 OSP_SHARD_SYNC=segment OSP_SHARD_NSEG=2 run 29823 4 resnet50
VAR=p4_barrier OSP_SHARD_SYNC=barrier run 29824 4 resnet50
VAR=p4_seg4_vgg OSP_SHARD_SYNC=segment run 29825 4 vgg16
VAR=p2_seg4 OSP_SHARD_SYNC=segment run 29826 2 resnet50
python -c "
import json
for line in open('gpurun_out/r2_seg_diag.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'])"
grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head -5
