# 4 GPUs: barrier form with phase 2 beside phase 1 (segments): parity, then timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_seg2_diag.txt; }
: > gpurun_out/r2_seg2_diag.txt; : > gpurun_out/r2_diag.err
VAR=p4_nseg4 run 29841 4 resnet50
VAR=p4_nseg1 OSP_SHARD_NSEG=1 run 29842 4 resnet50
VAR=p4_nseg8 OSP_SHARD_NSEG=8 run 29843 4 resnet50
VAR=p4_nseg2 OSP_SHARD_NSEG=2 run 29844 4 resnet50
VAR=p4_nseg4_vgg run 29845 4 vgg16
VAR=p4_nseg1_vgg OSP_SHARD_NSEG=1 run 29846 4 vgg16
VAR=p4_nseg4_r152 run 29847 4 resnet152
python -c "
import json
for line in open('gpurun_out/r2_seg2_diag.txt'):
    var, js = line.split(' ',1); d=json.loads(js); print(var, round(d['step_ms'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['sync'])"
grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head -5
