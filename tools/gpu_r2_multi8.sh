# 4 GPUs: barrier form (peer-apply kernel) vs tile flags at P=2/4; multi tests in both
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_diag7.txt; }
: > gpurun_out/r2_diag7.txt
VAR=p4_barrier OSP_SHARD_SYNC=barrier run 29651 4 resnet50
VAR=p4_barrier1024 OSP_SHARD_SYNC=barrier run 29652 4 resnet50 1024
VAR=p2_barrier OSP_SHARD_SYNC=barrier run 29653 2 resnet50
VAR=p2_barrier1024 OSP_SHARD_SYNC=barrier run 29654 2 resnet50 1024
VAR=p2_tile OSP_SHARD_SYNC=tile run 29655 2 resnet50
VAR=p4_vgg_barrier OSP_SHARD_SYNC=barrier run 29656 4 vgg16
VAR=p2_vgg_barrier OSP_SHARD_SYNC=barrier run 29657 2 vgg16
VAR=p2_vgg_tile OSP_SHARD_SYNC=tile run 29658 2 vgg16
OSP_SHARD_SYNC=barrier timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 > gpurun_out/r2_multi7.log
OSP_SHARD_SYNC=tile timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 >> gpurun_out/r2_multi7.log
cat gpurun_out/r2_diag7.txt | cut -c1-400; cat gpurun_out/r2_multi7.log
