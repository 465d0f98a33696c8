# 2 GPUs: exchange-kernel diagnostics, multi tests, bench P=2
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:2} 2>>gpurun_out/r2_diag.err | tail -1 >> gpurun_out/r2_diag2.jsonl; }
: > gpurun_out/r2_diag2.jsonl
run 29601 resnet50 1024
run 29605 resnet50 2048
OSP_SHARD_LAG=6 run 29602 resnet50 2048
run 29607 resnet50 4096
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 > gpurun_out/r2_multi4.log
cat gpurun_out/r2_diag2.jsonl gpurun_out/r2_multi4.log; grep -i "error\|Traceback" gpurun_out/r2_diag.err | head -5
