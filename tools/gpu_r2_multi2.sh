# 2 GPUs: exchange-kernel diagnostics sweep, multi tests, bench P=2
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:2} 2>>gpurun_out/r2_diag.err | tail -1 >> gpurun_out/r2_diag.jsonl; }
: > gpurun_out/r2_diag.jsonl
run 29601 resnet50 1024
OSP_SHARD_LAG=0 run 29602 resnet50 1024
OSP_SHARD_LAG=4 run 29603 resnet50 1024
run 29604 resnet50 1024
run 29605 resnet50 2048
run 29606 resnet50 2048
run 29607 resnet50 512
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3 > gpurun_out/r2_multi3.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small" 2>&1 | tail -3 >> gpurun_out/r2_multi3.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/r2_bench_g2.json 2> gpurun_out/r2_bench_g2.err
cat gpurun_out/r2_diag.jsonl gpurun_out/r2_multi3.log; tail -c 1500 gpurun_out/r2_bench_g2.json; grep -i "error\|Traceback" gpurun_out/r2_bench_g2.err gpurun_out/r2_diag.err | head -5
