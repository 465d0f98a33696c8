# 2 GPUs: the whole multi-GPU suite with the chain default, then the P=2 bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -4 > gpurun_out/r2_multi9.log
cat gpurun_out/r2_multi9.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/r2_bench_p2.json 2> gpurun_out/r2_bench_p2.err
tail -1 gpurun_out/r2_bench_p2.json | cut -c1-600
