set -x
free -g | head -2; nproc; nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 900 python -m pytest tests/test_gpu_multi.py -k "oversub" -x -q 2>&1 | tail -15 > gpurun_out/r2_multi_oversub.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | tail -15 > gpurun_out/r2_fullsize.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -8 > gpurun_out/r2_parity.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2>&1
cat gpurun_out/r2_multi_oversub.log gpurun_out/r2_fullsize.log gpurun_out/r2_parity.log
tail -c 600 gpurun_out/r2_bench.json
