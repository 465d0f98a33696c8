# 2-GPU box: parity (small step), multi-GPU parity, dist bench P=2 (both modes), MLP bench
nvidia-smi topo -m | head -5 > gpurun_out/r2_topo.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or pgp_rank" 2>&1 | tail -4 > gpurun_out/r2_parity4.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -15 > gpurun_out/r2_multi2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/r2_bench_g2.json 2> gpurun_out/r2_bench_g2.err
for lag in 1 4; do OSP_SHARD_LAG=$lag timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 200 --warmup 5 --overlap-ms 0 --e2e-steps 1 > gpurun_out/r2_bench_g2_lag$lag.json 2>> gpurun_out/r2_bench_g2.err; done
timeout 300 python bench.py --layout mlp --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlp_graph.json 2> gpurun_out/r2_mlp_graph.err
timeout 300 python bench.py --layout mlp_acc --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlpacc_graph.json 2> gpurun_out/r2_mlpacc_graph.err
cat gpurun_out/r2_parity4.log gpurun_out/r2_multi2.log
for f in r2_bench_g2 r2_bench_g2_lag1 r2_bench_g2_lag4 r2_mlp_graph r2_mlpacc_graph; do python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d.get('phase_ms'), d.get('roofline',{}).get('frac_vs_bidirectional_667'))" 2>/dev/null || tail -3 gpurun_out/$f.json; done
tail -20 gpurun_out/r2_bench_g2.err
