# parity (small step, certified façade resolve), drop-in, sharded (oversubscribed), MLP bench
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -8 > gpurun_out/r2_parity3.log
timeout 600 python -m pytest tests/test_dropin.py tests/test_gpu_engine.py -x -q 2>&1 | tail -8 > gpurun_out/r2_dropin.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -15 > gpurun_out/r2_multi.log
timeout 300 python bench.py --layout mlp --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlp_graph.json 2> gpurun_out/r2_mlp_graph.err
timeout 300 python bench.py --layout mlp --steps 2000 --warmup 20 --event-every 100000 --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlp_stream.json 2> gpurun_out/r2_mlp_stream.err
timeout 300 python bench.py --layout mlp_acc --steps 2000 --warmup 20 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_mlpacc_graph.json 2> gpurun_out/r2_mlpacc_graph.err
cat gpurun_out/r2_parity3.log gpurun_out/r2_dropin.log gpurun_out/r2_multi.log
for f in r2_mlp_graph r2_mlp_stream r2_mlpacc_graph; do python -c "
import json,sys
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step']*1e3, 'us', d['arm'].get('single_launch_step'), d['gpu_launches'])" 2>/dev/null || tail -3 gpurun_out/$f.err; done
