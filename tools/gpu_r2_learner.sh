# the gradient producer: tests, smoke, MLP bench lines with the training pass
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_learner.py -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py 2>&1 | tail -2
for L in mlp mlp_acc; do timeout 600 python bench.py --layout $L --steps 3200 --warmup 32 --graph --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_${L}_train.json 2> gpurun_out/r2_${L}_train.err
python -c "
import json
d=json.loads(open('gpurun_out/r2_${L}_train.json').read().strip().splitlines()[-1]); t=d['training']; print('$L sync', round(d['ms_per_step']*1e3,2), 'us; training', round(t['us_per_iteration'],2), 'us, producer', round(t['producer_us'],2), 'us; ref', t.get('reference_cpu'))" || tail -5 gpurun_out/r2_${L}_train.err; done
