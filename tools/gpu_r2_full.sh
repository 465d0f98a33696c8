# the driver's view: the whole GPU suite, smoke, the default bench; plus MLP lines
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_gpu_suite.log
timeout 300 python __graft_entry__.py > gpurun_out/r2_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
for L in mlp mlp_acc; do timeout 300 python bench.py --layout $L --steps 3200 --warmup 32 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_${L}_graph.json 2> gpurun_out/r2_${L}_graph.err; done
cat gpurun_out/r2_gpu_suite.log gpurun_out/r2_smoke.log
for L in mlp mlp_acc; do python -c "
import json
d=json.loads(open('gpurun_out/r2_${L}_graph.json').read().strip().splitlines()[-1]); print('$L', d['ms_per_step']*1e3, 'us')" || tail -3 gpurun_out/r2_${L}_graph.err; done
python -c "
import json
d=json.loads(open('gpurun_out/r2_bench_default.json').read().strip().splitlines()[-1]); o=d['overlap']; cl=o.pop('closed_loop')
print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['step_frac'], d['e2e']['ms_per_step'], o, cl['epoch_budgets'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
tail -1 gpurun_out/r2_bench_reference.json | cut -c1-400
