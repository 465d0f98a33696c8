df -h /tmp . | tail -2
LAYOUTS="vgg16" bash tools/dropin_bench.sh > /dev/null 2>&1; cp gpurun_out/dropin_bench.txt gpurun_out/r2_dropin_vgg.txt
bash tools/gpu_r2_profile.sh
for L in mlp mlp_acc; do timeout 300 python bench.py --layout $L --steps 3200 --warmup 32 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 > gpurun_out/r2_${L}_graph.json 2> gpurun_out/r2_${L}_graph.err; done
bash tools/gpu_r2_checked.sh
cat gpurun_out/r2_dropin_vgg.txt
for L in mlp mlp_acc; do python -c "
import json
d=json.loads(open('gpurun_out/r2_${L}_graph.json').read().strip().splitlines()[-1]); print('$L', d['ms_per_step']*1e3, 'us')" || tail -3 gpurun_out/r2_${L}_graph.err; done
head -12 gpurun_out/r2_prof_stage.csv | cut -c1-300; head -5 gpurun_out/r2_prof_small.csv | cut -c1-300
