for l in resnet50 resnet152 vgg16; do
timeout 300 python bench.py --layout $l --no-cpu-baseline --e2e-steps 2 --overlap-ms 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['breakdown_ms'].items() if k!='note'}, round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3))"
done
