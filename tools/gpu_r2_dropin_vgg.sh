# the VGG-16 façade flow against the reference engines: where do they differ?
lf=/tmp/osp_layers_vgg16.txt
python -c "from paper_2306_16926_b200 import layouts; print(','.join(map(str, layouts.get('vgg16'))))" > $lf
args="--layers-file $lf --workers 8 --budget-frac 0.5 --chunks 4 --seed 11"
rm -rf /tmp/g_ref /tmp/g_dev; mkdir -p /tmp/g_ref /tmp/g_dev
timeout 900 oracle/_ref/ref_driver golden $args --iters 3 --out /tmp/g_ref > /dev/null
timeout 900 oracle/_ref/dropin_driver golden $args --iters 3 --out /tmp/g_dev > /dev/null
python tools/dropin_diff.py /tmp/g_ref /tmp/g_dev > gpurun_out/r2_dropin_vgg_diff.txt 2>&1
cat gpurun_out/r2_dropin_vgg_diff.txt | head -60
